// Instantiates the double large-N IsoRank kernels (see tiers.h).
#define CFGSIM_TIER_TU
#include "tiers.h"

CFGSIM_BIG_LIST_T(double, CFGSIM_INSTANTIATE_BIG)
