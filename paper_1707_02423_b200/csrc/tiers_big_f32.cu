// Instantiates the float large-N IsoRank kernels (see tiers.h).
#define CFGSIM_TIER_TU
#include "tiers.h"

CFGSIM_BIG_LIST_T(float, CFGSIM_INSTANTIATE_BIG)
