// Instantiates the double low-rank IsoRank kernels (see tiers.h).
#define CFGSIM_TIER_TU
#include "tiers.h"

CFGSIM_INSTANTIATE_LR(double, 1, 4, 4, 64, 10)
CFGSIM_INSTANTIATE_LR(double, 2, 4, 8, 128, 4)
CFGSIM_INSTANTIATE_LR(double, 4, 4, 8, 512, 1)
