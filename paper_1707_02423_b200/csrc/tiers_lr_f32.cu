// Instantiates the float low-rank IsoRank kernels (see tiers.h).
#define CFGSIM_TIER_TU
#include "tiers.h"

CFGSIM_INSTANTIATE_LR(float, 1, 4, 4, 64, 10)
CFGSIM_INSTANTIATE_LR(float, 2, 4, 8, 128, 5)
CFGSIM_INSTANTIATE_LR(float, 4, 4, 8, 512, 1)
