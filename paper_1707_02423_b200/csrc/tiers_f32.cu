// Instantiates the float IsoRank tier kernels (see tiers.h).
#define CFGSIM_TIER_TU
#include "tiers.h"

CFGSIM_INSTANTIATE_TIER(float, 1, 4, 4, 6)
CFGSIM_INSTANTIATE_TIER(float, 2, 8, 4, 3)
CFGSIM_INSTANTIATE_TIER(float, 4, 16, 4, 1)
