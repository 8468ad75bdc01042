// Instantiates the double large-N IsoRank kernels (see tiers.h).
#define CFGSIM_TIER_TU
#include "tiers.h"

CFGSIM_BIG_LIST_T(double, CFGSIM_INSTANTIATE_BIG)
template __global__ void cfgsim::isorank_seqbig_kernel<8>(cfgsim::DevCorpus, cfgsim::SeqBigCombos, cfgsim::BigParams);
