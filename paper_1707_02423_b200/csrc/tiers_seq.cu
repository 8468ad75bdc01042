// Instantiates the two-stage small-N IsoRank kernels (isorank_seq.cuh).
#define CFGSIM_TIER_TU
#include "tiers.h"

template __global__ void cfgsim::isorank_seq_kernel<double, 2>(cfgsim::DevCorpus, cfgsim::SeqCombos, cfgsim::SeqParams,
                                                               double *, double *);
template __global__ void cfgsim::isorank_seq_kernel<float, 2>(cfgsim::DevCorpus, cfgsim::SeqCombos, cfgsim::SeqParams,
                                                              float *, double *);
#define CFGSIM_P2(T, KB, AR, BC, PW, MINB)                                                          \
  template __global__ void cfgsim::isorank_pair2_kernel<T, KB, AR, BC, PW, MINB>(                  \
      const int32_t *, cfgsim::PairWork, cfgsim::PairOut, cfgsim::Pair2Params, const T *, const double *, \
      const int64_t *, unsigned long long *);
CFGSIM_P2_LIST(CFGSIM_P2)
template __global__ void cfgsim::isorank_seq4_kernel<double, 2>(cfgsim::DevCorpus, cfgsim::SeqCombos, cfgsim::SeqParams,
                                                                double *, double *);
template __global__ void cfgsim::isorank_seq4_kernel<float, 2>(cfgsim::DevCorpus, cfgsim::SeqCombos, cfgsim::SeqParams,
                                                               float *, double *);
