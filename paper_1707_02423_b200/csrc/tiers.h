// Tier kernel instantiations live in tiers_f64.cu / tiers_f32.cu (compiled in
// parallel); cfgsim.cu only takes their addresses.
#pragma once
#include "isorank.cuh"
#include "isorank_lr.cuh"
#include "isorank_big.cuh"
#include "isorank_seq.cuh"

#define CFGSIM_TIER_LIST(X)      \
  X(double, 1, 4, 4, 6)          \
  X(double, 2, 8, 4, 3)          \
  X(double, 4, 16, 4, 1)         \
  X(float, 1, 4, 4, 6)           \
  X(float, 2, 8, 4, 3)           \
  X(float, 4, 16, 4, 1)

#define CFGSIM_EXTERN_TIER(T, KB, NW, R, MINB)                                              \
  extern template __global__ void cfgsim::isorank_pair_kernel<T, KB, NW, R, MINB>(         \
      cfgsim::DevCorpus, cfgsim::DevCorpus, cfgsim::PairWork, cfgsim::PairOut,              \
      cfgsim::PairParams, unsigned long long *);
#define CFGSIM_INSTANTIATE_TIER(T, KB, NW, R, MINB)                                         \
  template __global__ void cfgsim::isorank_pair_kernel<T, KB, NW, R, MINB>(                \
      cfgsim::DevCorpus, cfgsim::DevCorpus, cfgsim::PairWork, cfgsim::PairOut,              \
      cfgsim::PairParams, unsigned long long *);

#define CFGSIM_EXTERN_LR(T, KB, AR, BC, MAXT, MINB)                                                     \
  extern template __global__ void cfgsim::isorank_lowrank_kernel<T, KB, AR, BC, MAXT, MINB>(           \
      cfgsim::DevCorpus, cfgsim::DevCorpus, cfgsim::PairWork, cfgsim::PairOut,              \
      cfgsim::LRParams, unsigned long long *);
#define CFGSIM_INSTANTIATE_LR(T, KB, AR, BC, MAXT, MINB)                                                \
  template __global__ void cfgsim::isorank_lowrank_kernel<T, KB, AR, BC, MAXT, MINB>(                  \
      cfgsim::DevCorpus, cfgsim::DevCorpus, cfgsim::PairWork, cfgsim::PairOut,              \
      cfgsim::LRParams, unsigned long long *);
#define CFGSIM_LR_LIST(X) \
  X(double, 1, 4, 4, 64, 10)  \
  X(double, 2, 4, 8, 128, 4)  \
  X(double, 4, 4, 8, 512, 1)  \
  X(float, 1, 4, 4, 64, 10)   \
  X(float, 2, 4, 8, 128, 5)   \
  X(float, 4, 4, 8, 512, 1)

#define CFGSIM_EXTERN_BIG(T, KB)                                                              \
  extern template __global__ void cfgsim::isorank_big_kernel<T, KB>(                         \
      cfgsim::DevCorpus, cfgsim::DevCorpus, cfgsim::PairWork, cfgsim::PairOut,              \
      cfgsim::BigParams, unsigned long long *);
#define CFGSIM_INSTANTIATE_BIG(T, KB)                                                         \
  template __global__ void cfgsim::isorank_big_kernel<T, KB>(                                \
      cfgsim::DevCorpus, cfgsim::DevCorpus, cfgsim::PairWork, cfgsim::PairOut,              \
      cfgsim::BigParams, unsigned long long *);
// KB = sort chunks per lane: N <= 32 * KB
#define CFGSIM_BIG_LIST_T(T, X) X(T, 8) X(T, 16) X(T, 32)

// two-stage pair kernels: (T, KB, AR, BC, producer warps, MINB)
#define CFGSIM_P2_LIST(X) \
  X(double, 1, 4, 4, 2, 4) X(double, 2, 4, 8, 4, 2) X(float, 1, 4, 4, 2, 4) X(float, 2, 4, 8, 4, 2) \
  X(double, 2, 4, 8, 4, 3) X(float, 2, 4, 8, 4, 3) X(double, 1, 4, 4, 2, 6) X(float, 1, 4, 4, 2, 6) \
  X(double, 2, 4, 6, 4, 3) X(float, 2, 4, 6, 4, 3)
#define CFGSIM_EXTERN_P2(T, KB, AR, BC, PW, MINB)                                                   \
  extern template __global__ void cfgsim::isorank_pair2_kernel<T, KB, AR, BC, PW, MINB>(           \
      const int32_t *, cfgsim::PairWork, cfgsim::PairOut, cfgsim::Pair2Params, const T *, const double *, \
      const int64_t *, unsigned long long *);

#ifndef CFGSIM_TIER_TU
CFGSIM_P2_LIST(CFGSIM_EXTERN_P2)
extern template __global__ void cfgsim::isorank_seq_kernel<double, 2>(cfgsim::DevCorpus, cfgsim::SeqCombos,
                                                                      cfgsim::SeqParams, double *, double *);
extern template __global__ void cfgsim::isorank_seq_kernel<float, 2>(cfgsim::DevCorpus, cfgsim::SeqCombos,
                                                                     cfgsim::SeqParams, float *, double *);
extern template __global__ void cfgsim::isorank_seq4_kernel<double, 2>(cfgsim::DevCorpus, cfgsim::SeqCombos,
                                                                       cfgsim::SeqParams, double *, double *);
extern template __global__ void cfgsim::isorank_seq4_kernel<float, 2>(cfgsim::DevCorpus, cfgsim::SeqCombos,
                                                                      cfgsim::SeqParams, float *, double *);
CFGSIM_BIG_LIST_T(double, CFGSIM_EXTERN_BIG)
extern template __global__ void cfgsim::isorank_seqbig_kernel<8>(cfgsim::DevCorpus, cfgsim::SeqBigCombos,
                                                                   cfgsim::BigParams);
CFGSIM_BIG_LIST_T(float, CFGSIM_EXTERN_BIG)
CFGSIM_TIER_LIST(CFGSIM_EXTERN_TIER)
CFGSIM_LR_LIST(CFGSIM_EXTERN_LR)
#endif
