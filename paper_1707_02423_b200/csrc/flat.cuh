// Flat measures on size-normalised matrices:
//   euclidean  sqrt(sum |x-y|^2)               similarity.py:35-37
//   manhattan  sum |x-y|                       :40-42
//   minkowski  (sum |x-y|^p)^(1/p), p >= 1     :45-49
//   jaccard    sum (x-y)^2 / (x.x + y.y - x.y) :52-57
//   cosine     1 - x.y / (|x| |y|)             :60-66
// after normalize_pair (matrix.py:109-114): the smaller matrix is upscaled by
// interpolate_to (matrix.py:74-106), evaluated here on the fly with the
// reference's expression order (bit-identical entries), so the only
// difference from the reference is the summation order of the sums (numpy's
// pairwise sum over the flattened N^2 vector vs a fixed-order block
// reduction: deterministic, within a few ulps).
//
// One 128-thread CTA per pair; output row p at a time: the (up to two)
// source rows of each side are densified in shared memory, then every thread
// takes columns q = tid, tid + 128, ...
#pragma once
#include <math_constants.h>

#include "isorank.cuh"

namespace cfgsim {

enum { FLAT_EUC = 0, FLAT_MAN = 1, FLAT_MIN = 2, FLAT_JAC = 3, FLAT_COS = 4, FLAT_ALL = 5 };
constexpr int FLAT_THREADS = 128;

struct FlatWork {
  int32_t mode;       // 0: pair list (ia, ib, out[q]); 1: upper triangle a < b of one corpus, K x K output
  int64_t n_items;
  const int32_t *ia, *ib;
  int32_t K;
  int32_t measure;
  double p;
  int32_t nlim;       // max source size (shared row buffers)
  int64_t out_stride; // FLAT_ALL: measure m's outputs at out + m * out_stride
};

// FLAT_ALL (`compare --measure all`, cli.py:154-164): the five measures from
// ONE walk over each pair's size-normalised entries — the six sums share
// every interpolated entry, so the five reference pairwise() passes
// (similarity.py:247-255 per measure) become one kernel pass.

// source side of one pair: dense rows staged on demand
struct FlatSide {
  int n, N;
  const int32_t *rp, *cc;
  const double *rv;
};

__device__ __forceinline__ void flat_lofr(int t, int n, int N, int &l, double &f) {
  const double pos = __ddiv_rn((double)((long long)t * (n - 1)), (double)(N - 1));  // matrix.py:93
  l = (int)floor(pos);
  if (l > n - 2) l = n - 2;  // :94
  f = __dsub_rn(pos, (double)l);  // :95
}

// value of interpolate_to(side, N)[p, q] from dense source rows r0 (and r1)
__device__ __forceinline__ double flat_value(const FlatSide &S, const double *r0, const double *r1, double frp,
                                             int q) {
  if (S.n == S.N) return r0[q];
  if (S.n == 1) return r0[0];  // matrix.py:87-89
  int lq;
  double fq;
  flat_lofr(q, S.n, S.N, lq, fq);
  const double omc = __dsub_rn(1.0, fq);  // matrix.py:104, left to right, no contraction
  const double top = __dadd_rn(__dmul_rn(omc, r0[lq]), __dmul_rn(fq, r0[lq + 1]));
  const double bot = __dadd_rn(__dmul_rn(omc, r1[lq]), __dmul_rn(fq, r1[lq + 1]));
  return __dadd_rn(__dmul_rn(__dsub_rn(1.0, frp), top), __dmul_rn(frp, bot));
}

__global__ void __launch_bounds__(FLAT_THREADS)
    flat_pair_kernel(DevCorpus CA, DevCorpus CB, FlatWork work, double *out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *rows = (double *)smem_raw;  // 4 rows of nlim doubles: A r0, A r1, B r0, B r1
  __shared__ double red[6][FLAT_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = work.nlim;
  for (int64_t item = blockIdx.x; item < work.n_items; item += gridDim.x) {
    int a, b;
    int64_t o1 = -1, o2 = -1;
    if (work.mode == 0) {
      a = work.ia[item];
      b = work.ib[item];
      o1 = item;
    } else {  // unit -> (a < b): row a holds K - 1 - a units
      const int64_t K = work.K;
      const double bq = 2.0 * (double)K - 1.0;
      int64_t r = (int64_t)((bq - sqrt(bq * bq - 8.0 * (double)item)) * 0.5);
      auto rs = [&](int64_t x) { return x * (K - 1) - x * (x - 1) / 2; };
      if (r < 0) r = 0;
      if (r > K - 2) r = K - 2;
      while (r > 0 && rs(r) > item) r--;
      while (r + 1 < K - 1 && rs(r + 1) <= item) r++;
      a = (int)r;
      b = (int)(r + 1 + (item - rs(r)));
      o1 = (int64_t)a * K + b;
      o2 = (int64_t)b * K + a;
    }
    FlatSide SA, SB;
    SA.n = CA.n_nodes[a];
    SB.n = CB.n_nodes[b];
    const int N = SA.n > SB.n ? SA.n : SB.n;
    SA.N = SB.N = N;
    SA.rp = CA.rowptr + CA.rp_off[a];
    SA.cc = CA.col + CA.nz_off[a];
    SA.rv = CA.val + CA.nz_off[a];
    SB.rp = CB.rowptr + CB.rp_off[b];
    SB.cc = CB.col + CB.nz_off[b];
    SB.rv = CB.val + CB.nz_off[b];
    double s2 = 0.0, s1 = 0.0, sp = 0.0, sxx = 0.0, syy = 0.0, sxy = 0.0;
    for (int p = 0; p < N; p++) {
      // source rows of output row p, both sides
      int ra0, ra1, rb0, rb1;
      double fa = 0.0, fb = 0.0;
      auto rows_of = [&](const FlatSide &S, int &r0, int &r1, double &f) {
        if (S.n == S.N) { r0 = p; r1 = -1; }
        else if (S.n == 1) { r0 = 0; r1 = -1; }
        else { flat_lofr(p, S.n, S.N, r0, f); r1 = r0 + 1; }
      };
      rows_of(SA, ra0, ra1, fa);
      rows_of(SB, rb0, rb1, fb);
      __syncthreads();  // previous row's buffers are free
      for (int k = tid; k < 4 * L; k += FLAT_THREADS) rows[k] = 0.0;
      __syncthreads();
      auto scatter = [&](const FlatSide &S, int r, double *dst) {
        if (r < 0) return;
        for (int e = S.rp[r] + tid; e < S.rp[r + 1]; e += FLAT_THREADS) dst[S.cc[e]] = S.rv[e];
      };
      scatter(SA, ra0, rows);
      scatter(SA, ra1, rows + L);
      scatter(SB, rb0, rows + 2 * L);
      scatter(SB, rb1, rows + 3 * L);
      __syncthreads();
      for (int q = tid; q < N; q += FLAT_THREADS) {
        const double x = flat_value(SA, rows, rows + L, fa, q);
        const double y = flat_value(SB, rows + 2 * L, rows + 3 * L, fb, q);
        const double d = x - y, ad = fabs(d);
        switch (work.measure) {
          case FLAT_ALL:  // (x-y)^2 == |x-y|^2 exactly, so EUC and JAC share s2
            s2 += ad * ad; s1 += ad; sp += pow(ad, work.p); sxx += x * x; syy += y * y; sxy += x * y;
            break;
          case FLAT_EUC: s2 += ad * ad; break;
          case FLAT_MAN: s1 += ad; break;
          case FLAT_MIN: sp += pow(ad, work.p); break;
          case FLAT_JAC: s2 += d * d; sxx += x * x; syy += y * y; sxy += x * y; break;
          default: sxx += x * x; syy += y * y; sxy += x * y; break;
        }
      }
    }
    double v[6] = {s2, s1, sp, sxx, syy, sxy};
#pragma unroll
    for (int k = 0; k < 6; k++) {
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], m);
      if (lane == 0) red[k][warp] = v[k];
    }
    __syncthreads();
    if (tid == 0) {
      double t[6];
      for (int k = 0; k < 6; k++) {
        t[k] = 0.0;
        for (int w = 0; w < FLAT_THREADS / 32; w++) t[k] += red[k][w];
      }
      auto value = [&](int m) {
        switch (m) {
          case FLAT_EUC: return sqrt(t[0]);
          case FLAT_MAN: return t[1];
          case FLAT_MIN: return work.p >= 1.0 ? pow(t[2], 1.0 / work.p) : CUDART_NAN;  // BadOrder
          case FLAT_JAC: {
            const double den = t[3] + t[4] - t[5];
            return den == 0.0 ? CUDART_NAN : t[0] / den;  // DegenerateInput
          }
          default: {
            const double nx = sqrt(t[3]), ny = sqrt(t[4]);
            return (nx == 0.0 || ny == 0.0) ? CUDART_NAN : 1.0 - t[5] / (nx * ny);  // DegenerateInput
          }
        }
      };
      if (work.measure == FLAT_ALL) {
        for (int m = 0; m < 5; m++) {
          const double r = value(m);
          out[m * work.out_stride + o1] = r;
          if (o2 >= 0) out[m * work.out_stride + o2] = r;
        }
      } else {
        const double r = value(work.measure);
        out[o1] = r;
        if (o2 >= 0) out[o2] = r;
      }
    }
    __syncthreads();
  }
}

}  // namespace cfgsim
