// Ward-linkage agglomerative clustering (cluster.py:88-134),
// exact: the same double arithmetic as the reference's merge loop, the same
// tie rule, O(K^2) work instead of O(K^3).
//
// Reference: initial d(i,j) = sum_f (x_if - x_jf)^2 (Python sum, left to
// right, cluster.py:109-113); each step takes min over (d, (id_a, id_b))
// (:117), merges into id next_id and updates by Lance-Williams
//   d(m, j) = ((n_j+n_k) d(k,j) + (n_j+n_l) d(l,j) - n_j d(k,l)) / (n_j+n_k+n_l)
// evaluated left to right (:126-129).
//
// The initial distances are formed on the host (libm pow and CPython's
// compensated sum(), to match bit for bit) and uploaded.
// Here: D is a full symmetric K x K matrix in HBM indexed by slots; the
// merged cluster m takes the slot of its smaller-id member.  Every active
// slot caches the minimum of its "row" — (d, partner id) over partners with a
// LARGER id, so each pair belongs to the row of its smaller id and the global
// lexicographic minimum is the minimum over rows of (d, own id, partner id).
// After a merge only rows whose cached partner was merged are rescanned; the
// others compare against the one new entry d(j, m) (m has the largest id, so
// a tie keeps the existing partner).  One persistent CTA; per step: a block
// argmin, the Lance-Williams column update, warp rescans of flagged rows.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cfgsim {

constexpr int WARD_THREADS = 1024;

struct WardState {
  int K;
  double *D;           // K x K (slots)
  int64_t *id;         // cluster id per slot
  int64_t *size;       // cluster size per slot
  double *rmin;        // cached row minimum per slot
  int32_t *rarg;       // its partner slot (-1: empty row)
  uint8_t *alive;
  int32_t *flag;       // scratch: rows to rescan
  int64_t *out_a, *out_b, *out_size;
  double *out_d;
};

__device__ __forceinline__ bool ward_less(double d1, int64_t a1, int64_t b1, double d2, int64_t a2, int64_t b2) {
  if (d1 != d2) return d1 < d2;
  if (a1 != a2) return a1 < a2;
  return b1 < b2;
}

// row minimum of slot j over alive partners with a larger id; one warp
__device__ void ward_rescan(WardState &S, int j, int lane) {
  const int K = S.K;
  const int64_t idj = S.id[j];
  double bd = INFINITY;
  int64_t bid = INT64_MAX;
  int bs = -1;
  for (int x = lane; x < K; x += 32) {
    if (!S.alive[x] || x == j || S.id[x] <= idj) continue;
    const double v = S.D[(int64_t)j * K + x];
    if (v < bd || (v == bd && S.id[x] < bid)) { bd = v; bid = S.id[x]; bs = x; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bd, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bid, o);
    const int os = __shfl_xor_sync(0xffffffffu, bs, o);
    if (ov < bd || (ov == bd && oi < bid)) { bd = ov; bid = oi; bs = os; }
  }
  if (lane == 0) {
    S.rmin[j] = bd;
    S.rarg[j] = bs;
  }
}

__global__ void __launch_bounds__(WARD_THREADS, 1) ward_kernel(WardState S) {
  __shared__ double sd[WARD_THREADS / 32];
  __shared__ int64_t sa[WARD_THREADS / 32], sb[WARD_THREADS / 32];
  __shared__ int ss[WARD_THREADS / 32];
  __shared__ int nflag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = WARD_THREADS / 32;
  const int K = S.K;
  for (int s = tid; s < K; s += WARD_THREADS) {
    S.id[s] = s;
    S.size[s] = 1;
    S.alive[s] = 1;
  }
  __syncthreads();
  for (int j = warp; j < K; j += NW) ward_rescan(S, j, lane);
  __syncthreads();
  for (int step = 0; step < K - 1; step++) {
    // ---- global minimum over rows of (d, id_row, id_partner)
    double bd = INFINITY;
    int64_t ba = INT64_MAX, bb = INT64_MAX;
    int bsl = -1;
    for (int s = tid; s < K; s += WARD_THREADS) {
      if (!S.alive[s] || S.rarg[s] < 0) continue;
      const double v = S.rmin[s];
      const int64_t ia = S.id[s], ib = S.id[S.rarg[s]];
      if (bsl < 0 || ward_less(v, ia, ib, bd, ba, bb)) { bd = v; ba = ia; bb = ib; bsl = s; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bd, o);
      const int64_t oa = __shfl_xor_sync(0xffffffffu, ba, o);
      const int64_t ob = __shfl_xor_sync(0xffffffffu, bb, o);
      const int os = __shfl_xor_sync(0xffffffffu, bsl, o);
      if (os >= 0 && (bsl < 0 || ward_less(ov, oa, ob, bd, ba, bb))) { bd = ov; ba = oa; bb = ob; bsl = os; }
    }
    if (lane == 0) { sd[warp] = bd; sa[warp] = ba; sb[warp] = bb; ss[warp] = bsl; }
    if (tid == 0) nflag = 0;
    __syncthreads();
    bd = sd[0]; ba = sa[0]; bb = sb[0]; bsl = ss[0];
    for (int w = 1; w < NW; w++)
      if (ss[w] >= 0 && (bsl < 0 || ward_less(sd[w], sa[w], sb[w], bd, ba, bb))) {
        bd = sd[w]; ba = sa[w]; bb = sb[w]; bsl = ss[w];
      }
    const int sk = bsl, sl = S.rarg[sk];  // slots of k (smaller id) and l
    const int64_t nk = S.size[sk], nl = S.size[sl];
    const double dkl = bd;
    const int64_t mid = (int64_t)K + step;
    __syncthreads();  // everyone has read the winner before slots change
    if (tid == 0) {
      S.out_a[step] = ba;
      S.out_b[step] = bb;
      S.out_d[step] = dkl;
      S.out_size[step] = nk + nl;
      S.alive[sl] = 0;
      S.id[sk] = mid;
      S.size[sk] = nk + nl;
      S.rmin[sk] = INFINITY;  // m has the largest id: its row is empty
      S.rarg[sk] = -1;
    }
    // ---- Lance-Williams column update (cluster.py:126-129, left to right)
    for (int j = tid; j < K; j += WARD_THREADS) {
      if (!S.alive[j] || j == sk || j == sl) continue;
      const double nj = (double)S.size[j];
      const double dkj = S.D[(int64_t)j * K + sk], dlj = S.D[(int64_t)j * K + sl];
      const double t1 = __dmul_rn(__dadd_rn(nj, (double)nk), dkj);
      const double t2 = __dmul_rn(__dadd_rn(nj, (double)nl), dlj);
      const double t3 = __dmul_rn(nj, dkl);
      const double v = __ddiv_rn(__dsub_rn(__dadd_rn(t1, t2), t3), __dadd_rn(__dadd_rn(nj, (double)nk), (double)nl));
      S.D[(int64_t)j * K + sk] = v;
      S.D[(int64_t)sk * K + j] = v;
      const int ra = S.rarg[j];
      if (ra == sk || ra == sl) {
        S.flag[atomicAdd(&nflag, 1)] = j;  // cached partner merged: rescan
      } else if (v < S.rmin[j]) {          // equal: the existing partner has the smaller id
        S.rmin[j] = v;
        S.rarg[j] = sk;
      }
    }
    __syncthreads();
    for (int f = warp; f < nflag; f += NW) ward_rescan(S, S.flag[f], lane);
    __syncthreads();
  }
}

}  // namespace cfgsim
