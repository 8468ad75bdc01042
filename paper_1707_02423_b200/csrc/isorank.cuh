// IsoRank pair kernel for sm_100a — one CTA per CFG pair, state on-chip.
//
// Computes, per pair (a, b), exactly the reference's ISO measure
//   measure_distance(a, b, ISO)       similarity.py:176-189
//   = isorank_distance(isorank_align(normalize_pair(a, b)))
// with the Kronecker mat-vec kron(A',B')^T x (similarity.py:133,140)
// evaluated as the two sparse products  Y = A'^T X,  Z = Y B'.
//
// Layout (shared memory, per CTA):
//   Xs  (N+1) x P   X state (unnormalised F of the last sweep, scale r_old)
//                   + padding column N (g = X z_B) and row N (unused)
//   Ys  (N+1) x P   Y = A'^T X (+ column N: v = Y z_B)
//   lists A, B      column-tile lists of the row-normalised operators:
//                   tile t covers R consecutive columns; entry = (row i,
//                   R weights).  Uniform (zero-sum) rows are excluded and
//                   applied as rank-1 terms (u = z_A^T X, v = Y z_B).
//   P = (N+1)|1 (odd) so that column accesses with lanes over rows are
//   bank-conflict free for 8-byte elements.
// Each sweep (3 CTA barriers):
//   U: u[j] = sum_{i in zA} X[i,j];  X[i,N] = sum_{j in zB} X[i,j]
//   A: lanes over columns j (0..N), warps over row tiles of Y:
//        Y[k,j] = sum_e w_e[k] X[i_e,j] + u[j]/N       (column N gives v)
//   B: lanes over rows k, warps over column tiles of Z:
//        F[k,l] = (alpha*r_old) (sum_e w_e[l] Y[k,j_e] + v[k]/N) + (1-alpha)/N^2
//      reduce s = sum F, dp = sum |F - X_old|, m = sum sign(F - X_old) F
//   delta = sum |F/s - X_old| = dp + (1/s - 1) m   (exact to first order in
//   |1-s| ~ 1e-16), stop when delta < tol
//   (similarity.py:141-146).  X_old is re-read from Xs before F overwrites it.
// Epilogue: greedy matching with cached row maxima (same tie rule as
// similarity.py:96-108), W, d (similarity.py:150,160-173).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cfgsim {

struct DevCorpus {
  int32_t n_graphs;
  const int32_t *n_nodes;
  const int64_t *rp_off;
  const int32_t *rowptr;
  const int64_t *nz_off;
  const int32_t *col;
  const double *val;
  // transposed copy (CSC): graph g's column pointer is cscp[rp_off[g] ..],
  // its rows / values csc_row/csc_val[nz_off[g] + e], rows ascending
  const int32_t *cscp;
  const int32_t *csc_row;
  const double *csc_val;
};

enum { WORK_LIST = 0, WORK_TRIANGLE = 1, WORK_RECT = 2 };

struct PairWork {
  int32_t mode;
  int32_t ordered;   // triangle: compute both directions separately
  int64_t n_items;   // items in this launch
  // list mode
  const int32_t *ia;
  const int32_t *ib;
  const int64_t *slot;  // output slot per item (NULL: slot = item)
  // triangle mode: unit u = u0 + item; rows of the size-sorted corpus
  int64_t u0;
  int64_t out_base;          // unit that maps to output slot 0
  const int64_t *row_start;  // K+1
  const int32_t *perm;       // sorted position -> graph index
  int32_t K;
  // rect mode (query x corpus): item -> rectangle r (rect_start prefix),
  // rect[4r..4r+3] = q0, q1, c0, c1 in size-sorted positions of the two
  // corpora; output slot = (qperm[q] - qbase) * ld + (cperm[c] - cbase)
  int32_t nrect;
  const int64_t *rect_start;
  const int32_t *rect;
  const int32_t *qperm;
  const int32_t *cperm;
  int32_t qbase, cbase;
  int64_t ld;
};

// Work item -> (ga, gb, number of directions, first output slot).  Triangle
// mode computes one alignment per unordered pair in the caller's (lower
// index, higher index) direction — the reference's upper triangle — so
// results do not depend on the size-sorted schedule; `ordered` computes both.
__device__ __forceinline__ void decode_item(const PairWork &work, int64_t item, int &ga, int &gb, int &ndir,
                                            int64_t &slot0) {
  ndir = 1;
  if (work.mode == WORK_LIST) {
    ga = work.ia[item];
    gb = work.ib[item];
    slot0 = work.slot ? work.slot[item] : item;
    return;
  }
  if (work.mode == WORK_RECT) {
    int lo = 0, hi = work.nrect - 1;  // last r with rect_start[r] <= item
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (work.rect_start[mid] <= item) lo = mid; else hi = mid - 1;
    }
    const int32_t *R = work.rect + 4 * lo;
    const int64_t loc = item - work.rect_start[lo];
    const int w = R[3] - R[2];
    const int q = R[0] + (int)(loc / w), c = R[2] + (int)(loc % w);
    ga = work.qperm[q];
    gb = work.cperm[c];
    slot0 = (int64_t)(ga - work.qbase) * work.ld + (gb - work.cbase);
    return;
  }
  const int64_t u = work.u0 + item;
  int lo = 0, hi = work.K - 1;  // largest a with row_start[a] <= u
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (work.row_start[mid] <= u) lo = mid; else hi = mid - 1;
  }
  const int a = lo;
  const int b = a + (int)(u - work.row_start[a]);
  ga = work.perm[a];
  gb = work.perm[b];
  if (work.ordered) {
    slot0 = 2 * (u - work.out_base);
    ndir = (a == b) ? 1 : 2;
  } else {
    if (ga > gb) { const int t = ga; ga = gb; gb = t; }
    slot0 = u - work.out_base;
  }
}

struct PairOut {
  double *d;
  double *W;
  int32_t *iters;
  uint8_t *conv;
  double *X;          // single-pair: N*N normalised alignment matrix
  int32_t *match;     // single-pair: N
  const double *x0;   // single-pair: start / sum(start)
  int32_t *ovf_count; // overflowed (item, dir) records
  int64_t *ovf_list;
  int32_t ovf_cap;
};

struct PairParams {
  double alpha;
  double tol;
  int32_t max_iter;
  int32_t cap;      // list entries per side
  int32_t nlim;     // max N this launch is sized for
  int32_t force_m;  // accumulate the delta correction term every sweep
};

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double shfl_xor_d(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// numpy DOUBLE_pairwise_sum order (umath/loops_utils.h.src), stride 1 —
// the order of `out.sum(axis=1)` in similarity.py:89.  One thread.
__device__ inline double np_pairwise_leaf(const double *a, int n) {  // n <= 128
  if (n < 8) {
    double res = 0.;
    for (int i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; k++) r[k] = a[k];
  int i;
  for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int k = 0; k < 8; k++) r[k] = __dadd_rn(r[k], a[i + k]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; i++) res = __dadd_rn(res, a[i]);
  return res;
}

// The recursion `pw(a, n2) + pw(a + n2, n - n2)` (n2 = n/2 rounded down to a
// multiple of 8) unrolled with an explicit stack.
__device__ inline double np_pairwise_sum(const double *a, int n) {
  if (n <= 128) return np_pairwise_leaf(a, n);
  int off[24], len[24], state[24];
  double left[24];
  int sp = 0;
  off[0] = 0; len[0] = n; state[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    if (len[sp] <= 128) {
      ret = np_pairwise_leaf(a + off[sp], len[sp]);
      sp--;
      continue;
    }
    int n2 = len[sp] / 2;
    n2 -= n2 % 8;
    if (state[sp] == 0) {
      state[sp] = 1;
      off[sp + 1] = off[sp]; len[sp + 1] = n2; state[sp + 1] = 0;
      sp++;
    } else if (state[sp] == 1) {
      left[sp] = ret;
      state[sp] = 2;
      off[sp + 1] = off[sp] + n2; len[sp + 1] = len[sp] - n2; state[sp + 1] = 0;
      sp++;
    } else {
      ret = __dadd_rn(left[sp], ret);
      sp--;
    }
  }
  return ret;
}

// np_pairwise_sum computed by a warp, bit-identical: for 8 <= n <= 128 the
// eight strided partial sums r[k] = a[k] + a[k+8] + ... run on lanes 0..7 in
// numpy's order, then lane 0 combines them with numpy's fixed tree and adds
// the tail; other n use the serial routine on lane 0.  Result on all lanes.
__device__ inline double warp_pairwise_sum(const double *a, int n, int lane) {
  double res = 0.0;
  if (n >= 8 && n <= 128) {
    const int full = n - (n % 8);
    double r = 0.0;
    if (lane < 8) {
      r = a[lane];
      for (int i = 8 + lane; i < full; i += 8) r = __dadd_rn(r, a[i]);
    }
    const double r1 = __shfl_down_sync(0xffffffffu, r, 1);
    const double p01 = __dadd_rn(r, r1);          // lanes 0,2,4,6: r[k] + r[k+1]
    const double p23 = __shfl_down_sync(0xffffffffu, p01, 2);
    const double q = __dadd_rn(p01, p23);         // lanes 0,4: (r0+r1)+(r2+r3), (r4+r5)+(r6+r7)
    const double q4 = __shfl_down_sync(0xffffffffu, q, 4);
    if (lane == 0) {
      res = __dadd_rn(q, q4);
      for (int i = full; i < n; i++) res = __dadd_rn(res, a[i]);
    }
  } else if (lane == 0) {
    res = np_pairwise_sum(a, n);
  }
  return __shfl_sync(0xffffffffu, res, 0);
}

// R consecutive weights as one or two 16-byte shared loads (broadcast).
template <typename T, int R>
__device__ __forceinline__ void load_w(const T *p, T (&w)[R]) {
  if constexpr (sizeof(T) == 8 && R % 2 == 0) {
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      const double2 v = *reinterpret_cast<const double2 *>(p + r);
      w[r] = v.x;
      w[r + 1] = v.y;
    }
  } else if constexpr (sizeof(T) == 4 && R % 4 == 0) {
#pragma unroll
    for (int r = 0; r < R; r += 4) {
      const float4 v = *reinterpret_cast<const float4 *>(p + r);
      w[r] = v.x; w[r + 1] = v.y; w[r + 2] = v.z; w[r + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; r++) w[r] = p[r];
  }
}

// warp argmax with key (value desc, index asc) — the first-occurrence rule of
// np.argmax over a row-major scan.
template <typename T>
__device__ __forceinline__ void warp_argmax(T &v, int &idx) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    T ov = __shfl_xor_sync(0xffffffffu, v, m);
    int oi = __shfl_xor_sync(0xffffffffu, idx, m);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
}

// Total order of the reference's greedy matching inside one row:
// larger value first, then lower column (np.argmax first occurrence).
template <typename T>
__device__ __forceinline__ bool before(T v1, int c1, T v2, int c2) {
  return v1 > v2 || (v1 == v2 && c1 < c2);
}

// Warp-wide bitonic sort of 32*KB (value, column) pairs into `before` order;
// element e = cc*32 + lane lives in v[cc], c[cc].
template <typename T, int KB>
__device__ __forceinline__ void warp_sort_desc(T (&v)[KB], int (&c)[KB], int lane) {
  constexpr int n = 32 * KB;
#pragma unroll
  for (int k = 2; k <= n; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int cc = 0; cc < KB; cc++) {
          const int pc = cc ^ (j >> 5);
          if (pc > cc) {
            const bool up = ((cc * 32 + lane) & k) == 0;
            const bool sw = up ? before(v[pc], c[pc], v[cc], c[cc]) : before(v[cc], c[cc], v[pc], c[pc]);
            if (sw) {
              const T tv = v[cc]; v[cc] = v[pc]; v[pc] = tv;
              const int tc = c[cc]; c[cc] = c[pc]; c[pc] = tc;
            }
          }
        }
      } else {
#pragma unroll
        for (int cc = 0; cc < KB; cc++) {
          const T ov = __shfl_xor_sync(0xffffffffu, v[cc], j);
          const int oc = __shfl_xor_sync(0xffffffffu, c[cc], j);
          const bool lower = (lane & j) == 0;
          const bool up = ((cc * 32 + lane) & k) == 0;
          const bool take = (lower == up) ? before(ov, oc, v[cc], c[cc]) : before(v[cc], c[cc], ov, oc);
          if (take) { v[cc] = ov; c[cc] = oc; }
        }
      }
    }
  }
}

// Warp-wide bitonic sort of 32*KB distinct unsigned keys, descending.
template <int KB>
__device__ __forceinline__ void warp_sort_keys_desc(unsigned long long (&v)[KB], int lane) {
  constexpr int n = 32 * KB;
#pragma unroll
  for (int k = 2; k <= n; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int cc = 0; cc < KB; cc++) {
          const int pc = cc ^ (j >> 5);
          if (pc > cc) {
            const bool up = ((cc * 32 + lane) & k) == 0;
            const bool sw = up ? (v[pc] > v[cc]) : (v[cc] > v[pc]);
            if (sw) { const unsigned long long t = v[cc]; v[cc] = v[pc]; v[pc] = t; }
          }
        }
      } else {
#pragma unroll
        for (int cc = 0; cc < KB; cc++) {
          const unsigned long long ov = __shfl_xor_sync(0xffffffffu, v[cc], j);
          const bool lower = (lane & j) == 0;
          const bool up = ((cc * 32 + lane) & k) == 0;
          const unsigned long long hi = ov > v[cc] ? ov : v[cc], lo = ov > v[cc] ? v[cc] : ov;
          v[cc] = (lower == up) ? hi : lo;
        }
      }
    }
  }
}

// Phase A inner loop over one tile's entries: acc[c][r] += w_e[r] * X[i_e, lane+32c];
// EXTRA also accumulates column xcol (= N when N == 32*KB) uniformly.
template <typename T, int KB, int R, bool EXTRA>
__device__ __forceinline__ void tile_accumulate_rows(const int32_t *__restrict__ idx, const T *__restrict__ wts,
                                                     const T *__restrict__ Xs, int e0, int e1, int lane, int xcol,
                                                     T (&acc)[KB][R], T (&accx)[R]) {
#pragma unroll 2
  for (int e = e0; e < e1; e++) {
    const int ioff = idx[e];
    T w[R];
    load_w<T, R>(wts + e * R, w);
#pragma unroll
    for (int c = 0; c < KB; c++) {
      const T x = Xs[ioff + lane + 32 * c];
#pragma unroll
      for (int r = 0; r < R; r++) acc[c][r] = fma(w[r], x, acc[c][r]);
    }
    if (EXTRA) {
      const T x = Xs[ioff + xcol];
#pragma unroll
      for (int r = 0; r < R; r++) accx[r] = fma(w[r], x, accx[r]);
    }
  }
}

// Shared-memory carve-up, identical on host and device.
struct Smem {
  size_t x, y, idxA, wA, idxB, wB, toffA, toffB, ordA, ordB, zA, zB, uS, lo, fr, zflag, red, misc, total;
};

template <typename T, int R>
__host__ __device__ inline Smem smem_layout(int nlim, int cap) {
  Smem s;
  const int pm = (nlim + 1) | 1;
  const int ktm = (nlim + R - 1) / R;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += (bytes + 15) & ~size_t(15);
    return at;
  };
  const size_t xbytes = sizeof(T) * ((size_t)(nlim + 1) * pm + 64);
  s.x = take(xbytes);
  s.y = take(xbytes);
  s.idxA = take(sizeof(int32_t) * (size_t)cap);
  s.wA = take(sizeof(T) * (size_t)cap * R);
  s.idxB = take(sizeof(int32_t) * (size_t)cap);
  s.wB = take(sizeof(T) * (size_t)cap * R);
  s.toffA = take(sizeof(int32_t) * (ktm + 1));
  s.toffB = take(sizeof(int32_t) * (ktm + 1));
  s.ordA = take(sizeof(int32_t) * (ktm + 1));
  s.ordB = take(sizeof(int32_t) * (ktm + 1));
  s.zA = take(sizeof(int32_t) * (nlim + 1));
  s.zB = take(sizeof(int32_t) * (nlim + 1));
  s.uS = take(sizeof(T) * (nlim + 64));
  s.lo = take(sizeof(int32_t) * (nlim + 1));
  s.fr = take(sizeof(double) * (nlim + 1));
  s.zflag = take(sizeof(uint8_t) * (nlim + 1));
  s.red = take(sizeof(double) * 3 * 32);
  s.misc = take(64);
  s.total = o;
  return s;
}

// Build the row-normalised operator of one side (similarity.py:85-93 after
// matrix.py:74-106) into the dense fp64 scratch `dense` (N x N, pitch N),
// then extract its column-tile lists.  Returns false on list overflow.
// `dense` needs N * (N|1) doubles (shared or global memory).
template <typename T, int KB, int R, bool SORT_TILES>
__device__ bool build_side(const DevCorpus &G, int g, int N, int P, double *dense, int32_t *lo_s,
                           double *fr_s, uint8_t *zflag, int32_t *zlist, int32_t *nz_out,
                           int32_t *toff, int32_t *ord, int32_t *idx, T *wts, int cap,
                           bool premul_rows, int32_t *misc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  const int n = G.n_nodes[g];
  const int32_t *rp = G.rowptr + G.rp_off[g];
  const int32_t *cc = G.col + G.nz_off[g];
  const double *vv = G.val + G.nz_off[g];
  const bool interp = (n != N) && (n > 1);

  if (interp) {  // matrix.py:93-95
    for (int p = tid; p < N; p += NT) {
      double pos = __ddiv_rn((double)((long long)p * (n - 1)), (double)(N - 1));
      int l = (int)floor(pos);
      if (l > n - 2) l = n - 2;
      lo_s[p] = l;
      fr_s[p] = __dsub_rn(pos, (double)l);
    }
    __syncthreads();
  }

  // Rows of A-hat, one warp per target row (scratch pitch DP = N|1: odd, so
  // the column scans below are bank-conflict free).
  const int DP = N | 1;
  for (int p = warp; p < N; p += NW) {
    double *row = dense + (size_t)p * DP;
    if (n == N) {
      for (int q = lane; q < N; q += 32) row[q] = 0.0;
      __syncwarp();
      for (int e = rp[p] + lane; e < rp[p + 1]; e += 32) row[cc[e]] = vv[e];
    } else if (n == 1) {  // matrix.py:87-89
      const double c = (rp[1] > rp[0]) ? vv[0] : 0.0;
      for (int q = lane; q < N; q += 32) row[q] = c;
    } else {  // matrix.py:97-104, same operation order, no contraction
      const int r0 = lo_s[p];
      const double frp = fr_s[p];
      const int b0 = rp[r0], e0 = rp[r0 + 1], e1 = rp[r0 + 2];
      for (int q = lane; q < N; q += 32) {
        const int c = lo_s[q];
        const double fc = fr_s[q];
        double v00 = 0, v01 = 0, v10 = 0, v11 = 0;
        for (int e = b0; e < e0; e++) {
          const int k = cc[e];
          if (k == c) v00 = vv[e];
          if (k == c + 1) v01 = vv[e];
        }
        for (int e = e0; e < e1; e++) {
          const int k = cc[e];
          if (k == c) v10 = vv[e];
          if (k == c + 1) v11 = vv[e];
        }
        const double omc = __dsub_rn(1.0, fc);
        const double top = __dadd_rn(__dmul_rn(omc, v00), __dmul_rn(fc, v01));
        const double bot = __dadd_rn(__dmul_rn(omc, v10), __dmul_rn(fc, v11));
        row[q] = __dadd_rn(__dmul_rn(__dsub_rn(1.0, frp), top), __dmul_rn(frp, bot));
      }
    }
    __syncwarp();
    const double s = warp_pairwise_sum(row, N, lane);  // similarity.py:89
    if (lane == 0) zflag[p] = (s == 0.0);
    if (s != 0.0)
      for (int q = lane; q < N; q += 32)
        if (row[q] != 0.0) row[q] = __ddiv_rn(row[q], s);  // :92 (0/s == 0)
  }
  __syncthreads();

  // zero-row list (ascending) and column-tile entry counts
  const int KT = (N + R - 1) / R;
  if (warp == 0) {
    int cnt = 0;
#pragma unroll
    for (int c = 0; c < KB; c++) {
      const int i = lane + 32 * c;
      const bool z = (i < N) && zflag[i];
      const unsigned bal = __ballot_sync(0xffffffffu, z);
      if (z) zlist[cnt + __popc(bal & ((1u << lane) - 1))] = i;
      cnt += __popc(bal);
    }
    if (lane == 0) *nz_out = cnt;
  }
  for (int t = warp; t < KT; t += NW) {
    int cnt = 0;
#pragma unroll
    for (int c = 0; c < KB; c++) {
      const int i = lane + 32 * c;
      bool nzr = false;
      if (i < N && !zflag[i]) {
#pragma unroll
        for (int r = 0; r < R; r++) {
          const int k = t * R + r;
          if (k < N && dense[(size_t)i * DP + k] != 0.0) nzr = true;
        }
      }
      cnt += __popc(__ballot_sync(0xffffffffu, nzr));
    }
    if (lane == 0) toff[t + 1] = cnt;
  }
  __syncthreads();
  if (warp == 0) {  // inclusive scan of tile counts (KT <= 32 * KB / R * ... small)
    int carry = 0;
    for (int base = 0; base < KT; base += 32) {
      const int t = base + lane;
      int v = (t < KT) ? toff[t + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (t < KT) toff[t + 1] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) {
      toff[0] = 0;
      misc[0] = (carry > cap) ? 1 : 0;
    }
  }
  __syncthreads();
  if (misc[0]) return false;
  for (int t = warp; t < KT; t += NW) {
    int pos = toff[t];
#pragma unroll
    for (int c = 0; c < KB; c++) {
      const int i = lane + 32 * c;
      bool nzr = false;
      double w[R];
#pragma unroll
      for (int r = 0; r < R; r++) {
        const int k = t * R + r;
        w[r] = (i < N && k < N) ? dense[(size_t)i * DP + k] : 0.0;
        if (w[r] != 0.0) nzr = true;
      }
      if (i >= N || zflag[i]) nzr = false;
      const unsigned bal = __ballot_sync(0xffffffffu, nzr);
      if (nzr) {
        const int e = pos + __popc(bal & ((1u << lane) - 1));
        idx[e] = premul_rows ? i * P : i;
#pragma unroll
        for (int r = 0; r < R; r++) wts[(size_t)e * R + r] = (T)w[r];
      }
      pos += __popc(bal);
    }
  }
  // Tile schedule: tiles sorted by cost (entries) descending; phases hand
  // them to warps in boustrophedon order (longest first), which balances the
  // per-sweep work across warps for all ~70+ sweeps of this pair.
  if (SORT_TILES && warp == 0) {
    constexpr int SK = (32 * KB + R - 1) / R <= 32 ? 1 : ((32 * KB + R - 1) / R <= 64 ? 2 : 4);
    int cv[SK], ci[SK];
#pragma unroll
    for (int c = 0; c < SK; c++) {
      const int t = lane + 32 * c;
      ci[c] = t;
      cv[c] = (t < KT) ? (toff[t + 1] - toff[t] + 2) : -1;
    }
    warp_sort_desc<int, SK>(cv, ci, lane);
#pragma unroll
    for (int c = 0; c < SK; c++) {
      const int q = lane + 32 * c;
      if (q < KT) ord[q] = ci[c];
    }
  }
  __syncthreads();
  return true;
}

// q-th tile (0, 1, ...) of `warp` in the boustrophedon schedule; -1 when done.
template <int NW>
__device__ __forceinline__ int snake_slot(int m, int warp) {
  return m * NW + ((m & 1) ? (NW - 1 - warp) : warp);
}

// d from the matched weight, similarity.py:160-173
__device__ __forceinline__ double isorank_distance_of(double w, int N) {
  if (N == 1) return 1.0;
  double cn = (w - 1.0 / N) / (1.0 - 1.0 / N);
  cn = fmin(1.0, fmax(0.0, cn));
  return 1.0 + (1.0 - cn);
}

// Greedy matching, similarity.py:96-108, on X (N x N, pitch P, in shared
// memory).  Each row's columns are sorted once into the reference's order
// (value desc, column asc); a round then takes the best current head over
// active rows (ties -> lowest row, i.e. lowest row-major index overall) and
// advances only the rows whose head column was just taken — the same
// matching as repeated global argmax.  `scr` needs N*N + 4N + 32 bytes.
// Call with the whole CTA; returns W = sum_i X[i, match(i)] (similarity.py:150)
// to every thread.
template <typename T, int KB>
__device__ double greedy_match(const T *Xs, int P, int N, uint8_t *scr, int lane, int warp, int NW,
                               int32_t *match_out) {
  uint8_t *ord = scr;  // N x N column order (N <= 255)
  int32_t *mS = (int32_t *)(scr + (((size_t)N * N + 15) & ~(size_t)15));
  double *wres = (double *)(mS + ((N + 3) & ~3));
  // column bits and the exponent span a packed key can hold
  constexpr int CB = (32 * KB <= 64) ? 6 : ((32 * KB <= 128) ? 7 : 8);
  constexpr int EB = (sizeof(T) == 8) ? 12 - CB : 8;  // exponent bits left in 64
  for (int i = warp; i < N; i += NW) {
    T v[KB];
#pragma unroll
    for (int cc = 0; cc < KB; cc++) {
      const int j = lane + 32 * cc;
      v[cc] = (j < N) ? Xs[i * P + j] : (T)0;
    }
    // X > 0 (teleport floor): if the row's exponent span fits in EB bits,
    // (value desc, column asc) is one unsigned key: rebased exponent |
    // mantissa | (mask - column), sorted as integers (exact, no fp compare).
    int emin = 0x7fffffff, emax = -1;
#pragma unroll
    for (int cc = 0; cc < KB; cc++)
      if (lane + 32 * cc < N) {
        const int e = (sizeof(T) == 8) ? (int)((__double_as_longlong((double)v[cc]) >> 52) & 0x7ff)
                                       : (int)((__float_as_uint((float)v[cc]) >> 23) & 0xff);
        emin = min(emin, e);
        emax = max(emax, e);
      }
    emin = __reduce_min_sync(0xffffffffu, emin);
    emax = __reduce_max_sync(0xffffffffu, emax);
    if (emin > 0 && emax - emin < (1 << EB)) {
      unsigned long long key[KB];  // padding lanes (j >= N) keep 0 and sort last:
                                   // real keys have a column field >= 1 then
#pragma unroll
      for (int cc = 0; cc < KB; cc++) {
        const int j = lane + 32 * cc;
        unsigned long long k = 0ull;  // padding sorts last
        if (j < N) {
          if (sizeof(T) == 8) {
            const unsigned long long b = (unsigned long long)__double_as_longlong((double)v[cc]);
            const unsigned long long e = ((b >> 52) & 0x7ff) - (unsigned long long)emin;
            const unsigned long long m = b & ((1ull << 52) - 1);
            k = (e << (52 + CB)) | (m << CB) | (unsigned long long)((1 << CB) - 1 - j);
          } else {
            const unsigned int b = __float_as_uint((float)v[cc]);
            const unsigned long long e = ((b >> 23) & 0xff) - (unsigned)emin;
            k = (e << (23 + CB)) | ((unsigned long long)(b & 0x7fffff) << CB) |
                (unsigned long long)((1 << CB) - 1 - j);
          }
        }
        key[cc] = k;
      }
      warp_sort_keys_desc<KB>(key, lane);
#pragma unroll
      for (int cc = 0; cc < KB; cc++) {
        const int pos = lane + 32 * cc;
        if (pos < N) ord[i * N + pos] = (uint8_t)((1 << CB) - 1 - (int)(key[cc] & ((1ull << CB) - 1)));
      }
    } else {
      int c[KB];
#pragma unroll
      for (int cc = 0; cc < KB; cc++) {
        const int j = lane + 32 * cc;
        c[cc] = j;
        if (j >= N) v[cc] = (T)-1;
      }
      warp_sort_desc<T, KB>(v, c, lane);
#pragma unroll
      for (int cc = 0; cc < KB; cc++) {
        const int pos = lane + 32 * cc;
        if (pos < N) ord[i * N + pos] = (uint8_t)c[cc];
      }
    }
  }
  __syncthreads();
  if (warp == 0) {
    int ptr[KB], ccol[KB];
    T cur[KB];
    bool act[KB];
    uint32_t taken[KB];
#pragma unroll
    for (int cc = 0; cc < KB; cc++) {
      const int i = lane + 32 * cc;
      act[cc] = i < N;
      ptr[cc] = 0;
      taken[cc] = 0u;
      ccol[cc] = act[cc] ? (int)ord[i * N] : 0;
      cur[cc] = act[cc] ? Xs[i * P + ccol[cc]] : (T)-3;
    }
    for (int round = 0; round < N; round++) {
      T bv = (T)0;
      int brow = 0x7fffffff;
#pragma unroll
      for (int cc = 0; cc < KB; cc++)
        if (act[cc] && (brow == 0x7fffffff || cur[cc] > bv)) { bv = cur[cc]; brow = lane + 32 * cc; }
      // warp argmax (value desc, row asc) with integer reductions: X > 0, so
      // the IEEE bit pattern orders like the value
      if (sizeof(T) == 8) {
        const unsigned long long b = (brow == 0x7fffffff) ? 0ull : (unsigned long long)__double_as_longlong((double)bv);
        const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        brow = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)brow : 0x7fffffffu);
      } else {
        const unsigned b = (brow == 0x7fffffff) ? 0u : __float_as_uint((float)bv);
        const unsigned mb = __reduce_max_sync(0xffffffffu, b);
        brow = (int)__reduce_min_sync(0xffffffffu, b == mb ? (unsigned)brow : 0x7fffffffu);
      }
      int mycol = 0;
#pragma unroll
      for (int cc = 0; cc < KB; cc++)
        if (cc == (brow >> 5)) mycol = ccol[cc];
      const int bcol = __shfl_sync(0xffffffffu, mycol, brow & 31);
      if (lane == 0) mS[brow] = bcol;
#pragma unroll
      for (int cc = 0; cc < KB; cc++) {
        if (lane + 32 * cc == brow) act[cc] = false;
        if (cc == (bcol >> 5)) taken[cc] |= 1u << (bcol & 31);
      }
#pragma unroll
      for (int cc = 0; cc < KB; cc++) {
        if (act[cc] && ccol[cc] == bcol) {
          const int i = lane + 32 * cc;
          int p = ptr[cc], col;
          bool tk;
          do {
            ++p;
            col = ord[i * N + p];
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < KB; q++)
              if (q == (col >> 5)) word = taken[q];
            tk = (word >> (col & 31)) & 1u;
          } while (tk);
          ptr[cc] = p;
          ccol[cc] = col;
          cur[cc] = Xs[i * P + col];
        }
      }
    }
    __syncwarp();
    __syncwarp();
    if (lane == 0) {  // similarity.py:150: Python's sum, row order
      double wsum = 0.0;
      for (int i = 0; i < N; i++) wsum += (double)Xs[i * P + mS[i]];
      *wres = wsum;
    }
    if (match_out)
      for (int i = lane; i < N; i += 32) match_out[i] = mS[i];
  }
  __syncthreads();
  return *wres;
}

// Phase A of one sweep for this warp: Y[k, j] = u[j]/N + sum_e w_e[k] X[i_e, j]
// over its tiles (output rows k = t*R .. t*R+R-1), lanes over columns j.
template <typename T, int KB, int NW, int R>
__device__ __forceinline__ void phase_a(const T *__restrict__ Xs, T *__restrict__ Ys, const int32_t *__restrict__ idxA,
                                        const T *__restrict__ wA, const int32_t *__restrict__ toffA,
                                        const int32_t *__restrict__ ordA, const int32_t *__restrict__ zA, int nzA,
                                        int N, int P, int KT, T invN, int lane, int warp) {
  T ucol[KB];  // u[j] / N, computed by every warp from the uniform rows of A'
#pragma unroll
  for (int c = 0; c < KB; c++) ucol[c] = 0;
  for (int e = 0; e < nzA; e++) {
    const int zo = zA[e] * P + lane;
#pragma unroll
    for (int c = 0; c < KB; c++) ucol[c] += Xs[zo + 32 * c];
  }
#pragma unroll
  for (int c = 0; c < KB; c++) ucol[c] *= invN;
  for (int m = 0;; m++) {
    const int q = snake_slot<NW>(m, warp);
    if (q >= KT) break;
    const int t = ordA[q];
    T acc[KB][R], accx[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      accx[r] = 0;
#pragma unroll
      for (int c = 0; c < KB; c++) acc[c][r] = ucol[c];
    }
    tile_accumulate_rows<T, KB, R, false>(idxA, wA, Xs, toffA[t], toffA[t + 1], lane, N, acc, accx);
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int k = t * R + r;
      T *yrow = Ys + k * P;
#pragma unroll
      for (int c = 0; c < KB; c++) {
        const int j = lane + 32 * c;
        if (k < N && j < N) yrow[j] = acc[c][r];
      }
    }
  }
}

// Phase B of one sweep for this warp: F[k, l] = alpha' (v[k]/N + sum_e w_e[l]
// Y[k, j_e]) + teleport over its tiles (columns l), lanes over rows k.  X_old
// is re-read from Xs just before F overwrites it.  Branch-free: padded lanes
// and columns run on finite data and are masked out of the sums.
template <typename T, int KB, int NW, int R, bool NEEDM>
__device__ __forceinline__ void phase_b(T *__restrict__ Xs, const T *__restrict__ Ys, const int32_t *__restrict__ idxB,
                                        const T *__restrict__ wB, const int32_t *__restrict__ toffB,
                                        const int32_t *__restrict__ ordB, const int32_t *__restrict__ zB, int nzB,
                                        int N, int P, int KT, T invN, T alpha_eff, T rold, T teleport, int lane,
                                        int warp, T &sl, T &dl, T &ml) {
  T vrow[KB], mk[KB];
  int krow[KB];
#pragma unroll
  for (int c = 0; c < KB; c++) {
    const int k = lane + 32 * c;
    krow[c] = (k < N ? k : N - 1) * P;
    mk[c] = (k < N) ? (T)1 : (T)0;
    vrow[c] = 0;
  }
  for (int e = 0; e < nzB; e++) {
    const int zj = zB[e];
#pragma unroll
    for (int c = 0; c < KB; c++) vrow[c] += Ys[krow[c] + zj];
  }
#pragma unroll
  for (int c = 0; c < KB; c++) vrow[c] *= invN;
  for (int m = 0;; m++) {
    const int q = snake_slot<NW>(m, warp);
    if (q >= KT) break;
    const int t = ordB[q];
    T acc[KB][R];
#pragma unroll
    for (int c = 0; c < KB; c++)
#pragma unroll
      for (int r = 0; r < R; r++) acc[c][r] = vrow[c];
    const int e1 = toffB[t + 1];
#pragma unroll 2
    for (int e = toffB[t]; e < e1; e++) {
      const int j = idxB[e];
      T w[R];
      load_w<T, R>(wB + e * R, w);
#pragma unroll
      for (int c = 0; c < KB; c++) {
        const T y = Ys[krow[c] + j];
#pragma unroll
        for (int r = 0; r < R; r++) acc[c][r] = fma(w[r], y, acc[c][r]);
      }
    }
    const int lv = N - t * R;  // valid columns in this tile (>= 1)
#pragma unroll
    for (int c = 0; c < KB; c++) {
      const int k = lane + 32 * c;
      T *xrow = Xs + krow[c] + t * R;
#pragma unroll
      for (int r = 0; r < R; r++) {
        const T msk = (r < lv) ? mk[c] : (T)0;
        const T f = fma(alpha_eff, acc[c][r], teleport);
        const T diff = fma(-xrow[r], rold, f);
        sl = fma(msk, f, sl);
        dl = fma(msk, fabs(diff), dl);
        if (NEEDM) ml = fma(msk, copysign(f, diff), ml);
        if (k < N && r < lv) xrow[r] = f;
      }
    }
  }
}

template <typename T, int KB, int NW, int R, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
    isorank_pair_kernel(DevCorpus CA, DevCorpus CB, PairWork work, PairOut out, PairParams prm,
                        unsigned long long *counter) {
  constexpr int NT = NW * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Smem L = smem_layout<T, R>(prm.nlim, prm.cap);
  T *Xs = (T *)(smem_raw + L.x);
  T *Ys = (T *)(smem_raw + L.y);
  double *dense = (double *)(smem_raw + L.x);  // prologue scratch (spans Xs, Ys)
  int32_t *idxA = (int32_t *)(smem_raw + L.idxA);
  T *wA = (T *)(smem_raw + L.wA);
  int32_t *idxB = (int32_t *)(smem_raw + L.idxB);
  T *wB = (T *)(smem_raw + L.wB);
  int32_t *toffA = (int32_t *)(smem_raw + L.toffA);
  int32_t *toffB = (int32_t *)(smem_raw + L.toffB);
  int32_t *ordA = (int32_t *)(smem_raw + L.ordA);
  int32_t *ordB = (int32_t *)(smem_raw + L.ordB);
  int32_t *zA = (int32_t *)(smem_raw + L.zA);
  int32_t *zB = (int32_t *)(smem_raw + L.zB);
  T *uS = (T *)(smem_raw + L.uS);
  int32_t *lo_s = (int32_t *)(smem_raw + L.lo);
  double *fr_s = (double *)(smem_raw + L.fr);
  uint8_t *zflag = (uint8_t *)(smem_raw + L.zflag);
  double *red = (double *)(smem_raw + L.red);
  int32_t *misc = (int32_t *)(smem_raw + L.misc);
  int64_t *s_item = (int64_t *)(misc + 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (;;) {
    if (tid == 0) *s_item = (int64_t)atomicAdd(counter, 1ull);
    __syncthreads();
    const int64_t item = *s_item;
    if (item >= work.n_items) break;

    // ---- decode the work item
    int ga, gb, ndir;
    int64_t slot0;
    decode_item(work, item, ga, gb, ndir, slot0);

    for (int dir = 0; dir < ndir; dir++) {
      const int g1 = dir ? gb : ga, g2 = dir ? ga : gb;
      const int64_t slot = slot0 + dir;
      const int na = CA.n_nodes[g1];
      const int nb = (dir ? CA : CB).n_nodes[g2];
      // dir == 1 only occurs in triangle mode, where CA and CB are the same corpus
      const DevCorpus &C2 = dir ? CA : CB;
      const int N = na > nb ? na : nb;
      const int P = (N + 1) | 1;
      const int KT = (N + R - 1) / R;
      const double invN = 1.0 / (double)N;

      // ---- prologue: both operators (normalize_pair + _row_normalized)
      int32_t *nzA = misc + 1, *nzB = misc + 2;
      bool ok = build_side<T, KB, R, true>(dir ? CB : CA, g1, N, P, dense, lo_s, fr_s, zflag, zA, nzA,
                                         toffA, ordA, idxA, wA, prm.cap, true, misc);
      if (ok)
        ok = build_side<T, KB, R, true>(C2, g2, N, P, dense, lo_s, fr_s, zflag, zB, nzB, toffB, ordB,
                                      idxB, wB, prm.cap, false, misc);
      if (!ok) {
        if (tid == 0) {
          const int k = atomicAdd(out.ovf_count, 1);
          if (k < out.ovf_cap) out.ovf_list[k] = ((work.mode == WORK_TRIANGLE ? work.u0 + item : item) << 2) | (dir << 1);
          if (out.iters) out.iters[slot] = -1;
        }
        __syncthreads();
        continue;
      }
      const int nzAv = *nzA, nzBv = *nzB;

      // ---- X_0 (similarity.py:134-135)
      const double uni = 1.0 / (double)((long long)N * N);
      for (int e = tid; e < (N + 1) * P; e += NT) {
        const int i = e / P, j = e - (e / P) * P;
        T v = 0;
        if (i < N && j < N) v = out.x0 ? (T)out.x0[(size_t)i * N + j] : (T)uni;
        Xs[e] = v;
      }
      __syncthreads();

      const T teleport = (T)((1.0 - prm.alpha) * uni);  // (1-alpha)*uniform, :140
      double r_old = 1.0, dp_prev = 1e300;
      int it_done = prm.max_iter;
      bool converged = false, ambiguous = false;

      for (int it = 1; it <= prm.max_iter; it++) {
        // ---- phase A: Y = A'^T X = S_A^T X + 1 u^T / N   (u = z_A^T X)
        phase_a<T, KB, NW, R>(Xs, Ys, idxA, wA, toffA, ordA, zA, nzAv, N, P, KT, (T)invN, lane, warp);
        __syncthreads();

        // ---- phase B: F = alpha' (Y S_B + v 1^T / N) + teleport  (v = Y z_B);
        //      m (first-order normalisation correction of delta) is only
        //      accumulated once delta is within 64x of tol.
        const bool need_m = prm.force_m || (dp_prev < 64.0 * prm.tol);
        T sl = 0, dl = 0, ml = 0;
        const T alpha_eff = (T)(prm.alpha * r_old);
        if (need_m)
          phase_b<T, KB, NW, R, true>(Xs, Ys, idxB, wB, toffB, ordB, zB, nzBv, N, P, KT, (T)invN, alpha_eff,
                                      (T)r_old, teleport, lane, warp, sl, dl, ml);
        else
          phase_b<T, KB, NW, R, false>(Xs, Ys, idxB, wB, toffB, ordB, zB, nzBv, N, P, KT, (T)invN, alpha_eff,
                                       (T)r_old, teleport, lane, warp, sl, dl, ml);

        // block reduction in a fixed order (deterministic, no atomics)
        double s3[3] = {(double)sl, (double)dl, (double)ml};
#pragma unroll
        for (int q = 0; q < 3; q++)
#pragma unroll
          for (int m = 16; m > 0; m >>= 1) s3[q] += shfl_xor_d(s3[q], m);
        if (lane == 0) {
          red[warp * 3 + 0] = s3[0];
          red[warp * 3 + 1] = s3[1];
          red[warp * 3 + 2] = s3[2];
        }
        __syncthreads();
        // every lane sums the NW partials with the same butterfly: identical
        // results in all warps
        const int src = lane % NW;
        double s = red[src * 3 + 0], dp = red[src * 3 + 1], mm = red[src * 3 + 2];
#pragma unroll
        for (int m = NW / 2; m > 0; m >>= 1) {
          s += shfl_xor_d(s, m);
          dp += shfl_xor_d(dp, m);
          mm += shfl_xor_d(mm, m);
        }
        const double r = 1.0 / s;  // fresh /= fresh.sum(), :141
        // sum |fresh - x| (:142) = dp + (r - 1) m to first order in |1 - s|
        const double delta = need_m ? dp + (r - 1.0) * mm : dp;
        if (!need_m && fabs(dp - prm.tol) <= 1.01 * fabs(1.0 - s) + 1e-300) {
          ambiguous = true;  // cannot decide without m: re-run this pair with force_m
          break;
        }
        r_old = r;
        dp_prev = dp;
        if (delta < prm.tol) {  // :144
          it_done = it;
          converged = true;
          break;
        }
      }
      if (ambiguous) {
        if (tid == 0) {
          const int k = atomicAdd(out.ovf_count, 1);
          if (k < out.ovf_cap) out.ovf_list[k] = ((work.mode == WORK_TRIANGLE ? work.u0 + item : item) << 2) | (dir << 1) | 1;
          if (out.iters) out.iters[slot] = -2;
        }
        __syncthreads();
        continue;
      }

      // ---- epilogue: X = F * r (normalised) in place
      {
        const T rr = (T)r_old;
        for (int e = tid; e < N * P; e += NT) {
          const int i = e / P, j = e - (e / P) * P;
          if (j < N) Xs[i * P + j] *= rr;
        }
      }
      __syncthreads();
      {
        const double wsum = greedy_match<T, KB>(Xs, P, N, (uint8_t *)Ys, lane, warp, NT >> 5, out.match);
        if (tid == 0) {
          if (out.d) out.d[slot] = isorank_distance_of(wsum, N);
          if (out.W) out.W[slot] = wsum;
          if (out.iters) out.iters[slot] = it_done;
          if (out.conv) out.conv[slot] = converged ? 1 : 0;
        }
      }
      if (out.X)
        for (int e = tid; e < N * N; e += NT) out.X[e] = (double)Xs[(e / N) * P + (e % N)];
      __syncthreads();
    }
  }
}

}  // namespace cfgsim
