// Large-N IsoRank pair kernel for sm_100a (129 <= N <= 1024; configs C4/C5).
//
// Same closed form as isorank_lr.cuh (start vector = uniform):
//     X_K = sum_{m<K} c alpha^m u_m v_m^T + (alpha^K/N^2) u_K v_K^T,
//     u_m = (A'^T)^m 1,  v_m = (B'^T)^m 1,   c = (1-alpha)/N^2,
// but nothing N x N lives on-chip.  One persistent CTA (256 threads) per pair;
// per pair and CTA a global-memory slab (L2-resident working set) holds the
// u/v histories, X and the sorted row orders.  Phases:
//
//  1. Operators (matrix.py:74-114, similarity.py:85-93).  The bilinear
//     upscale is the separable map  A_hat = W A W^T  (W: N x n, two nonzeros
//     per row, (1-fr_p) at lo_p and fr_p at lo_p+1), so the sweep
//     mat-vec  A'^T u = W A^T W^T D^-1 u + (1/N)(z^T u) 1  costs O(N + nnz(A))
//     per sweep from the source CSR/CSC, whatever the interpolation density.
//     D = row sums of A_hat (zero rows -> the uniform rank-1 term, :90-91).
//  2. Sweeps k = 1, 2, ...: two phases (t = A^T W^T D^-1 u_{k-1}, then
//     u_k = W t + zsum/N), u_k/v_k appended to the histories.  The stopping
//     test delta_k < tol (similarity.py:142-144) uses the exact bracket
//         (alpha^k/N) max(Da, Db) <= delta_k <= (alpha^k/N)(Da + Db),
//         Da = ||u_k - u_{k-1}||_1,  Db = ||v_k - v_{k-1}||_1
//     (both follow from 1^T u = 1^T v = N); only sweeps whose bracket
//     straddles tol evaluate delta_k exactly (N^2 pass, ~4 of ~75 sweeps).
//  3. X = U_coef V^T: register-tiled fp64 (or fp32) GEMM over the histories
//     (128 x 64 tiles, 8 x 4 per thread), the reference's fma order per
//     entry (m ascending, as the low-rank kernel's P accumulation).
//  4. Rows sorted into (value desc, column asc) by a warp bitonic sort of
//     packed 64-bit keys (exact; near-ties inside a truncated key are
//     re-ordered on exact values), then the greedy matching of
//     similarity.py:96-108 as "best head over active rows" rounds, W (:150,
//     summed in row order like Python's sum) and d (:160-173).
#pragma once
#include "isorank.cuh"

namespace cfgsim {

constexpr int BIG_THREADS = 256;
constexpr int BIG_WARPS = BIG_THREADS / 32;
constexpr int BIG_TM = 128, BIG_TN = 64, BIG_KC = 16;  // GEMM tile and k-chunk
constexpr int BIG_UP = BIG_TM + 8, BIG_VP = BIG_TN + 8;  // staged row pitches (== 8 mod 16 doubles)
constexpr int BIG_CB = 10;                            // column bits of a sort key (N <= 1024)
constexpr int BIG_R = 1024 / BIG_THREADS;             // greedy rows per thread

struct BigParams {
  double alpha;
  double tol;
  double eps;        // relative safety margin of the delta bracket
  int32_t max_iter;
  int32_t kcap;      // history capacity (iterations <= kcap by the bracket)
  int32_t nlim;      // max N of this launch
  unsigned char *slab;
  int64_t slab_bytes;  // per CTA
  int32_t *status;     // != 0: internal error (history overflow)
  unsigned long long *phase;  // optional (CFGSIM_PHASES=1): cycles per phase, summed over CTAs
  // given-X mode (isorank_align(start=...) for N > 128): X after the sweeps
  // was computed outside (isorank_start.cuh); the kernel only sorts and
  // matches it.  One pair, fp64.
  const double *xg;
  int32_t kg, convg;
  // history mode (all-pairs, fp64): the sequences u_m of every (graph, N)
  // come precomputed from isorank_seqbig_kernel (combo of sorted position q
  // = hcbase + q; rows of pitch big_hpitch(N)), so the pair skips its sweeps
  const double *hu;
  const double *hd;      // Du_m per combo, (kcap + 1) each
  int64_t hstride;       // combo -> offset of its row 0 in hu: combo * hstride
  int64_t hcbase;
  const double *hapow;   // alpha^m by sequential products (the sweeps' ak)
};

// history row pitch (doubles, 16-byte rows)
__host__ __device__ inline int big_hpitch(int N) { return (N + 1) & ~1; }

// per-CTA global slab
struct BigSlab {
  size_t coef, uh, vh, x, sval, scol, total;
};

template <typename T>
__host__ __device__ inline BigSlab big_slab_layout(int nlim, int kcap) {
  BigSlab s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o += (b + 255) & ~size_t(255);
    return at;
  };
  s.coef = take(sizeof(T) * (size_t)(kcap + 2));
  s.uh = take(sizeof(T) * (size_t)(kcap + 1) * nlim);
  s.vh = take(sizeof(T) * (size_t)(kcap + 1) * nlim);
  s.x = take(sizeof(T) * (size_t)nlim * nlim);
  s.sval = take(sizeof(unsigned long long) * (size_t)nlim * nlim);  // sorted exact value bits
  s.scol = take(sizeof(uint16_t) * (size_t)nlim * nlim);            // sorted columns
  s.total = o;
  return s;
}

// staged row: element e at e + (e >> 5) (one pad word per 32), so the sort's
// lane-contiguous reads (lane l: elements l * KB ..) spread over the banks
__host__ __device__ inline int big_row_pitch(int nlim) { return nlim + (nlim >> 5) + 1; }
__device__ __forceinline__ int big_rpos(int e) { return e + (e >> 5); }

// dynamic shared memory: a persistent head + a union of the phase regions
struct BigSmem {
  // sweep region (per side s = 0 (A), 1 (B))
  size_t lo[2], fr[2], rinv[2], pst[2], zf[2], t[2], ring[2], scr;
  // gemm region
  size_t us, vs;
  // sort region: one staged X row per warp
  size_t rows;
  // greedy region
  size_t taken, gslot, mrow, mval;
  size_t red, misc, total;
};

template <typename T>
__host__ __device__ inline BigSmem big_smem_layout(int nlim) {
  BigSmem s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o += (b + 15) & ~size_t(15);
    return at;
  };
  s.red = take(sizeof(double) * 2 * BIG_WARPS * 4);
  s.misc = take(256);
  const size_t base = o;
  for (int d = 0; d < 2; d++) {
    s.lo[d] = take(sizeof(int16_t) * nlim);
    s.fr[d] = take(sizeof(double) * nlim);
    s.rinv[d] = take(sizeof(double) * nlim);
    s.pst[d] = take(sizeof(int16_t) * (nlim + 2));
    s.zf[d] = take(sizeof(uint8_t) * nlim);
    s.t[d] = take(sizeof(T) * nlim);
    s.ring[d] = take(sizeof(T) * 2 * nlim);
  }
  s.scr = take(sizeof(double) * 2 * nlim);  // operator build scratch (colW, rowAW)
  const size_t sweep_end = o;
  o = base;
  s.us = take(sizeof(T) * 2 * BIG_KC * BIG_UP);  // double-buffered
  s.vs = take(sizeof(T) * 2 * BIG_KC * BIG_VP);
  const size_t gemm_end = o;
  o = base;
  s.rows = take(sizeof(T) * BIG_WARPS * (size_t)big_row_pitch(nlim));
  const size_t sort_end = o;
  o = base;
  s.taken = take(sizeof(uint32_t) * 64);  // two generations of taken columns
  s.gslot = take(sizeof(unsigned long long) * 2 * BIG_WARPS + sizeof(int32_t) * (4 * BIG_WARPS + 2));
  s.mrow = take(sizeof(int32_t) * nlim);
  s.mval = take(sizeof(unsigned long long) * nlim);
  const size_t greedy_end = o;
  size_t e = sweep_end > gemm_end ? sweep_end : gemm_end;
  e = e > greedy_end ? e : greedy_end;
  e = e > sort_end ? e : sort_end;
  s.total = e;
  return s;
}

// One side's operator, as the sweep phases see it.
struct BigSide {
  int n, N;
  int kind;  // 0: n == N (W = I), 1: interpolated, 2: n == 1 (every row uniform)
  const int32_t *rp, *cc;    // source CSR (row pointer local, columns)
  const double *rv;
  const int32_t *cp, *cr;    // source CSC (column pointer local, rows)
  const double *cv;
  int16_t *lo;               // interpolation: lo_p, fr_p (matrix.py:93-95)
  double *fr;
  double *rinv;              // 1 / D_p (0 on uniform rows)
  int16_t *pst;              // pst[r] = first p with lo_p >= r (r <= n)
  uint8_t *zf;               // uniform-row flag
  double zcount;             // number of uniform rows
};

// D_p and the uniform rows; interpolation tables.  Whole CTA.
__device__ inline void big_build_side(BigSide &S, double *scratch_n) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int n = S.n, N = S.N;
  if (S.kind == 1) {
    for (int p = tid; p < N; p += NT) {  // matrix.py:93-95, same operation order
      const double pos = __ddiv_rn((double)((long long)p * (n - 1)), (double)(N - 1));
      int l = (int)floor(pos);
      if (l > n - 2) l = n - 2;
      S.lo[p] = (int16_t)l;
      S.fr[p] = __dsub_rn(pos, (double)l);
    }
    __syncthreads();
    // pst[r] = first p with lo_p >= r, r = 0..n (lo is non-decreasing)
    for (int r = tid; r <= n; r += NT) {
      int a = 0, b = N;
      while (a < b) {
        const int m = (a + b) >> 1;
        if (S.lo[m] < r) a = m + 1; else b = m;
      }
      S.pst[r] = (int16_t)a;
    }
    // colW[c] = sum_q W[q, c];  rowAW[r] = sum_c A[r, c] colW[c]
    double *colW = scratch_n, *rowAW = scratch_n + n;
    __syncthreads();
    for (int c = tid; c < n; c += NT) {
      double s = 0.0;
      if (c <= n - 2)
        for (int q = S.pst[c]; q < S.pst[c + 1]; q++) s += 1.0 - S.fr[q];
      if (c >= 1)
        for (int q = S.pst[c - 1]; q < S.pst[c]; q++) s += S.fr[q];
      colW[c] = s;
    }
    __syncthreads();
    for (int r = tid; r < n; r += NT) {
      double s = 0.0;
      for (int e = S.rp[r]; e < S.rp[r + 1]; e++) s += S.rv[e] * colW[S.cc[e]];
      rowAW[r] = s;
    }
    __syncthreads();
    for (int p = tid; p < N; p += NT) {
      const int l = S.lo[p];
      const double f = S.fr[p];
      const double D = (1.0 - f) * rowAW[l] + f * rowAW[l + 1];
      S.zf[p] = (D == 0.0);
      S.rinv[p] = (D == 0.0) ? 0.0 : 1.0 / D;
    }
  } else if (S.kind == 0) {
    for (int p = tid; p < N; p += NT) {
      double s = 0.0;
      for (int e = S.rp[p]; e < S.rp[p + 1]; e++) s += S.rv[e];
      S.zf[p] = (s == 0.0);
      S.rinv[p] = (s == 0.0) ? 0.0 : 1.0 / s;
    }
  } else {
    for (int p = tid; p < N; p += NT) {
      S.zf[p] = 1;
      S.rinv[p] = 0.0;
    }
  }
  __syncthreads();
  // number of uniform rows (zsum_0 = |z| since u_0 = 1)
  int cnt = 0;
  for (int p = tid; p < N; p += NT) cnt += S.zf[p];
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  __shared__ int zc_sh[BIG_WARPS];
  if ((tid & 31) == 0) zc_sh[tid >> 5] = cnt;
  __syncthreads();
  int tot = 0;
  for (int w = 0; w < (NT >> 5); w++) tot += zc_sh[w];
  S.zcount = (double)tot;
  __syncthreads();
}

// phase 1: t[c] = sum_r A[r, c] s_r,  s = W^T D^-1 u  (n-vector), c < n
template <typename T>
__device__ __forceinline__ T big_t_entry(const BigSide &S, const T *u, int c) {
  double acc = 0.0;
  if (S.kind == 0) {
    for (int e = S.cp[c]; e < S.cp[c + 1]; e++) {
      const int r = S.cr[e];
      acc = fma(S.cv[e], (double)u[r] * S.rinv[r], acc);
    }
  } else {
    const int n = S.n;
    for (int e = S.cp[c]; e < S.cp[c + 1]; e++) {
      const int r = S.cr[e];
      double s = 0.0;  // s_r = sum_{lo_p = r} (1-fr_p) y_p + sum_{lo_p = r-1} fr_p y_p
      if (r <= n - 2)
        for (int p = S.pst[r]; p < S.pst[r + 1]; p++) s = fma(1.0 - S.fr[p], (double)u[p] * S.rinv[p], s);
      if (r >= 1)
        for (int p = S.pst[r - 1]; p < S.pst[r]; p++) s = fma(S.fr[p], (double)u[p] * S.rinv[p], s);
      acc = fma(S.cv[e], s, acc);
    }
  }
  return (T)acc;
}

// phase 1a (interpolated sides): s_r = sum_{lo_p = r} (1-fr_p) y_p +
// sum_{lo_p = r-1} fr_p y_p, y = D^-1 u — the same fma chain big_t_entry
// forms inline, computed once per source row r instead of once per entry
// of column r in every column's sum (deg_in(r) times, by only n threads)
template <typename T>
__device__ __forceinline__ double big_s_entry(const BigSide &S, const T *u, int r) {
  const int n = S.n;
  double s = 0.0;
  if (r <= n - 2)
    for (int p = S.pst[r]; p < S.pst[r + 1]; p++) s = fma(1.0 - S.fr[p], (double)u[p] * S.rinv[p], s);
  if (r >= 1)
    for (int p = S.pst[r - 1]; p < S.pst[r]; p++) s = fma(S.fr[p], (double)u[p] * S.rinv[p], s);
  return s;
}

// phase 1b: t[c] = sum_r A[r, c] s_r over column c (bitwise big_t_entry)
template <typename T>
__device__ __forceinline__ T big_t_from_s(const BigSide &S, const double *sb, int c) {
  double acc = 0.0;
  for (int e = S.cp[c]; e < S.cp[c + 1]; e++) acc = fma(S.cv[e], sb[S.cr[e]], acc);
  return (T)acc;
}

// phase 2: u'[q] = (W t)[q] + zsum / N
template <typename T>
__device__ __forceinline__ T big_u_entry(const BigSide &S, const T *t, int q, double zterm) {
  if (S.kind == 2) return (T)zterm;
  if (S.kind == 0) return (T)((double)t[q] + zterm);
  const int l = S.lo[q];
  const double f = S.fr[q];
  return (T)((1.0 - f) * (double)t[l] + f * (double)t[l + 1] + zterm);
}

template <typename T>
__device__ __forceinline__ unsigned long long big_sort_key(T v, int col, int emin, int shift) {
  if (sizeof(T) == 8) {
    const unsigned long long b = (unsigned long long)__double_as_longlong((double)v);
    const unsigned long long e = ((b >> 52) & 0x7ff) - (unsigned long long)emin;
    const unsigned long long m = b & ((1ull << 52) - 1);
    const unsigned long long vp = ((e << 52) | m) >> shift;
    return (vp << BIG_CB) | (unsigned long long)((1 << BIG_CB) - 1 - col);
  } else {
    const unsigned int b = __float_as_uint((float)v);
    return ((unsigned long long)b << BIG_CB) | (unsigned long long)((1 << BIG_CB) - 1 - col);
  }
}

template <typename T>
__device__ __forceinline__ int big_exponent(T v) {
  return (sizeof(T) == 8) ? (int)((__double_as_longlong((double)v) >> 52) & 0x7ff)
                          : (int)((__float_as_uint((float)v) >> 23) & 0xff);
}

template <typename T>
__device__ __forceinline__ unsigned long long big_bits(T v) {
  return (sizeof(T) == 8) ? (unsigned long long)__double_as_longlong((double)v)
                          : (unsigned long long)__float_as_uint((float)v);
}

__device__ __forceinline__ int big_key_col(unsigned long long k) {
  return (1 << BIG_CB) - 1 - (int)(k & ((1ull << BIG_CB) - 1));
}

// greedy rounds: entries prefetched to L2 ahead of a row's register window
#ifndef CFGSIM_BIG_L2_AHEAD
constexpr int BIG_L2_AHEAD = 16;
#else
constexpr int BIG_L2_AHEAD = CFGSIM_BIG_L2_AHEAD;
#endif
__device__ __forceinline__ void big_prefetch_l2(const void *p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

__device__ __forceinline__ void big_cp_async_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// B-byte async copy global -> shared; zero-fills the destination when !valid
template <int B>
__device__ __forceinline__ void big_cp_async_zfill(void *smem_dst, const void *gsrc, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int n = valid ? B : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(d), "l"(gsrc), "n"(B), "r"(n) : "memory");
}

__device__ __forceinline__ void big_cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int G>
__device__ __forceinline__ void big_cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(G) : "memory"); }

// compare-exchange of registers c and c ^ J inside each lane, larger key to
// the lower register (every block descending: see big_sort_desc)
template <typename K, int KB, int J>
__device__ __forceinline__ void big_stage_reg(K (&v)[KB]) {
#pragma unroll
  for (int c = 0; c < KB; c++) {
    if ((c & J) == 0) {
      const K a = v[c], b = v[c | J];
      v[c] = a > b ? a : b;
      v[c | J] = a > b ? b : a;
    }
  }
}

// Warp bitonic sort of 32*KB distinct keys, descending; element e = lane*KB + c
// (each lane holds a contiguous run, so only log2(32) of every merge's stages
// cross lanes).  During merge level k the blocks with bit k of e set sort
// ascending; they hold their keys complemented (~key), so every
// compare-exchange runs descending with no per-exchange direction select, and
// one xor per key re-targets the complement between levels.  Stage loops stay
// rolled: the fully unrolled 1024-key network does not fit the instruction cache.
template <typename K, int KB>
__device__ __forceinline__ void big_sort_desc(K (&v)[KB], int lane) {
  constexpr int n = 32 * KB;
  auto flip = [&](int c, int k) -> K { return (((lane * KB + c) & k) != 0) ? ~K(0) : K(0); };
#pragma unroll
  for (int c = 0; c < KB; c++) v[c] ^= flip(c, 2);
#pragma unroll 1
  for (int k = 2; k <= n; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= KB) {
        const int lm = j / KB;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int c = 0; c < KB; c++) {
          const K o = __shfl_xor_sync(0xffffffffu, v[c], lm);
          v[c] = lower ? (o > v[c] ? o : v[c]) : (o > v[c] ? v[c] : o);
        }
      } else {
        switch (j) {
          case 1: big_stage_reg<K, KB, 1>(v); break;
          case 2: if constexpr (KB > 2) big_stage_reg<K, KB, 2>(v); break;
          case 4: if constexpr (KB > 4) big_stage_reg<K, KB, 4>(v); break;
          case 8: if constexpr (KB > 8) big_stage_reg<K, KB, 8>(v); break;
          case 16: if constexpr (KB > 16) big_stage_reg<K, KB, 16>(v); break;
          default: break;
        }
      }
    }
    if (k < n) {  // level 2k's complement (bit k of e ends up 0 at the last level)
#pragma unroll
      for (int c = 0; c < KB; c++) v[c] ^= flip(c, k) ^ flip(c, 2 * k);
    }
  }
}

// per-phase cycle accounting (debug): phase k's time = clock at mark k+1 - mark k
#define BIG_PHASE(k)                                                                  \
  do {                                                                                \
    if (prm.phase && threadIdx.x == 0) {                                              \
      const unsigned long long now = clock64();                                       \
      if ((k) > 0) atomicAdd(prm.phase + (k) - 1, now - t_phase);                      \
      t_phase = now;                                                                  \
    }                                                                                 \
  } while (0)

// one side's operator tables in shared memory region `sd` (0 / 1)
__device__ __forceinline__ void big_side_init(BigSide &S, const DevCorpus &Cs, int g, int N, unsigned char *smem_raw,
                                              const BigSmem &L, int sd) {
  S.n = Cs.n_nodes[g];
  S.N = N;
  S.kind = (S.n == N) ? 0 : (S.n == 1 ? 2 : 1);
  S.rp = Cs.rowptr + Cs.rp_off[g];
  S.cc = Cs.col + Cs.nz_off[g];
  S.rv = Cs.val + Cs.nz_off[g];
  S.cp = Cs.cscp + Cs.rp_off[g];
  S.cr = Cs.csc_row + Cs.nz_off[g];
  S.cv = Cs.csc_val + Cs.nz_off[g];
  S.lo = (int16_t *)(smem_raw + L.lo[sd]);
  S.fr = (double *)(smem_raw + L.fr[sd]);
  S.rinv = (double *)(smem_raw + L.rinv[sd]);
  S.pst = (int16_t *)(smem_raw + L.pst[sd]);
  S.zf = (uint8_t *)(smem_raw + L.zf[sd]);
  big_build_side(S, (double *)(smem_raw + L.scr));
}

template <typename T, int KB>
__global__ void __launch_bounds__(BIG_THREADS, 2)
    isorank_big_kernel(DevCorpus CA, DevCorpus CB, PairWork work, PairOut out, BigParams prm,
                       unsigned long long *counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const BigSmem L = big_smem_layout<T>(prm.nlim);
  const BigSlab G = big_slab_layout<T>(prm.nlim, prm.kcap);
  unsigned char *slab = prm.slab + (size_t)blockIdx.x * prm.slab_bytes;
  T *coef = (T *)(slab + G.coef);
  T *Uh = (T *)(slab + G.uh);
  T *Vh = (T *)(slab + G.vh);
  T *X = prm.xg ? (T *)prm.xg : (T *)(slab + G.x);
  unsigned long long *sval = (unsigned long long *)(slab + G.sval);
  uint16_t *scol = (uint16_t *)(slab + G.scol);
  double *red = (double *)(smem_raw + L.red);
  int64_t *s_item = (int64_t *)(smem_raw + L.misc);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = BIG_THREADS;
  unsigned long long t_phase = 0;

  for (;;) {
    if (tid == 0) *s_item = (int64_t)atomicAdd(counter, 1ull);
    __syncthreads();
    const int64_t item = *s_item;
    if (item >= work.n_items) break;
    int ga, gb, ndir;
    int64_t slot0;
    decode_item(work, item, ga, gb, ndir, slot0);

    for (int dir = 0; dir < ndir; dir++) {
      const int g1 = dir ? gb : ga, g2 = dir ? ga : gb;
      const int64_t slot = slot0 + dir;
      const DevCorpus &C1 = dir ? CB : CA;
      const DevCorpus &C2 = dir ? CA : CB;
      const int na = C1.n_nodes[g1], nb = C2.n_nodes[g2];
      const int N = na > nb ? na : nb;

      int it_done = prm.max_iter;
      bool converged = false;
      int emin = 0x7fffffff, emax = -1;
      if (prm.xg) {  // given X: its exponent range only
        it_done = prm.kg;
        converged = prm.convg != 0;
        for (int e = tid; e < N * N; e += NT) {
          const int x = big_exponent(X[e]);
          emin = min(emin, x);
          emax = max(emax, x);
        }
      } else {
      int K = 0;
      const double invN = 1.0 / (double)N;
      const double inv_nn = 1.0 / (double)((long long)N * N);
      const double c = (1.0 - prm.alpha) * inv_nn;  // (1-alpha)*uniform, similarity.py:140
      const double *hUA = nullptr, *hUB = nullptr;
      const int HP = big_hpitch(N);
      if (prm.hu) {
        // ---- 1-2 (history mode). The stopping sweep from the precomputed
        // Du_m / Dv_m: every sweep's bracket in parallel, then the exact
        // delta (the sweeps' formula and reduction, bitwise) only for the
        // straddling sweeps before the first certain stop, in order
        BIG_PHASE(0);
        int pa, pb;
        {
          const int64_t u = work.u0 + item;
          int lo = 0, hi = work.K - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (work.row_start[mid] <= u) lo = mid; else hi = mid - 1;
          }
          pa = lo;
          pb = lo + (int)(u - work.row_start[lo]);
          if (work.perm[pa] > work.perm[pb]) { const int t = pa; pa = pb; pb = t; }  // side A = lower graph id
        }
        const int64_t ca = prm.hcbase + pa, cb = prm.hcbase + pb;
        hUA = prm.hu + ca * prm.hstride;
        hUB = prm.hu + cb * prm.hstride;
        const double *DA = prm.hd + ca * (int64_t)(prm.kcap + 1), *DB = prm.hd + cb * (int64_t)(prm.kcap + 1);
        int *s_first = (int *)(smem_raw + L.misc + 128);
        uint32_t *amb = (uint32_t *)(smem_raw + L.misc + 160);  // kcap <= 511
        const int mmax = prm.max_iter < prm.kcap ? prm.max_iter : prm.kcap;
        if (tid == 0) *s_first = 0x7fffffff;
        for (int q = tid; q < 16; q += NT) amb[q] = 0u;
        __syncthreads();
        for (int m = tid + 1; m <= mmax; m += NT) {
          const double ak = prm.hapow[m];
          const double da = DA[m], db = DB[m];
          const double hiB = ak * invN * (da + db) * (1.0 + prm.eps);
          const double loB = ak * invN * fmax(da, db) * (1.0 - prm.eps);
          if (hiB < prm.tol) atomicMin(s_first, m);
          else if (loB < prm.tol) atomicOr(amb + (m >> 5), 1u << (m & 31));
        }
        __syncthreads();
        const int first = *s_first;
        K = mmax;
        if (first != 0x7fffffff) { K = first; converged = true; }
        const int lim = first == 0x7fffffff ? mmax : first - 1;
        for (int wd = 0; wd <= (lim >> 5); wd++) {
          uint32_t bits = amb[wd];
          bool done = false;
          while (bits) {
            const int m = wd * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            if (m > lim) break;
            const double *un = hUA + (size_t)m * HP, *uo = hUA + (size_t)(m - 1) * HP;
            const double *vn = hUB + (size_t)m * HP, *vo = hUB + (size_t)(m - 1) * HP;
            double dl = 0.0, dl2 = 0.0;
            for (int i = warp; i < N; i += BIG_WARPS) {
              const double a = un[i], b = uo[i];
              for (int j = lane; j < N; j += 64) {
                dl += fabs(fma(-b, vo[j], a * vn[j]));
                if (j + 32 < N) dl2 += fabs(fma(-b, vo[j + 32], a * vn[j + 32]));
              }
            }
            dl += dl2;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dl += __shfl_xor_sync(0xffffffffu, dl, o);
            __syncthreads();  // (red reused)
            if (lane == 0) red[warp * 4] = dl;
            __syncthreads();
            double Ssum = 0.0;
            for (int w = 0; w < BIG_WARPS; w++) Ssum += red[w * 4];
            if (prm.hapow[m] * inv_nn * Ssum < prm.tol) {  // similarity.py:144
              K = m;
              converged = true;
              done = true;
              break;
            }
          }
          if (done) break;
        }
        it_done = converged ? K : prm.max_iter;
        if (!converged && prm.max_iter > prm.kcap) {  // cannot happen: the bracket stops by kcap
          if (tid == 0) {
            atomicExch(prm.status, 1);
            if (out.iters) out.iters[slot] = -2;
          }
          __syncthreads();
          continue;
        }
        __syncthreads();
      } else {
      BIG_PHASE(0);
      // ---- 1. operators
      BigSide SA, SB;
      auto setup = [&](BigSide &S, const DevCorpus &Cs, int g, int sd) { big_side_init(S, Cs, g, N, smem_raw, L, sd); };
      setup(SA, C1, g1, 0);
      setup(SB, C2, g2, 1);
      T *ring[2] = {(T *)(smem_raw + L.ring[0]), (T *)(smem_raw + L.ring[1])};
      double *sbuf = (double *)(smem_raw + L.scr);  // s per source row (2 sides, nlim each); free after setup
      const int nlim_s = prm.nlim;
      T *tv[2] = {(T *)(smem_raw + L.t[0]), (T *)(smem_raw + L.t[1])};

      BIG_PHASE(1);
      // ---- 2. sweeps
      for (int q = tid; q < N; q += NT) {
        ring[0][q] = (T)1;
        ring[1][q] = (T)1;
        Uh[q] = (T)1;
        Vh[q] = (T)1;
      }
      double zsum[2] = {SA.zcount, SB.zcount};
      double ak1 = 1.0;                             // alpha^(k-1)
      int k = 1;
      __syncthreads();
      for (;; k++) {
        const int cur = (k - 1) & 1, nxt = k & 1;  // ring slots of u_{k-1}, u_k
        // phase 1: t = A^T W^T D^-1 u_{k-1}; interpolated sides in two steps
        // (s = W^T D^-1 u per source row into the operator-build scratch,
        // then the column sums), identical arithmetic to the fused form
        {
          const int n0 = SA.kind == 2 ? 0 : SA.n;
          const int n1 = SB.kind == 2 ? 0 : SB.n;
          if (SA.kind == 1 || SB.kind == 1) {
            const int m0 = SA.kind == 1 ? SA.n : 0, m1 = SB.kind == 1 ? SB.n : 0;
            for (int q = tid; q < m0 + m1; q += NT) {
              if (q < m0) sbuf[q] = big_s_entry<T>(SA, ring[0] + cur * N, q);
              else sbuf[nlim_s + q - m0] = big_s_entry<T>(SB, ring[1] + cur * N, q - m0);
            }
            __syncthreads();
          }
          for (int q = tid; q < n0 + n1; q += NT) {
            if (q < n0)
              tv[0][q] = SA.kind == 1 ? big_t_from_s<T>(SA, sbuf, q) : big_t_entry<T>(SA, ring[0] + cur * N, q);
            else
              tv[1][q - n0] = SB.kind == 1 ? big_t_from_s<T>(SB, sbuf + nlim_s, q - n0)
                                           : big_t_entry<T>(SB, ring[1] + cur * N, q - n0);
          }
        }
        __syncthreads();
        // phase 2: u_k = W t + zsum/N; partial sums of |u_k - u_{k-1}| and z^T u_k
        double part[4] = {0.0, 0.0, 0.0, 0.0};
        {
          // (each side with the same thread mapping, q = tid + NT j, as the
          // per-(graph, N) history kernel: identical per-thread partial sums,
          // hence bitwise-identical sequences on both paths)
          const double za = zsum[0] * invN, zb = zsum[1] * invN;
          for (int q = tid; q < N; q += NT) {
            const T un = big_u_entry<T>(SA, tv[0], q, za);
            const T uo = ring[0][cur * N + q];
            ring[0][nxt * N + q] = un;
            if (k <= prm.kcap) Uh[(size_t)k * N + q] = un;
            part[0] += fabs((double)un - (double)uo);
            if (SA.zf[q]) part[1] += (double)un;
          }
          for (int i = tid; i < N; i += NT) {
            const T un = big_u_entry<T>(SB, tv[1], i, zb);
            const T uo = ring[1][cur * N + i];
            ring[1][nxt * N + i] = un;
            if (k <= prm.kcap) Vh[(size_t)k * N + i] = un;
            part[2] += fabs((double)un - (double)uo);
            if (SB.zf[i]) part[3] += (double)un;
          }
        }
#pragma unroll
        for (int v = 0; v < 4; v++) {
#pragma unroll
          for (int m = 16; m > 0; m >>= 1) part[v] += __shfl_xor_sync(0xffffffffu, part[v], m);
        }
        double *rb = red + (k & 1) * BIG_WARPS * 4;
        if (lane == 0)
#pragma unroll
          for (int v = 0; v < 4; v++) rb[warp * 4 + v] = part[v];
        __syncthreads();
        double tot[4] = {0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < BIG_WARPS; w++)
#pragma unroll
          for (int v = 0; v < 4; v++) tot[v] += rb[w * 4 + v];
        zsum[0] = tot[1];
        zsum[1] = tot[3];
        const double ak = ak1 * prm.alpha;
        const double da = tot[0], db = tot[2];
        const double hi = ak * invN * (da + db) * (1.0 + prm.eps);
        const double lo = ak * invN * fmax(da, db) * (1.0 - prm.eps);
        bool stop = false;
        if (hi < prm.tol) {
          stop = true;
        } else if (lo < prm.tol) {
          // bracket straddles tol: exact delta_k = alpha^k/N^2 sum |u_k v_k^T - u_{k-1} v_{k-1}^T|
          const T *un = ring[0] + nxt * N, *uo = ring[0] + cur * N;
          const T *vn = ring[1] + nxt * N, *vo = ring[1] + cur * N;
          double dl = 0.0, dl2 = 0.0;
          for (int i = warp; i < N; i += BIG_WARPS) {
            const T a = un[i], b = uo[i];
            for (int j = lane; j < N; j += 64) {
              dl += fabs((double)fma(-b, vo[j], a * vn[j]));
              if (j + 32 < N) dl2 += fabs((double)fma(-b, vo[j + 32], a * vn[j + 32]));
            }
          }
          dl += dl2;
#pragma unroll
          for (int m = 16; m > 0; m >>= 1) dl += __shfl_xor_sync(0xffffffffu, dl, m);
          __syncthreads();  // everyone has read rb
          if (lane == 0) rb[warp * 4] = dl;
          __syncthreads();
          double S = 0.0;
          for (int w = 0; w < BIG_WARPS; w++) S += rb[w * 4];
          stop = ak * inv_nn * S < prm.tol;  // similarity.py:144
        }
        if (stop) {
          it_done = k;
          converged = true;
          break;
        }
        if (k >= prm.max_iter) break;
        ak1 = ak;
      }
      K = k;  // x after K sweeps (similarity.py:139-148)
      if (K > prm.kcap) {  // cannot happen: the bracket stops by kcap
        if (tid == 0) {
          atomicExch(prm.status, 1);
          if (out.iters) out.iters[slot] = -2;
        }
        __syncthreads();
        continue;
      }
      }  // (sweeps)
      // coefficients: c alpha^m (m < K), alpha^K / N^2 (m = K)
      if (tid == 0) {
        double a = 1.0;
        for (int m = 0; m < K; m++) {
          coef[m] = (T)(c * a);
          a *= prm.alpha;
        }
        coef[K] = (T)(a * inv_nn);
      }
      __syncthreads();

      BIG_PHASE(2);
      // ---- 3. X = sum_m coef_m u_m v_m^T  (128 x 64 tiles, 8 x 4 per thread,
      //         k-chunks of the histories double-buffered with cp.async);
      //         exponent range of X for the pair-wide sort keys.
      //         u_m is pre-scaled by coef_m in place (the product the
      //         low-rank kernel forms as cak * u).
      if (prm.hu) {  // the product's operands from the histories: coef_m u_m, v_m (pitch N)
        for (int e = tid; e < (K + 1) * N; e += NT) {
          const int m = e / N, i = e - m * N;
          Uh[e] = coef[m] * (T)hUA[(size_t)m * HP + i];
          Vh[e] = (T)hUB[(size_t)m * HP + i];
        }
      } else {
        for (int e = tid; e < (K + 1) * N; e += NT) Uh[e] = coef[e / N] * Uh[e];
      }
      __syncthreads();
      {
        T *Us = (T *)(smem_raw + L.us);
        T *Vs = (T *)(smem_raw + L.vs);
        const int ty = tid >> 4, tx = tid & 15;
        const int nch = (K + BIG_KC) / BIG_KC;  // chunks covering m = 0..K
        auto stage = [&](int i0, int j0, int ch, int bufi) {
          T *us = Us + bufi * BIG_KC * BIG_UP, *vs = Vs + bufi * BIG_KC * BIG_VP;
          for (int e = tid; e < BIG_KC * (BIG_TM + BIG_TN); e += NT) {
            int mm, x, lim;
            const T *src;
            T *dst;
            if (e < BIG_KC * BIG_TM) {
              mm = e / BIG_TM; x = e % BIG_TM; lim = N - i0;
              src = Uh + (size_t)(ch * BIG_KC + mm) * N + i0 + x;
              dst = us + mm * BIG_UP + x;
            } else {
              const int f = e - BIG_KC * BIG_TM;
              mm = f / BIG_TN; x = f % BIG_TN; lim = N - j0;
              src = Vh + (size_t)(ch * BIG_KC + mm) * N + j0 + x;
              dst = vs + mm * BIG_VP + x;
            }
            const bool ok = (ch * BIG_KC + mm <= K) && x < lim;
            big_cp_async_zfill<sizeof(T)>(dst, ok ? (const void *)src : (const void *)Uh, ok);
          }
          big_cp_async_commit();
        };
        if constexpr (sizeof(T) == 8) {
          // fp64 tensor cores: mma.m8n8k4 is the fma chain over k in order
          // (bitwise equal to the scalar m-ascending accumulation; probed:
          // tools/probes/dmma_probe.cu).  8 warps as 4 x 2, 4 x 4 tiles each.
          const int wr = warp & 3, wc = warp >> 2;
          const int lr = lane >> 2, lk = lane & 3;
          for (int i0 = 0; i0 < N; i0 += BIG_TM)
            for (int j0 = 0; j0 < N; j0 += BIG_TN) {
              double acc[4][4][2];
#pragma unroll
              for (int x = 0; x < 4; x++)
#pragma unroll
                for (int y = 0; y < 4; y++) acc[x][y][0] = acc[x][y][1] = 0.0;
              __syncthreads();  // previous tile done with both buffers
              stage(i0, j0, 0, 0);
              for (int ch = 0; ch < nch; ch++) {
                if (ch + 1 < nch) {
                  stage(i0, j0, ch + 1, (ch + 1) & 1);
                  big_cp_async_wait_group<1>();
                } else {
                  big_cp_async_wait_group<0>();
                }
                __syncthreads();
                const double *us = (const double *)Us + (ch & 1) * BIG_KC * BIG_UP;
                const double *vs = (const double *)Vs + (ch & 1) * BIG_KC * BIG_VP;
#pragma unroll
                for (int k0 = 0; k0 < BIG_KC; k0 += 4) {
                  double af[4], bf[4];
#pragma unroll
                  for (int x = 0; x < 4; x++) af[x] = us[(k0 + lk) * BIG_UP + wr * 32 + x * 8 + lr];
#pragma unroll
                  for (int y = 0; y < 4; y++) bf[y] = vs[(k0 + lk) * BIG_VP + wc * 32 + y * 8 + lr];
#pragma unroll
                  for (int x = 0; x < 4; x++)
#pragma unroll
                    for (int y = 0; y < 4; y++)
                      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                   : "+d"(acc[x][y][0]), "+d"(acc[x][y][1])
                                   : "d"(af[x]), "d"(bf[y]));
                }
                __syncthreads();  // buffer (ch & 1) is re-staged by chunk ch + 2
              }
#pragma unroll
              for (int x = 0; x < 4; x++)
#pragma unroll
                for (int y = 0; y < 4; y++)
#pragma unroll
                  for (int h = 0; h < 2; h++) {
                    const int i = i0 + wr * 32 + x * 8 + lr, j = j0 + wc * 32 + y * 8 + 2 * lk + h;
                    if (i < N && j < N) {
                      X[(size_t)i * N + j] = (T)acc[x][y][h];
                      const int e = big_exponent(acc[x][y][h]);
                      emin = min(emin, e);
                      emax = max(emax, e);
                    }
                  }
            }
        } else {
        for (int i0 = 0; i0 < N; i0 += BIG_TM)
            for (int j0 = 0; j0 < N; j0 += BIG_TN) {
              T acc[8][4];
#pragma unroll
              for (int a = 0; a < 8; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) acc[a][b] = (T)0;
              __syncthreads();  // previous tile done with both buffers
              stage(i0, j0, 0, 0);
              for (int ch = 0; ch < nch; ch++) {
                if (ch + 1 < nch) {
                  stage(i0, j0, ch + 1, (ch + 1) & 1);
                  big_cp_async_wait_group<1>();
                } else {
                  big_cp_async_wait_group<0>();
                }
                __syncthreads();
                const T *us = Us + (ch & 1) * BIG_KC * BIG_UP, *vs = Vs + (ch & 1) * BIG_KC * BIG_VP;
#pragma unroll
                for (int mm = 0; mm < BIG_KC; mm++) {
                  T ua[8], vb[4];
#pragma unroll
                  for (int a = 0; a < 8; a++) ua[a] = us[mm * BIG_UP + ty + 16 * a];
#pragma unroll
                  for (int b = 0; b < 4; b++) vb[b] = vs[mm * BIG_VP + tx + 16 * b];
#pragma unroll
                  for (int a = 0; a < 8; a++)
#pragma unroll
                    for (int b = 0; b < 4; b++) acc[a][b] = fma(ua[a], vb[b], acc[a][b]);
                }
                __syncthreads();  // buffer (ch & 1) is re-staged by chunk ch + 2
              }
#pragma unroll
              for (int a = 0; a < 8; a++) {
                const int i = i0 + ty + 16 * a;
#pragma unroll
                for (int b = 0; b < 4; b++) {
                  const int j = j0 + tx + 16 * b;
                  if (i < N && j < N) {
                    X[(size_t)i * N + j] = acc[a][b];
                    const int e = big_exponent(acc[a][b]);
                    emin = min(emin, e);
                    emax = max(emax, e);
                  }
                }
              }
            }
        }
      }
      }  // (phases 1-3)
      {
        int *ered = (int *)(smem_raw + L.misc + 32);
        emin = __reduce_min_sync(0xffffffffu, emin);
        emax = __reduce_max_sync(0xffffffffu, emax);
        if (lane == 0) {
          ered[warp] = emin;
          ered[BIG_WARPS + warp] = emax;
        }
        __syncthreads();
        for (int w = 0; w < BIG_WARPS; w++) {
          emin = min(emin, ered[w]);
          emax = max(emax, ered[BIG_WARPS + w]);
        }
      }
      // low mantissa bits dropped so that (rebased exponent | mantissa | column)
      // fits 64 bits; the same base for every row keeps keys comparable across rows
      int shift = 0;
      if (sizeof(T) == 8) {
        shift = (32 - __clz(emax - emin)) + 52 + BIG_CB - 64;
        if (shift < 0) shift = 0;
      }
      __syncthreads();

      BIG_PHASE(3);
      // ---- 4a. row orders (value desc, column asc).  One warp per row sorts
      // 32-bit keys (top 22 bits of the row-rebased value | inverted column),
      // then gathers the exact values into pair-wide 64-bit keys in sorted
      // order; equal 22-bit prefixes with different exact values (near-ties,
      // ~1e-6 relative) are repaired by odd-even transposition on the exact
      // keys.  Exactly tied values keep column order from the key's low bits.
      T *rbuf = (T *)(smem_raw + L.rows) + (size_t)warp * big_row_pitch(prm.nlim);
      for (int i = warp; i < N; i += BIG_WARPS) {
        // row i staged in shared memory with one coalesced pass (the sort's
        // key build, exact-value gathers and near-tie repair then read it
        // there instead of re-reading the HBM slab lane-strided / at random)
        const T *grow = X + (size_t)i * N;
        const T *row = rbuf;
        int rmin = 0x7fffffff, rmax = -1;
#pragma unroll 8
        for (int j = lane; j < N; j += 32) {
          const T v = grow[j];
          rbuf[big_rpos(j)] = v;
          const int e = big_exponent(v);
          rmin = min(rmin, e);
          rmax = max(rmax, e);
        }
        __syncwarp();
        rmin = __reduce_min_sync(0xffffffffu, rmin);
        rmax = __reduce_max_sync(0xffffffffu, rmax);
        constexpr int MB = sizeof(T) == 8 ? 52 : 23;
        const int rshift = (32 - __clz(rmax - rmin)) + MB - 22;  // value bits above the 22 kept
        uint32_t key[KB];
#pragma unroll
        for (int c = 0; c < KB; c++) {
          const int j = lane * KB + c;
          uint32_t k = 0u;  // padding sorts last (a real key's column field is >= 1024 - N >= 1 then)
          if (j < N) {
            const unsigned long long b = big_bits(row[big_rpos(j)]);
            const unsigned long long v =
                ((((b >> MB) & (sizeof(T) == 8 ? 0x7ffull : 0xffull)) - (unsigned long long)rmin) << MB) |
                (b & ((1ull << MB) - 1));
            k = ((uint32_t)(v >> rshift) << BIG_CB) | (uint32_t)((1 << BIG_CB) - 1 - j);
          }
          key[c] = k;
        }
        big_sort_desc<uint32_t, KB>(key, lane);
        // The 32-bit order is exact except where neighbours share a 22-bit
        // prefix but differ in value (exactly equal values are already in
        // column order: the key's low bits).  Typically no row has such a
        // pair — then the order is final; else the repair below.
        auto kcol = [&](uint32_t k) { return (1 << BIG_CB) - 1 - (int)(k & ((1u << BIG_CB) - 1)); };
        bool need = false;
#pragma unroll
        for (int c = 0; c + 1 < KB; c++)
          if (lane * KB + c + 1 < N && (key[c] >> BIG_CB) == (key[c + 1] >> BIG_CB))
            need = need || row[big_rpos(kcol(key[c]))] != row[big_rpos(kcol(key[c + 1]))];
        {
          const uint32_t nk = __shfl_down_sync(0xffffffffu, key[0], 1);
          if (lane < 31 && lane * KB + KB < N && (key[KB - 1] >> BIG_CB) == (nk >> BIG_CB))
            need = need || row[big_rpos(kcol(key[KB - 1]))] != row[big_rpos(kcol(nk))];
        }
        if (!__any_sync(0xffffffffu, need)) {
          unsigned long long *ov = sval + (size_t)i * N;
          uint16_t *oc = scol + (size_t)i * N;
#pragma unroll
          for (int c = 0; c < KB; c++) {
            const int pos = lane * KB + c;
            if (pos < N) {
              const int col = kcol(key[c]);
              ov[pos] = big_bits(row[big_rpos(col)]);  // exact value bits for the matching
              oc[pos] = (uint16_t)col;
            }
          }
          __syncwarp();  // rbuf is restaged for the warp's next row
          continue;
        }
        // pair-wide 64-bit keys (exponent | mantissa truncated by `shift` bits |
        // column) in sorted order; odd-even transposition repairs inversions
        // among equal 22-bit prefixes, then neighbours whose truncated keys
        // tie are put in exact (value desc, column asc) order from X
        unsigned long long ek[KB];
#pragma unroll
        for (int c = 0; c < KB; c++) {
          const int pos = lane * KB + c;
          const int col = (1 << BIG_CB) - 1 - (int)(key[c] & ((1u << BIG_CB) - 1));
          ek[c] = (pos < N) ? big_sort_key<T>(row[big_rpos(col)], col, emin, shift) : 0ull;
        }
        // `after(x, y)`: y must precede x — (value desc, column asc), exact:
        // equal truncated values are decided on X (keys' low bits only hold
        // the column, which ties exact values)
        auto after = [&](unsigned long long x, unsigned long long y) {
          if ((x >> BIG_CB) != (y >> BIG_CB)) return (x >> BIG_CB) < (y >> BIG_CB);
          if (shift > 0) {
            const T vx = row[big_rpos(big_key_col(x))], vy = row[big_rpos(big_key_col(y))];
            if (vx != vy) return vx < vy;
          }
          return (x & ((1ull << BIG_CB) - 1)) < (y & ((1ull << BIG_CB) - 1));  // lower column first
        };
        for (int pass = 0;; pass++) {
          bool sw = false;
#pragma unroll
          for (int c = (pass & 1); c + 1 < KB; c += 2)
            if (lane * KB + c + 1 < N && after(ek[c], ek[c + 1])) {
              const unsigned long long t = ek[c]; ek[c] = ek[c + 1]; ek[c + 1] = t;
              sw = true;
            }
          if (((KB - 1) & 1) == (pass & 1)) {  // lane boundary pair (KB*l + KB-1, KB*(l+1))
            const unsigned long long nv = __shfl_down_sync(0xffffffffu, ek[0], 1);
            const unsigned long long pv = __shfl_up_sync(0xffffffffu, ek[KB - 1], 1);
            const bool xl = lane < 31 && lane * KB + KB < N && after(ek[KB - 1], nv);
            const bool xr = lane > 0 && lane * KB < N && after(pv, ek[0]);
            if (xl) { ek[KB - 1] = nv; sw = true; }
            if (xr) { ek[0] = pv; sw = true; }
          }
          if ((!__any_sync(0xffffffffu, sw) && pass > 0) || pass > 64 * KB) break;  // (bounded: odd-even transposition sorts in n passes)
        }
        unsigned long long *ov = sval + (size_t)i * N;
        uint16_t *oc = scol + (size_t)i * N;
#pragma unroll
        for (int c = 0; c < KB; c++) {
          const int pos = lane * KB + c;
          if (pos < N) {
            const int col = big_key_col(ek[c]);
            ov[pos] = big_bits(row[big_rpos(col)]);  // exact value bits for the matching
            oc[pos] = (uint16_t)col;
          }
        }
        __syncwarp();  // rbuf is restaged for the warp's next row
      }
      __syncthreads();

      BIG_PHASE(4);
      // ---- 4b. greedy matching rounds, similarity.py:96-108, whole CTA.
      // Thread t owns rows t + 256 r (r < R); each active row's head is
      // its best untaken column, compared across rows on exact value bits
      // with ties to the lowest row (np.argmax's first occurrence).  A round:
      // per-warp best -> shared slots (value, row, column) -> one barrier ->
      // every thread picks the same winner, marks the column, and advances
      // its rows whose head column was taken.  The next three sorted entries
      // of every row are already in registers (loads issued rounds earlier),
      // so no HBM round trip sits on the per-round critical path.
      {
        uint32_t *taken = (uint32_t *)(smem_raw + L.taken);
        // per warp and round parity: {value bits, row << 32 | column} (one
        // 16-byte load per slot in the scan)
        ulonglong2 *gsl = (ulonglong2 *)(smem_raw + L.gslot);
        int32_t *mrow = (int32_t *)(smem_raw + L.mrow);
        unsigned long long *mval = (unsigned long long *)(smem_raw + L.mval);
        for (int w = tid; w < 64; w += NT) taken[w] = 0u;
        // rows per thread R = N-bound / 256 (1, 2, 4 for KB = 8, 16, 32) and
        // a register window of PF = 12 / R sorted entries per row (the same
        // 36 registers in every variant): the shorter rows of the smaller
        // classes get a deeper window, so fewer head advances ("deep skips"
        // past taken columns) wait on a dependent HBM load inside a round
        constexpr int R = (32 * KB) / BIG_THREADS < 1 ? 1 : (32 * KB) / BIG_THREADS;
#ifndef CFGSIM_BIG_PF
        constexpr int PF = 12 / R;
#else
        constexpr int PF = CFGSIM_BIG_PF;
#endif
        unsigned long long hv[R], qv[R][PF];
        int hc[R], qc[R][PF], ptr[R];
        uint32_t act = 0u;
#pragma unroll
        for (int r = 0; r < R; r++) {
          const int i = tid + BIG_THREADS * r;
          hv[r] = 0ull;
          hc[r] = 0;
          ptr[r] = 0;
#pragma unroll
          for (int f = 0; f < PF; f++) { qv[r][f] = 0ull; qc[r][f] = 0; }
          if (i < N) {
            act |= 1u << r;
            hv[r] = sval[(size_t)i * N];
            hc[r] = scol[(size_t)i * N];
#pragma unroll
            for (int f = 0; f < PF; f++)
              if (1 + f < N) {
                qv[r][f] = sval[(size_t)i * N + 1 + f];
                qc[r][f] = scol[(size_t)i * N + 1 + f];
              }
            if (KB <= 16) {
              for (int e = 1 + PF; e < 1 + PF + BIG_L2_AHEAD && e < N; e += 16) big_prefetch_l2(sval + (size_t)i * N + e);
              if (1 + PF < N) big_prefetch_l2(scol + (size_t)i * N + 1 + PF);
            }
          }
        }
        __syncthreads();
        if (prm.phase && tid == 0) atomicAdd(prm.phase + 7, (unsigned long long)N);
        unsigned adv_steps = 0, adv_deep = 0;
        int prev_col = 0;
        for (int round = 0; round < N; round++) {
          unsigned long long bv = 0ull;
          int brow = 0x7fffffff, bcl = 0;
#pragma unroll
          for (int r = 0; r < R; r++)
            if (((act >> r) & 1u) && (brow == 0x7fffffff || hv[r] > bv)) {
              bv = hv[r];
              brow = tid + BIG_THREADS * r;
              bcl = hc[r];
            }
          const bool has = brow != 0x7fffffff;
          const unsigned hi = (unsigned)(bv >> 32), lo = (unsigned)bv;
          const unsigned mhi = __reduce_max_sync(0xffffffffu, has ? hi : 0u);
          const unsigned mlo = __reduce_max_sync(0xffffffffu, (has && hi == mhi) ? lo : 0u);
          const bool cand = has && hi == mhi && lo == mlo;
          const int wrow = (int)__reduce_min_sync(0xffffffffu, cand ? (unsigned)brow : 0x7fffffffu);
          const int buf = round & 1;
          if (wrow != 0x7fffffff && brow == wrow) {  // the owner lane publishes value, row, column
            gsl[buf * BIG_WARPS + warp] = make_ulonglong2(bv, ((unsigned long long)wrow << 32) | (unsigned)bcl);
          } else if (wrow == 0x7fffffff && lane == 0) {
            gsl[buf * BIG_WARPS + warp] = make_ulonglong2(0ull, 0x7fffffffull << 32);
          }
          __syncthreads();
          unsigned long long gv = 0ull;
          int grow = 0x7fffffff, bcol = 0;
#pragma unroll
          for (int w = 0; w < BIG_WARPS; w++) {
            const ulonglong2 sl = gsl[buf * BIG_WARPS + w];
            const int rw = (int)(sl.y >> 32);
            if (rw == 0x7fffffff) continue;
            if (grow == 0x7fffffff || sl.x > gv || (sl.x == gv && rw < grow)) {
              gv = sl.x;
              grow = rw;
              bcol = (int)(unsigned)sl.y;
            }
          }
          // taken columns, two generations: round r reads T_r from buffer r & 1
          // (plus this round's column, in registers); thread 0 writes T_{r+1}
          // into the other buffer, whose last readers were in round r - 1
          const uint32_t *tk_cur = taken + (round & 1) * 32;
          if (tid == 0) {
            uint32_t *tk_nxt = taken + ((round + 1) & 1) * 32;
            if (round > 0) tk_nxt[prev_col >> 5] |= 1u << (prev_col & 31);
            tk_nxt[bcol >> 5] |= 1u << (bcol & 31);
          }
          prev_col = bcol;
          if ((grow & (BIG_THREADS - 1)) == tid) {
            act &= ~(1u << (grow / BIG_THREADS));
            mrow[grow] = bcol;
            mval[grow] = gv;
          }
          // advance rows whose head column was taken
#pragma unroll
          for (int r = 0; r < R; r++) {
            if (((act >> r) & 1u) && hc[r] == bcol) {
              const int i = tid + BIG_THREADS * r;
              int p = ptr[r];
              const int p0 = p;
              do {  // p + 1 < N: an active row always has an untaken column
                ++p;
                hv[r] = qv[r][0];
                hc[r] = qc[r][0];
#pragma unroll
                for (int f = 0; f + 1 < PF; f++) { qv[r][f] = qv[r][f + 1]; qc[r][f] = qc[r][f + 1]; }
                if (p + PF < N) {
                  qv[r][PF - 1] = sval[(size_t)i * N + p + PF];
                  qc[r][PF - 1] = scol[(size_t)i * N + p + PF];
                }
              } while (hc[r] == bcol || ((tk_cur[hc[r] >> 5] >> (hc[r] & 31)) & 1u));
              ptr[r] = p;
              // keep the row's coming entries in L2: later window refills
              // and skips past the window then wait on L2, not HBM (the
              // slabs of all resident CTAs do not stay in L2 on their own).
              // N <= 512 only: measured +6.7% on a C5 subset, -4% at
              // N <= 1024 (C4), where 4 rows per thread prefetch 4x the lines
              if (KB <= 16 && p + PF + BIG_L2_AHEAD < N) {
                big_prefetch_l2(sval + (size_t)i * N + p + PF + BIG_L2_AHEAD);
                big_prefetch_l2(scol + (size_t)i * N + p + PF + BIG_L2_AHEAD);
              }
              adv_steps += (unsigned)(p - p0);  // diagnostics (registers; one atomic per pair)
              adv_deep += (p - p0 > PF) ? 1u : 0u;
            }
          }
        }
        if (prm.phase) {  // advances, advances past the prefetched window
          atomicAdd(prm.phase + 5, (unsigned long long)adv_steps);
          atomicAdd(prm.phase + 6, (unsigned long long)adv_deep);
        }
        __syncthreads();
        if (tid == 0) {  // similarity.py:150: Python sum in row order
          double wsum = 0.0;
          for (int i = 0; i < N; i++) wsum += (sizeof(T) == 8) ? __longlong_as_double((long long)mval[i])
                                                               : (double)__uint_as_float((unsigned)mval[i]);
          if (out.d) out.d[slot] = isorank_distance_of(wsum, N);
          if (out.W) out.W[slot] = wsum;
          if (out.iters) out.iters[slot] = it_done;
          if (out.conv) out.conv[slot] = converged ? 1 : 0;
        }
        if (out.match)
          for (int i = tid; i < N; i += NT) out.match[i] = mrow[i];
      }
      BIG_PHASE(5);
      if (out.X)
        for (int e = tid; e < N * N; e += NT) out.X[e] = (double)X[e];
      __syncthreads();
    }
  }
}

// Per-(graph, N) sequences for the history mode of the large-N kernel: one
// CTA per combo (grid-stride), the side's operator exactly as the pair kernel
// builds it, kcap sweeps with the pair kernel's per-side arithmetic and
// thread mapping (bitwise the same u_m and Du_m), rows stored at pitch
// big_hpitch(N).  A size group of the triangle (rows a with n_a = N) shares
// the sequences of every partner graph, so each sequence is computed once
// per group instead of once per pair.
struct SeqBigCombos {
  int64_t n;
  int32_t N;
  const int32_t *g;     // combo -> graph (the size-sorted permutation from the group's first row)
  int64_t stride;       // combo -> offset of row 0: combo * stride
  double *hu;
  double *hd;           // (kcap + 1) per combo
};

template <int KB>
__global__ void __launch_bounds__(BIG_THREADS, 2)
    isorank_seqbig_kernel(DevCorpus C, SeqBigCombos cb, BigParams prm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const BigSmem L = big_smem_layout<double>(prm.nlim);
  double *red = (double *)(smem_raw + L.red);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = BIG_THREADS;
  const int N = cb.N, HP = big_hpitch(N);
  const double invN = 1.0 / (double)N;
  for (int64_t c = blockIdx.x; c < cb.n; c += gridDim.x) {
    BigSide S;
    big_side_init(S, C, cb.g[c], N, smem_raw, L, 0);
    double *ring = (double *)(smem_raw + L.ring[0]);
    double *tv = (double *)(smem_raw + L.t[0]);
    double *sbuf = (double *)(smem_raw + L.scr);
    double *U = cb.hu + c * cb.stride;
    double *D = cb.hd + c * (int64_t)(prm.kcap + 1);
    for (int q = tid; q < N; q += NT) {
      ring[q] = 1.0;
      U[q] = 1.0;
    }
    if (tid == 0) D[0] = 0.0;
    double zsum = S.zcount;
    __syncthreads();
    for (int k = 1; k <= prm.kcap; k++) {
      const int cur = (k - 1) & 1, nxt = k & 1;
      const int n0 = S.kind == 2 ? 0 : S.n;
      if (S.kind == 1) {
        for (int q = tid; q < S.n; q += NT) sbuf[q] = big_s_entry<double>(S, ring + cur * N, q);
        __syncthreads();
      }
      for (int q = tid; q < n0; q += NT)
        tv[q] = S.kind == 1 ? big_t_from_s<double>(S, sbuf, q) : big_t_entry<double>(S, ring + cur * N, q);
      __syncthreads();
      double part[2] = {0.0, 0.0};
      const double z = zsum * invN;
      for (int q = tid; q < N; q += NT) {
        const double un = big_u_entry<double>(S, tv, q, z);
        const double uo = ring[cur * N + q];
        ring[nxt * N + q] = un;
        U[(size_t)k * HP + q] = un;
        part[0] += fabs(un - uo);
        if (S.zf[q]) part[1] += un;
      }
#pragma unroll
      for (int v = 0; v < 2; v++) {
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) part[v] += __shfl_xor_sync(0xffffffffu, part[v], m);
      }
      double *rb = red + (k & 1) * BIG_WARPS * 4;
      if (lane == 0) {
        rb[warp * 4] = part[0];
        rb[warp * 4 + 1] = part[1];
      }
      __syncthreads();
      double tot[2] = {0.0, 0.0};
      for (int w = 0; w < BIG_WARPS; w++) {
        tot[0] += rb[w * 4];
        tot[1] += rb[w * 4 + 1];
      }
      zsum = tot[1];
      if (tid == 0) D[k] = tot[0];
    }
    __syncthreads();  // smem tables are rebuilt for the next combo
  }
}

}  // namespace cfgsim
