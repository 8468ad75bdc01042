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
constexpr int BIG_TM = 128, BIG_TN = 64, BIG_KC = 8;  // GEMM tile and k-chunk
constexpr int BIG_CB = 10;                            // column bits of a sort key (N <= 1024)

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
};

// per-CTA global slab
struct BigSlab {
  size_t coef, uh, vh, x, ord, total;
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
  s.ord = take(sizeof(uint16_t) * (size_t)nlim * nlim);
  s.total = o;
  return s;
}

// dynamic shared memory: a persistent head + a union of the phase regions
struct BigSmem {
  // sweep region (per side s = 0 (A), 1 (B))
  size_t lo[2], fr[2], rinv[2], pst[2], zf[2], t[2], ring[2], scr;
  // gemm region
  size_t us, vs;
  // greedy region
  size_t hptr, hcol, hval, mrow;
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
  s.misc = take(128);
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
  s.us = take(sizeof(T) * BIG_KC * BIG_TM);
  s.vs = take(sizeof(T) * BIG_KC * BIG_TN);
  const size_t gemm_end = o;
  o = base;
  s.hptr = take(sizeof(uint16_t) * nlim);
  s.hcol = take(sizeof(uint16_t) * nlim);
  s.hval = take(sizeof(T) * nlim);
  s.mrow = take(sizeof(int32_t) * nlim);
  const size_t greedy_end = o;
  size_t e = sweep_end > gemm_end ? sweep_end : gemm_end;
  e = e > greedy_end ? e : greedy_end;
  s.total = e;
  return s;
}

// Decode work item -> (ga, gb, number of directions, first output slot).
__device__ __forceinline__ void decode_item(const PairWork &work, int64_t item, int &ga, int &gb, int &ndir,
                                            int64_t &slot0) {
  ndir = 1;
  if (work.mode == WORK_LIST) {
    ga = work.ia[item];
    gb = work.ib[item];
    slot0 = work.slot ? work.slot[item] : item;
    return;
  }
  const int64_t u = work.u0 + item;
  int lo = 0, hi = work.K - 1;
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
  T *X = (T *)(slab + G.x);
  uint16_t *ord = (uint16_t *)(slab + G.ord);
  double *red = (double *)(smem_raw + L.red);
  int64_t *s_item = (int64_t *)(smem_raw + L.misc);
  double *s_scr = (double *)(smem_raw + L.misc + 16);  // 2 doubles

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = BIG_THREADS;

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

      // ---- 1. operators
      BigSide SD[2];
#pragma unroll
      for (int s = 0; s < 2; s++) {
        const DevCorpus &Cs = s ? C2 : C1;
        const int g = s ? g2 : g1;
        BigSide &S = SD[s];
        S.n = Cs.n_nodes[g];
        S.N = N;
        S.kind = (S.n == N) ? 0 : (S.n == 1 ? 2 : 1);
        S.rp = Cs.rowptr + Cs.rp_off[g];
        S.cc = Cs.col + Cs.nz_off[g];
        S.rv = Cs.val + Cs.nz_off[g];
        S.cp = Cs.cscp + Cs.rp_off[g];
        S.cr = Cs.csc_row + Cs.nz_off[g];
        S.cv = Cs.csc_val + Cs.nz_off[g];
        S.lo = (int16_t *)(smem_raw + L.lo[s]);
        S.fr = (double *)(smem_raw + L.fr[s]);
        S.rinv = (double *)(smem_raw + L.rinv[s]);
        S.pst = (int16_t *)(smem_raw + L.pst[s]);
        S.zf = (uint8_t *)(smem_raw + L.zf[s]);
        big_build_side(S, (double *)(smem_raw + L.scr));
      }
      T *ring[2] = {(T *)(smem_raw + L.ring[0]), (T *)(smem_raw + L.ring[1])};
      T *tv[2] = {(T *)(smem_raw + L.t[0]), (T *)(smem_raw + L.t[1])};

      // ---- 2. sweeps
      for (int q = tid; q < N; q += NT) {
        ring[0][q] = (T)1;
        ring[1][q] = (T)1;
        Uh[q] = (T)1;
        Vh[q] = (T)1;
      }
      double zsum[2] = {SD[0].zcount, SD[1].zcount};
      const double invN = 1.0 / (double)N;
      const double inv_nn = 1.0 / (double)((long long)N * N);
      const double c = (1.0 - prm.alpha) * inv_nn;  // (1-alpha)*uniform, similarity.py:140
      double ak1 = 1.0;                             // alpha^(k-1)
      int it_done = prm.max_iter;
      bool converged = false;
      int k = 1;
      __syncthreads();
      for (;; k++) {
        const int cur = (k - 1) & 1, nxt = k & 1;  // ring slots of u_{k-1}, u_k
        // phase 1: t = A^T W^T D^-1 u_{k-1}
        {
          const int n0 = SD[0].kind == 2 ? 0 : SD[0].n;
          const int n1 = SD[1].kind == 2 ? 0 : SD[1].n;
          for (int q = tid; q < n0 + n1; q += NT) {
            if (q < n0)
              tv[0][q] = big_t_entry<T>(SD[0], ring[0] + cur * N, q);
            else
              tv[1][q - n0] = big_t_entry<T>(SD[1], ring[1] + cur * N, q - n0);
          }
        }
        __syncthreads();
        // phase 2: u_k = W t + zsum/N; partial sums of |u_k - u_{k-1}| and z^T u_k
        double part[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q = tid; q < 2 * N; q += NT) {
          const int s = q >= N, i = q - s * N;
          const T un = big_u_entry<T>(SD[s], tv[s], i, zsum[s] * invN);
          const T uo = ring[s][cur * N + i];
          ring[s][nxt * N + i] = un;
          if (k <= prm.kcap) (s ? Vh : Uh)[(size_t)k * N + i] = un;
          part[2 * s] += fabs((double)un - (double)uo);
          if (SD[s].zf[i]) part[2 * s + 1] += (double)un;
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
      const int K = k;  // x after K sweeps (similarity.py:139-148)
      if (K > prm.kcap) {  // cannot happen: the bracket stops by kcap
        if (tid == 0) {
          atomicExch(prm.status, 1);
          if (out.iters) out.iters[slot] = -2;
        }
        __syncthreads();
        continue;
      }
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

      // ---- 3. X = sum_m coef_m u_m v_m^T  (128 x 64 tiles, 8 x 4 per thread)
      {
        T *Us = (T *)(smem_raw + L.us);
        T *Vs = (T *)(smem_raw + L.vs);
        const int ty = tid >> 4, tx = tid & 15;
        for (int i0 = 0; i0 < N; i0 += BIG_TM)
          for (int j0 = 0; j0 < N; j0 += BIG_TN) {
            T acc[8][4];
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
              for (int b = 0; b < 4; b++) acc[a][b] = (T)0;
            for (int m0 = 0; m0 <= K; m0 += BIG_KC) {
              __syncthreads();
              for (int e = tid; e < BIG_KC * BIG_TM; e += NT) {
                const int mm = e / BIG_TM, i = e % BIG_TM, m = m0 + mm;
                Us[e] = (m <= K && i0 + i < N) ? coef[m] * Uh[(size_t)m * N + i0 + i] : (T)0;
              }
              for (int e = tid; e < BIG_KC * BIG_TN; e += NT) {
                const int mm = e / BIG_TN, j = e % BIG_TN, m = m0 + mm;
                Vs[e] = (m <= K && j0 + j < N) ? Vh[(size_t)m * N + j0 + j] : (T)0;
              }
              __syncthreads();
#pragma unroll
              for (int mm = 0; mm < BIG_KC; mm++) {
                T ua[8], vb[4];
#pragma unroll
                for (int a = 0; a < 8; a++) ua[a] = Us[mm * BIG_TM + ty + 16 * a];
#pragma unroll
                for (int b = 0; b < 4; b++) vb[b] = Vs[mm * BIG_TN + tx + 16 * b];
#pragma unroll
                for (int a = 0; a < 8; a++)
#pragma unroll
                  for (int b = 0; b < 4; b++) acc[a][b] = fma(ua[a], vb[b], acc[a][b]);
              }
            }
#pragma unroll
            for (int a = 0; a < 8; a++) {
              const int i = i0 + ty + 16 * a;
#pragma unroll
              for (int b = 0; b < 4; b++) {
                const int j = j0 + tx + 16 * b;
                if (i < N && j < N) X[(size_t)i * N + j] = acc[a][b];
              }
            }
          }
      }
      __syncthreads();

      // ---- 4a. row orders (value desc, column asc) as packed keys
      for (int i = warp; i < N; i += BIG_WARPS) {
        const T *row = X + (size_t)i * N;
        int emin = 0x7fffffff, emax = -1;
        for (int j = lane; j < N; j += 32) {
          const int e = (sizeof(T) == 8) ? (int)((__double_as_longlong((double)row[j]) >> 52) & 0x7ff)
                                         : (int)((__float_as_uint((float)row[j]) >> 23) & 0xff);
          emin = min(emin, e);
          emax = max(emax, e);
        }
        emin = __reduce_min_sync(0xffffffffu, emin);
        emax = __reduce_max_sync(0xffffffffu, emax);
        int shift = 0;  // low mantissa bits dropped so exponent|mantissa|column fits 64 bits
        if (sizeof(T) == 8) {
          const int eb = 32 - __clz(emax - emin);
          shift = eb + 52 + BIG_CB - 64;
          if (shift < 0) shift = 0;
        }
        unsigned long long key[KB];
#pragma unroll
        for (int cc = 0; cc < KB; cc++) {
          const int j = lane + 32 * cc;
          key[cc] = (j < N) ? big_sort_key<T>(row[j], j, emin, shift) : 0ull;  // padding sorts last
        }
        warp_sort_keys_desc<KB>(key, lane);
        uint16_t *o = ord + (size_t)i * N;
        bool tie = false;
#pragma unroll
        for (int cc = 0; cc < KB; cc++) {
          const int pos = lane + 32 * cc;  // sorted position of key[cc]
          const int col = (1 << BIG_CB) - 1 - (int)(key[cc] & ((1ull << BIG_CB) - 1));
          if (pos < N) o[pos] = (uint16_t)col;
          if (shift > 0) {
            // neighbour at pos + 1: lane + 1 of this chunk, or lane 0 of the next
            unsigned long long nk = __shfl_down_sync(0xffffffffu, key[cc], 1);
            const unsigned long long n0 = __shfl_sync(0xffffffffu, key[cc + 1 < KB ? cc + 1 : cc], 0);
            if (lane == 31) nk = n0;
            if (pos + 1 < N && (key[cc] >> BIG_CB) == (nk >> BIG_CB)) {
              // equal truncated value: misordered only if the exact values differ
              const int ncol = (1 << BIG_CB) - 1 - (int)(nk & ((1ull << BIG_CB) - 1));
              if (row[col] != row[ncol]) tie = true;
            }
          }
        }
        __syncwarp();
        if (__any_sync(0xffffffffu, tie) && lane == 0) {
          // insertion pass on exact (value desc, column asc); keys are already
          // ordered up to the dropped bits, so only near-tied runs move
          for (int p = 1; p < N; p++) {
            const int cp = o[p];
            const T vp = row[cp];
            int q = p - 1;
            while (q >= 0) {
              const int cq = o[q];
              const T vq = row[cq];
              if (vq > vp || (vq == vp && cq < cp)) break;
              o[q + 1] = (uint16_t)cq;
              q--;
            }
            o[q + 1] = (uint16_t)cp;
          }
        }
        __syncwarp();
      }
      __syncthreads();

      // ---- 4b. greedy matching rounds (warp 0), similarity.py:96-108
      {
        uint16_t *hptr = (uint16_t *)(smem_raw + L.hptr);
        uint16_t *hcol = (uint16_t *)(smem_raw + L.hcol);
        T *hval = (T *)(smem_raw + L.hval);
        int32_t *mrow = (int32_t *)(smem_raw + L.mrow);
        if (warp == 0) {
          uint32_t act = 0u;     // bit c: row lane + 32c active
          uint32_t taken = 0u;   // bit w of lane l: column 32 l + w taken (this lane's word)
#pragma unroll
          for (int cc = 0; cc < KB; cc++) {
            const int i = lane + 32 * cc;
            if (i < N) {
              act |= 1u << cc;
              const int c0 = ord[(size_t)i * N];
              hptr[i] = 0;
              hcol[i] = (uint16_t)c0;
              hval[i] = X[(size_t)i * N + c0];
            }
          }
          __syncwarp();
          for (int round = 0; round < N; round++) {
            T bv = (T)0;
            int brow = 0x7fffffff;
#pragma unroll
            for (int cc = 0; cc < KB; cc++) {
              if (act & (1u << cc)) {
                const T hv = hval[lane + 32 * cc];
                if (brow == 0x7fffffff || hv > bv) { bv = hv; brow = lane + 32 * cc; }
              }
            }
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
            const int bcol = hcol[brow];
            if (lane == 0) mrow[brow] = bcol;
            if ((brow & 31) == lane) act &= ~(1u << (brow >> 5));
            if ((bcol >> 5) == lane) taken |= 1u << (bcol & 31);
            __syncwarp();
            // advance the rows whose head column was just taken
#pragma unroll
            for (int cc = 0; cc < KB; cc++) {
              const int i = lane + 32 * cc;
              const bool need = (act & (1u << cc)) && hcol[i] == bcol;
              if (__any_sync(0xffffffffu, need)) {
                int p = need ? hptr[i] : 0, col = 0;
                bool more = need;
                while (__any_sync(0xffffffffu, more)) {
                  if (more) {
                    ++p;
                    col = ord[(size_t)i * N + p];
                  }
                  const uint32_t word = __shfl_sync(0xffffffffu, taken, (col >> 5) & 31);
                  if (more && !((word >> (col & 31)) & 1u)) more = false;
                }
                if (need) {
                  hptr[i] = (uint16_t)p;
                  hcol[i] = (uint16_t)col;
                  hval[i] = X[(size_t)i * N + col];
                }
              }
            }
            __syncwarp();
          }
          if (lane == 0) {  // similarity.py:150: Python sum in row order
            double wsum = 0.0;
            for (int i = 0; i < N; i++) wsum += (double)X[(size_t)i * N + mrow[i]];
            s_scr[0] = wsum;
            if (out.d) out.d[slot] = isorank_distance_of(wsum, N);
            if (out.W) out.W[slot] = wsum;
            if (out.iters) out.iters[slot] = it_done;
            if (out.conv) out.conv[slot] = converged ? 1 : 0;
          }
          if (out.match)
            for (int i = lane; i < N; i += 32) out.match[i] = mrow[i];
        }
      }
      if (out.X)
        for (int e = tid; e < N * N; e += NT) out.X[e] = (double)X[e];
      __syncthreads();
    }
  }
}

}  // namespace cfgsim
