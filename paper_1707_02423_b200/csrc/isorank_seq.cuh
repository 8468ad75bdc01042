// Two-stage IsoRank for all-pairs / query batches of small graphs (N <= 64).
//
// In the closed form of isorank_lr.cuh,
//     X_K = sum_{m<K} c alpha^m u_m v_m^T + (alpha^K/N^2) u_K v_K^T,
//     u_m = (A'^T)^m 1,   v_m = (B'^T)^m 1,
// the sequence u_0, u_1, ... depends only on the graph and the common size N
// (A' = row-normalised interpolate_to(A, N), similarity.py:85-93 after
// matrix.py:74-106) — not on the partner.  A corpus of K graphs has K^2/2
// pairs but only ~K * (#sizes)/2 distinct (graph, N) "combos", so:
//
//  stage 1 (isorank_seq_kernel): per combo, build A' exactly as the pair
//    kernels do (build_side: bit-exact interpolation, numpy-order row sums)
//    and run the mat-vec recurrence for kcap sweeps, storing u_m and
//    Du_m = ||u_m - u_{m-1}||_1 in HBM.  The recurrence is the same
//    arithmetic as the per-pair low-rank kernel (lr_matvec_entry).
//  stage 2 (isorank_pair2_kernel): per pair, the stopping sweep K from the
//    bracket  (alpha^k/N) max(Du_k, Dv_k) <= delta_k <= (alpha^k/N)(Du_k + Dv_k)
//    (exact delta_k, an N^2 pass, only where the bracket straddles tol),
//    then X_K as a rank-K product accumulated in registers in the low-rank
//    kernel's order (m ascending), the greedy matching and d.
//
// Per pair this removes every sweep barrier and mat-vec: what remains is
// ~K N^2 FMAs, one sort per row and N greedy rounds.
#pragma once
#include "isorank_lr.cuh"
#include "isorank_big.cuh"

namespace cfgsim {

struct SeqParams {
  double alpha;
  double tol;
  double eps;       // relative margin of the delta bracket
  int32_t max_iter;
  int32_t kcap;     // sweeps stored per combo (the bracket stops by then)
  int32_t cap;      // operator list capacity (entries)
  int32_t nlim;
};

// Combo table: combo c is graph combo_g[c] at size combo_n[c]; its u_m live
// at useq[uoff[c] + m * combo_n[c] + t], Du_m at dseq[c * (kcap + 1) + m].
struct SeqCombos {
  int64_t n;
  const int64_t *list;  // NULL: combos 0..n-1, else the combo ids to build
  const int32_t *g;
  const int32_t *nn;
  const int64_t *uoff;
  int32_t *status;  // per combo: 0 ok, 1 list overflow (re-run with dense lists)
};

struct SeqSmem {
  size_t dense, idx, w, toff, z, u, lo, fr, zflag, red, misc, total;
};

template <typename T>
__host__ __device__ inline SeqSmem seq_smem_layout(int nlim, int cap) {
  SeqSmem s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o += (b + 15) & ~size_t(15);
    return at;
  };
  s.dense = take(sizeof(double) * (size_t)nlim * (nlim | 1));
  s.idx = take(sizeof(int32_t) * (size_t)cap);
  s.w = take(sizeof(T) * (size_t)cap);
  s.toff = take(sizeof(int32_t) * (nlim + 1));
  s.z = take(sizeof(int32_t) * (nlim + 1));
  s.u = take(sizeof(T) * 2 * nlim);
  s.lo = take(sizeof(int32_t) * (nlim + 1));
  s.fr = take(sizeof(double) * (nlim + 1));
  s.zflag = take(sizeof(uint8_t) * (nlim + 1));
  s.red = take(sizeof(double) * 32);
  s.misc = take(64);
  s.total = o;
  return s;
}

// Stage 1: one CTA per combo (grid-stride), KB = N/32 chunks for build_side.
template <typename T, int KB>
__global__ void __launch_bounds__(64 * KB) isorank_seq_kernel(DevCorpus C, SeqCombos cb, SeqParams prm, T *useq,
                                                              double *dseq) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const SeqSmem L = seq_smem_layout<T>(prm.nlim, prm.cap);
  double *dense = (double *)(smem_raw + L.dense);
  int32_t *idx = (int32_t *)(smem_raw + L.idx);
  T *w = (T *)(smem_raw + L.w);
  int32_t *toff = (int32_t *)(smem_raw + L.toff);
  int32_t *zl = (int32_t *)(smem_raw + L.z);
  T *u = (T *)(smem_raw + L.u);
  int32_t *lo_s = (int32_t *)(smem_raw + L.lo);
  double *fr_s = (double *)(smem_raw + L.fr);
  uint8_t *zflag = (uint8_t *)(smem_raw + L.zflag);
  double *red = (double *)(smem_raw + L.red);
  int32_t *misc = (int32_t *)(smem_raw + L.misc);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NW = blockDim.x >> 5;

  for (int64_t ci = blockIdx.x; ci < cb.n; ci += gridDim.x) {
    const int64_t c = cb.list ? cb.list[ci] : ci;
    const int g = cb.g[c], N = cb.nn[c];
    int32_t *nz = misc + 1;
    const bool ok = build_side<T, KB, 1, false>(C, g, N, N | 1, dense, lo_s, fr_s, zflag, zl, nz, toff, nullptr,
                                                idx, w, prm.cap, false, misc);
    if (!ok) {
      if (tid == 0) cb.status[c] = 1;
      __syncthreads();
      continue;
    }
    const int nzv = *nz;
    const T invN = (T)(1.0 / (double)N);
    T *U = useq + cb.uoff[c];
    double *D = dseq + c * (int64_t)(prm.kcap + 1);
    for (int t = tid; t < N; t += blockDim.x) {
      u[t] = (T)1;
      U[t] = (T)1;
    }
    if (tid == 0) D[0] = 0.0;
    __syncthreads();
    for (int m = 1; m <= prm.kcap; m++) {
      const T *uo = u + ((m - 1) & 1) * N;
      T *un = u + (m & 1) * N;
      double part = 0.0;
      for (int t = tid; t < N; t += blockDim.x) {
        const T v = lr_matvec_entry(toff, idx, w, zl, nzv, uo, t, invN);
        un[t] = v;
        U[(size_t)m * N + t] = v;
        part += fabs((double)v - (double)uo[t]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) red[(m & 1) * 16 + warp] = part;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
        for (int q = 0; q < NW; q++) s += red[(m & 1) * 16 + q];
        D[m] = s;
      }
    }
    if (tid == 0) cb.status[c] = 0;
    __syncthreads();
  }
}

// Stage 2 work: the all-pairs triangle in size-sorted order, restricted to
// rows of one N; combo of sorted position b for this N = cbase + b.
struct Pair2Params {
  double alpha;
  double tol;
  double eps;
  int32_t max_iter;
  int32_t kcap;
  int32_t N;
  int32_t ty, tx;   // thread grid of the AR x BC entry blocks
  int64_t cbase;    // combo index = cbase + sorted position
  const double *apow;  // alpha^m, m = 0..kcap, by sequential products (host)
};

// Shared memory of the stage-2 kernel: X (N x P) aliased with the
// double-buffered u/v staging, then the greedy scratch, the bracket flags.
constexpr int P2_KC = 16;   // sweeps per staged chunk
constexpr int P2_MW = 64;   // words of the ambiguous-sweep bitmask (kcap < 2048)

__host__ __device__ inline size_t p2_x_bytes(int N, int tsize) {
  const size_t xb = (size_t)tsize * N * (N | 1), sb = (size_t)tsize * 2 * P2_KC * 2 * N;
  return ((xb > sb ? xb : sb) + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t p2_smem_bytes(int N, int tsize) {
  return p2_x_bytes(N, tsize) + (((size_t)N * N + 4 * N + 64 + 15) & ~(size_t)15) + 2 * 32 * sizeof(double) +
         P2_MW * sizeof(uint32_t) + 64;
}

template <typename T, int KB, int AR, int BC, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
    isorank_pair2_kernel(const int32_t *n_nodes, PairWork work, PairOut out, Pair2Params prm, const T *useq,
                         const double *dseq, const int64_t *uoff, unsigned long long *counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = prm.N, P = N | 1;
  T *Xs = (T *)smem_raw;  // N x P (aliases the staging buffers)
  T *stg = (T *)smem_raw;
  uint8_t *scr = smem_raw + p2_x_bytes(N, sizeof(T));
  double *red = (double *)(scr + ((((size_t)N * N + 4 * N + 64) + 15) & ~(size_t)15));
  uint32_t *amb = (uint32_t *)(red + 2 * 32);
  int64_t *s_item = (int64_t *)(amb + P2_MW);
  int32_t *s_first = (int32_t *)(s_item + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  const int TY = prm.ty, TX = prm.tx;
  const bool owner = tid < TY * TX;
  const int ty = owner ? tid / TX : 0, tx = owner ? tid - (tid / TX) * TX : 0;
  const double invN = 1.0 / (double)N;
  const double inv_nn = 1.0 / (double)((long long)N * N);
  const double c = (1.0 - prm.alpha) * inv_nn;
  const int mmax = prm.max_iter < prm.kcap ? prm.max_iter : prm.kcap;

  for (;;) {
    if (tid == 0) {
      *s_item = (int64_t)atomicAdd(counter, 1ull);
      *s_first = 0x7fffffff;
    }
    for (int q = tid; q < P2_MW; q += NT) amb[q] = 0u;
    __syncthreads();
    const int64_t item = *s_item;
    if (item >= work.n_items) break;
    // triangle unit -> sorted rows a <= b; the alignment runs in the caller's
    // (lower graph index, higher graph index) direction
    const int64_t uu = work.u0 + item;
    int lo = 0, hi = work.K - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (work.row_start[mid] <= uu) lo = mid; else hi = mid - 1;
    }
    const int a = lo, b = a + (int)(uu - work.row_start[a]);
    int pa = a, pb = b;
    if (work.perm[pa] > work.perm[pb]) { const int t = pa; pa = pb; pb = t; }
    const int64_t slot = uu - work.out_base;
    const int64_t ca = prm.cbase + pa, cb = prm.cbase + pb;
    const T *UA = useq + uoff[ca];
    const T *UB = useq + uoff[cb];
    const double *DA = dseq + ca * (int64_t)(prm.kcap + 1);
    const double *DB = dseq + cb * (int64_t)(prm.kcap + 1);

    // ---- stopping sweep K (similarity.py:139-146): every sweep's bracket in
    // parallel (alpha^m from the host's table, the same sequential products),
    // then exact delta only for the ambiguous sweeps before the first
    // certain stop, in order
    for (int m = tid + 1; m <= mmax; m += NT) {
      const double ak = prm.apow[m];
      const double da = DA[m], db = DB[m];
      const double hiB = ak * invN * (da + db) * (1.0 + prm.eps);
      const double loB = ak * invN * fmax(da, db) * (1.0 - prm.eps);
      if (hiB < prm.tol) atomicMin(s_first, m);
      else if (loB < prm.tol) atomicOr(amb + (m >> 5), 1u << (m & 31));
    }
    __syncthreads();
    int K = mmax;
    bool conv = false;
    {
      const int first = *s_first;
      if (first != 0x7fffffff) { K = first; conv = true; }
      const int lim = first == 0x7fffffff ? mmax : first - 1;  // ambiguous sweeps that can still decide
      for (int wd = 0; wd <= (lim >> 5); wd++) {
        uint32_t bits = amb[wd];
        while (bits) {
          const int m = wd * 32 + __ffs(bits) - 1;
          bits &= bits - 1;
          if (m > lim) break;
          // exact delta_m = alpha^m/N^2 sum_ij |u_m[i] v_m[j] - u_{m-1}[i] v_{m-1}[j]|
          const T *un = UA + (size_t)m * N, *uo = UA + (size_t)(m - 1) * N;
          const T *vn = UB + (size_t)m * N, *vo = UB + (size_t)(m - 1) * N;
          double dl = 0.0;
          for (int e = tid; e < N * N; e += NT) {
            const int i = e / N, j = e - (e / N) * N;
            dl += fabs((double)fma(-uo[i], vo[j], un[i] * vn[j]));
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) dl += __shfl_xor_sync(0xffffffffu, dl, o);
          if (lane == 0) red[warp] = dl;
          __syncthreads();
          double S = 0.0;
          for (int q = 0; q < NW; q++) S += red[q];
          __syncthreads();  // red is rewritten by the next exact pass
          if (prm.apow[m] * inv_nn * S < prm.tol) {  // similarity.py:144
            K = m;
            conv = true;
            wd = P2_MW;
            break;
          }
        }
      }
    }

    // ---- X_K = sum_{m<K} (c alpha^m) u_m v_m^T + (alpha^K/N^2) u_K v_K^T, the
    // u/v rows staged through shared memory in chunks of P2_KC sweeps
    T Pacc[AR][BC];
#pragma unroll
    for (int x = 0; x < AR; x++)
#pragma unroll
      for (int y = 0; y < BC; y++) Pacc[x][y] = 0;
    const int nch = (K + 1 + P2_KC - 1) / P2_KC;  // rows m = 0..K
    auto stage = [&](int ch) {
      T *dst = stg + (ch & 1) * P2_KC * 2 * N;
      const int m0 = ch * P2_KC;
      const int rows = (K + 1 - m0) < P2_KC ? (K + 1 - m0) : P2_KC;
      for (int e = tid; e < rows * 2 * N; e += NT) {
        const int mm = e / (2 * N), r = e - mm * 2 * N;
        const T *src = (r < N ? UA + (size_t)(m0 + mm) * N + r : UB + (size_t)(m0 + mm) * N + (r - N));
        big_cp_async_zfill<sizeof(T)>(dst + e, src, true);
      }
      big_cp_async_commit();
    };
    stage(0);
    int ii[AR], jj[BC];
#pragma unroll
    for (int x = 0; x < AR; x++) { ii[x] = ty + TY * x; if (ii[x] >= N) ii[x] = N - 1; }
#pragma unroll
    for (int y = 0; y < BC; y++) { jj[y] = tx + TX * y; if (jj[y] >= N) jj[y] = N - 1; }
    T uK[AR], vK[BC];
    for (int ch = 0; ch < nch; ch++) {
      if (ch + 1 < nch) {
        stage(ch + 1);
        big_cp_async_wait_group<1>();
      } else {
        big_cp_async_wait_group<0>();
      }
      __syncthreads();
      const T *buf = stg + (ch & 1) * P2_KC * 2 * N;
      const int m0 = ch * P2_KC;
      const int rows = (K + 1 - m0) < P2_KC ? (K + 1 - m0) : P2_KC;
      if (owner) {
        for (int mm = 0; mm < rows; mm++) {
          const int m = m0 + mm;
          const T *um = buf + mm * 2 * N, *vm = um + N;
          if (m == K) {  // last term
#pragma unroll
            for (int x = 0; x < AR; x++) uK[x] = um[ii[x]];
#pragma unroll
            for (int y = 0; y < BC; y++) vK[y] = vm[jj[y]];
            break;
          }
          const T cak = (T)(c * prm.apow[m]);
          T vb[BC];
#pragma unroll
          for (int y = 0; y < BC; y++) vb[y] = vm[jj[y]];
#pragma unroll
          for (int x = 0; x < AR; x++) {
            const T cu = cak * um[ii[x]];
#pragma unroll
            for (int y = 0; y < BC; y++) Pacc[x][y] = fma(cu, vb[y], Pacc[x][y]);
          }
        }
      }
      __syncthreads();  // buffer (ch & 1) is re-staged by chunk ch + 2 / X overwrites it
    }
    if (owner) {
      const T sc = (T)(prm.apow[K] * inv_nn);
#pragma unroll
      for (int x = 0; x < AR; x++) {
        const int i = ty + TY * x;
        const T su = sc * uK[x];
#pragma unroll
        for (int y = 0; y < BC; y++) {
          const int j = tx + TX * y;
          if (i < N && j < N) Xs[i * P + j] = fma(su, vK[y], Pacc[x][y]);
        }
      }
    }
    __syncthreads();
    const double wsum = greedy_match<T, KB>(Xs, P, N, scr, lane, warp, NW, nullptr);
    if (tid == 0) {
      if (out.d) out.d[slot] = isorank_distance_of(wsum, N);
      if (out.W) out.W[slot] = wsum;
      if (out.iters) out.iters[slot] = K;
      if (out.conv) out.conv[slot] = conv ? 1 : 0;
    }
    __syncthreads();
  }
}

}  // namespace cfgsim
