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
//    then X_K as a rank-K product on the fp64 tensor cores (mma.m8n8k4: the
//    low-rank kernel's m-ascending fma chain, bitwise), the row orders, the
//    greedy matching (a consumer warp overlapping the next pair) and d.
//
// Per pair this removes every sweep barrier and mat-vec: what remains is
// ~K N^2 mma work, one sort per row and N greedy rounds.
#pragma once
#ifdef CFGSIM_DEBUG_SEQ4
#include <cstdio>
#endif
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

// Combo table: combo c is graph combo_g[c] at size N = combo_n[c]; its u_m
// live at useq[uoff[c] + m * seq_pitch<T>(N) + t] (16-byte aligned rows), Du_m
// at dseq[c * (kcap + 1) + m].
struct SeqCombos {
  int64_t n;
  int64_t id0;          // combos id0 .. id0 + n - 1 (when list == NULL)
  const int64_t *list;  // else the combo ids to build
  int32_t redo;         // 1: only combos whose status is 1 (dense-bound list re-run)
  const int32_t *g;
  const int32_t *nn;
  const int64_t *uoff;
  int32_t *status;  // per combo: 0 ok, 1 list overflow (re-run with dense lists)
};

// history row pitch: a multiple of 16 bytes
template <typename T>
__host__ __device__ inline int seq_pitch(int N) {
  constexpr int e = 16 / (int)sizeof(T);
  return (N + e - 1) / e * e;
}

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
    const int64_t c = cb.list ? cb.list[ci] : cb.id0 + ci;
    if (cb.redo && cb.status[c] == 0) continue;  // (uniform per CTA)
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
    const int NPt = seq_pitch<T>(N);  // 16-byte aligned rows for the stage-2 copies
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
        U[(size_t)m * NPt + t] = v;
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

// Stage 1, four combos per CTA: the CTA builds the four operators one after
// the other (build_side needs the whole CTA and the dense scratch), then each
// warp runs one combo's recurrence warp-synchronously (no CTA barrier per
// sweep).  Same arithmetic as isorank_seq_kernel (lr_matvec_entry, same
// lists), so the u histories are bitwise identical.  Combos whose lists
// overflow are flagged for the one-per-CTA kernel's dense re-run.
constexpr int SEQ4 = 8;  // combos (= warps) per CTA

struct Seq4Smem {
  size_t dense, idx, w, toff, z, nz, u, lo, fr, zflag, misc, total;
};

template <typename T>
__host__ __device__ inline Seq4Smem seq4_smem_layout(int nlim, int cap) {
  Seq4Smem s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o += (b + 15) & ~size_t(15);
    return at;
  };
  s.dense = take(sizeof(double) * (size_t)nlim * (nlim | 1));
  s.idx = take(sizeof(int32_t) * (size_t)cap * SEQ4);
  s.w = take(sizeof(T) * (size_t)cap * SEQ4);
  s.toff = take(sizeof(int32_t) * (nlim + 1) * SEQ4);
  s.z = take(sizeof(int32_t) * (nlim + 1) * SEQ4);
  s.nz = take(sizeof(int32_t) * 4 * SEQ4);
  s.u = take(sizeof(T) * 2 * nlim * SEQ4);
  s.lo = take(sizeof(int32_t) * (nlim + 1));
  s.fr = take(sizeof(double) * (nlim + 1));
  s.zflag = take(sizeof(uint8_t) * (nlim + 1));
  s.misc = take(64);
  s.total = o;
  return s;
}

template <typename T, int KB>
__global__ void __launch_bounds__(32 * SEQ4) isorank_seq4_kernel(DevCorpus C, SeqCombos cb, SeqParams prm, T *useq,
                                                                double *dseq) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Seq4Smem L = seq4_smem_layout<T>(prm.nlim, prm.cap);
  double *dense = (double *)(smem_raw + L.dense);
  int32_t *lo_s = (int32_t *)(smem_raw + L.lo);
  double *fr_s = (double *)(smem_raw + L.fr);
  uint8_t *zflag = (uint8_t *)(smem_raw + L.zflag);
  int32_t *misc = (int32_t *)(smem_raw + L.misc);
  int32_t *nzs = (int32_t *)(smem_raw + L.nz);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nl = prm.nlim;
  for (int64_t g0 = (int64_t)blockIdx.x * SEQ4; g0 < cb.n; g0 += (int64_t)gridDim.x * SEQ4) {
    // ---- build up to four operators (whole CTA), lists in slot s
    for (int s = 0; s < SEQ4 && g0 + s < cb.n; s++) {
      const int64_t c = cb.id0 + g0 + s;
      int32_t *idx = (int32_t *)(smem_raw + L.idx) + (size_t)s * prm.cap;
      T *w = (T *)(smem_raw + L.w) + (size_t)s * prm.cap;
      int32_t *toff = (int32_t *)(smem_raw + L.toff) + s * (nl + 1);
      int32_t *zl = (int32_t *)(smem_raw + L.z) + s * (nl + 1);
      const bool ok = build_side<T, KB, 1, false>(C, cb.g[c], cb.nn[c], cb.nn[c] | 1, dense, lo_s, fr_s, zflag, zl,
                                                  nzs + 4 * s, toff, nullptr, idx, w, prm.cap, false, misc);
      if (tid == 0) {
        nzs[4 * s + 1] = ok ? 1 : 0;
        cb.status[c] = ok ? 0 : 1;
      }
      __syncthreads();
    }
    // ---- warp s: recurrence of combo g0 + s
    if (g0 + warp < cb.n && nzs[4 * warp + 1]) {
      const int64_t c = cb.id0 + g0 + warp;
      const int N = cb.nn[c];
      const int32_t *idx = (const int32_t *)(smem_raw + L.idx) + (size_t)warp * prm.cap;
      const T *w = (const T *)(smem_raw + L.w) + (size_t)warp * prm.cap;
      const int32_t *toff = (const int32_t *)(smem_raw + L.toff) + warp * (nl + 1);
      const int32_t *zl = (const int32_t *)(smem_raw + L.z) + warp * (nl + 1);
      const int nzv = nzs[4 * warp];
#ifdef CFGSIM_DEBUG_SEQ4
      if (lane == 0) {
        const int ntot = toff[N];
        bool bad = N > nl || N < 1 || ntot > prm.cap || ntot < 0 || nzv < 0 || nzv > N;
        for (int t = 0; t < N && !bad; t++) bad = toff[t + 1] < toff[t];
        for (int e = 0; e < ntot && e < prm.cap && !bad; e++) bad = idx[e] < 0 || idx[e] >= N;
        if (bad)
          printf("seq4 bad list: block %d warp %d combo %lld g %d N %d n %d toff[N] %d cap %d nzv %d ok %d\n",
                 blockIdx.x, warp, (long long)c, cb.g[c], N, C.n_nodes[cb.g[c]], ntot, prm.cap, nzv, nzs[4 * warp + 1]);
      }
#endif
      T *u = (T *)(smem_raw + L.u) + (size_t)warp * 2 * nl;
      const T invN = (T)(1.0 / (double)N);
      const int NPt = seq_pitch<T>(N);
      T *U = useq + cb.uoff[c];
      double *D = dseq + c * (int64_t)(prm.kcap + 1);
      for (int t = lane; t < N; t += 32) {
        u[t] = (T)1;
        U[t] = (T)1;
      }
      if (lane == 0) D[0] = 0.0;
      __syncwarp();
      for (int m = 1; m <= prm.kcap; m++) {
        const T *uo = u + ((m - 1) & 1) * nl;
        T *un = u + (m & 1) * nl;
        // lr_matvec_entry with the uniform-row term hoisted (computed once per
        // lane, same operation order) and the lane's two outputs interleaved
        T z0 = 0, z1 = 0;
        {
          int e = 0;
          for (; e + 1 < nzv; e += 2) {
            z0 += uo[zl[e]];
            z1 += uo[zl[e + 1]];
          }
          if (e < nzv) z0 += uo[zl[e]];
        }
        const T zt = (z0 + z1) * invN;
        const int t0 = lane, t1 = lane + 32;
        T a0 = zt, a1 = 0, b0 = zt, b1 = 0;
        {
          // only live rows read their list offsets: slots past N hold whatever
          // an earlier kernel left in shared memory (e.g. the stage-2 kernel's
          // 0x7fffffff sentinels), and e + 1 < e1 must never see them
          int e = t0 < N ? toff[t0] : 0, e1 = t0 < N ? toff[t0 + 1] : 0;
          int f = t1 < N ? toff[t1] : 0, f1 = t1 < N ? toff[t1 + 1] : 0;
          while (e + 1 < e1 || f + 1 < f1) {
            if (e + 1 < e1) {
              a0 = fma(w[e], uo[idx[e]], a0);
              a1 = fma(w[e + 1], uo[idx[e + 1]], a1);
              e += 2;
            }
            if (f + 1 < f1) {
              b0 = fma(w[f], uo[idx[f]], b0);
              b1 = fma(w[f + 1], uo[idx[f + 1]], b1);
              f += 2;
            }
          }
          if (e < e1) a0 = fma(w[e], uo[idx[e]], a0);
          if (f < f1) b0 = fma(w[f], uo[idx[f]], b0);
        }
        double part = 0.0;
        if (t0 < N) {
          const T v = a0 + a1;
          un[t0] = v;
          U[(size_t)m * NPt + t0] = v;
          part += fabs((double)v - (double)uo[t0]);
        }
        if (t1 < N) {
          const T v = b0 + b1;
          un[t1] = v;
          U[(size_t)m * NPt + t1] = v;
          part += fabs((double)v - (double)uo[t1]);
        }
        // (fixed order; may differ from the CTA kernel's D in the last bits —
        // D only feeds the bracket, whose 1e-6 margin makes K independent of it)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) D[m] = part;
        __syncwarp();
      }
    }
    __syncthreads();  // lists / rings are rebuilt for the next group
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
  int64_t cbase;    // combo index = cbase + sorted position (triangle; rect: query side)
  int64_t cbase2;   // rect mode: combo index of the corpus side = cbase2 + sorted position
  const double *apow;  // alpha^m, m = 0..kcap, by sequential products (host)
  unsigned long long *phase;  // optional (CFGSIM_PHASES=1): cycles per phase, summed over CTAs
};

// per-phase cycle accounting of the stage-2 kernel (debug; phase == nullptr
// in production): slot k accumulates the cycles from mark k to the next mark
// of the same role (producer warp 0 lane 0: slots 0-4; consumer lane 0: 8-9)
#define P2_PHASE(k)                                                     \
  do {                                                                  \
    if (prm.phase && (tid == 0 || tid == NP)) {                         \
      const unsigned long long now_ = clock64();                        \
      if (ph_last >= 0) atomicAdd(prm.phase + ph_last, now_ - ph_t);    \
      ph_t = now_;                                                      \
      ph_last = (k);                                                    \
    }                                                                   \
  } while (0)

// Stage-2 kernel, warp-specialised: warps 0..PW-1 ("producers") compute pair
// p's stopping sweep, X_K and row orders into one of two shared-memory
// buffers while warp PW ("consumer") runs the greedy rounds of pair p-1 from
// the other buffer.  Hand-off through named barriers (full / empty per
// buffer, bar.sync / bar.arrive), so the sequential rounds overlap the GEMM
// and sorts of the next pair.
constexpr int P2_KC = 8;    // sweeps per staged chunk
constexpr int P2_NS = 3;    // staging ring depth (chunks in flight while one is consumed)
constexpr int P2_KMAX = 512;  // kcap bound of the two-stage path (host checks)

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

struct P2Meta {
  int64_t slot;
  int32_t K, conv, valid, keys, emin, pad;
};

struct P2Smem {
  size_t x[2], ord[2], meta, red, amb, item, first, mrow, tab, total;
};

// staged history row pitch (elements; holds u_m and v_m side by side, >= 2
// NPt) such that the mma fragment loads (lane = 4 lr + lk reads row lk,
// column lr) are conflict-free: fp64 — a 64-bit request is served per
// half-warp, and 2 pitch mod 32 banks must be 8 or 24 so that the four rows
// lk land in disjoint bank octets (pitch == 4 mod 16; pitch == 8 mod 16 put
// rows 0 and 2 on the same banks: 2-way conflicts, ncu-measured);  fp32 —
// rows at pitch == 8 mod 16 floats start on bank octets 0/8/16/24.
__host__ __device__ inline int p2_stage_pitch(int npt, int tsize) {
  return tsize == 8 ? ((2 * npt + 11) / 16) * 16 + 4 : ((2 * npt + 7) / 16) * 16 + 8;
}

// row-order pitch (bytes): rows start 4-byte aligned so the orders are
// written as packed 32-bit words
__host__ __device__ inline int p2_ord_pitch(int N) { return (N + 3) & ~3; }

__host__ __device__ inline P2Smem p2_smem_layout(int N, int tsize, int kcap) {
  P2Smem s;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o += (b + 15) & ~size_t(15);
    return at;
  };
  const int npt = (N + 3) & ~3;
  const int spd = p2_stage_pitch(npt, 8) > p2_stage_pitch(npt, 4) ? p2_stage_pitch(npt, 8) : p2_stage_pitch(npt, 4);
  size_t xb = (size_t)tsize * N * (N | 1), sb = (size_t)8 * P2_NS * P2_KC * spd;
  const size_t kb = 8 * (size_t)N * (N <= 32 ? 33 : 65);  // key rows (pitch 32 KB + 1)
  if (kb > xb) xb = kb;
  for (int q = 0; q < 2; q++) {
    s.x[q] = take(xb > sb ? xb : sb);  // X_K (aliases the u/v staging while it is built)
    s.ord[q] = take((size_t)N * p2_ord_pitch(N));  // row orders (columns, value desc / column asc)
  }
  s.meta = take(2 * sizeof(P2Meta));
  s.red = take(8 * sizeof(double));  // one partial per producer warp
  s.amb = take(((kcap >> 5) + 1) * sizeof(uint32_t));
  s.item = take(sizeof(int64_t));
  s.first = take(sizeof(int32_t) * 4);  // first stop, emin, emax
  s.mrow = take(sizeof(int32_t) * 128);  // the consumer's winners: column (value path) / key hi, lo
  s.tab = take(sizeof(double) * (kcap + 2));  // alpha^m
  s.total = o;
  return s;
}
// (every region sized by N and kcap: 76.6 KB at N = 64, kcap = 137, so three
// CTAs share an SM at every N <= 64)
__host__ __device__ inline size_t p2_smem_bytes(int N, int tsize, int kcap) {
  return p2_smem_layout(N, tsize, kcap).total;
}

// One row of X (pitch P) into ord[0..N): (value desc, column asc), the order
// of np.argmax's first occurrence in similarity.py:103.  Exact: keys are
// (exponent rebased on the row | mantissa | inverted column) when the row's
// exponent span fits, else a (value, column) sort.  One warp.
template <typename T, int KB>
__device__ __forceinline__ void p2_sort_row(const T *row, int N, uint8_t *ord, int lane) {
  constexpr int CB = (32 * KB <= 64) ? 6 : 7;
  constexpr int EB = (sizeof(T) == 8) ? 12 - CB : 8;
  T v[KB];
  int emin = 0x7fffffff, emax = -1;
#pragma unroll
  for (int cc = 0; cc < KB; cc++) {
    const int j = lane + 32 * cc;
    v[cc] = (j < N) ? row[j] : (T)0;
    if (j < N) {
      const int e = big_exponent(v[cc]);
      emin = min(emin, e);
      emax = max(emax, e);
    }
  }
  emin = __reduce_min_sync(0xffffffffu, emin);
  emax = __reduce_max_sync(0xffffffffu, emax);
  if (emin > 0 && emax - emin < (1 << EB)) {
    unsigned long long key[KB];
#pragma unroll
    for (int cc = 0; cc < KB; cc++) {
      const int j = lane + 32 * cc;
      unsigned long long k = 0ull;  // padding sorts last (real column fields are >= 1)
      if (j < N) {
        if (sizeof(T) == 8) {
          const unsigned long long b = (unsigned long long)__double_as_longlong((double)v[cc]);
          const unsigned long long e = ((b >> 52) & 0x7ff) - (unsigned long long)emin;
          k = (e << (52 + CB)) | ((b & ((1ull << 52) - 1)) << CB) | (unsigned long long)((1 << CB) - 1 - j);
        } else {
          const unsigned int b = __float_as_uint((float)v[cc]);
          const unsigned long long e = ((b >> 23) & 0xff) - (unsigned)emin;
          k = (e << (23 + CB)) | ((unsigned long long)(b & 0x7fffff) << CB) | (unsigned long long)((1 << CB) - 1 - j);
        }
      }
      key[cc] = k;
    }
    warp_sort_keys_desc<KB>(key, lane);
#pragma unroll
    for (int cc = 0; cc < KB; cc++) {
      const int pos = lane + 32 * cc;
      if (pos < N) ord[pos] = (uint8_t)((1 << CB) - 1 - (int)(key[cc] & ((1ull << CB) - 1)));
    }
  } else {
    int cidx[KB];
#pragma unroll
    for (int cc = 0; cc < KB; cc++) {
      const int j = lane + 32 * cc;
      cidx[cc] = j;
      if (j >= N) v[cc] = (T)-1;
    }
    warp_sort_desc<T, KB>(v, cidx, lane);
#pragma unroll
    for (int cc = 0; cc < KB; cc++) {
      const int pos = lane + 32 * cc;
      if (pos < N) ord[pos] = (uint8_t)cidx[cc];
    }
  }
}

// Greedy rounds (similarity.py:96-108) on sorted rows, one warp: each round
// takes the best current head over active rows (ties -> lowest row) and
// advances the rows whose head column was taken.  Returns W (:150) on lane 0
// (row-order sum), mrow[i] = matched column.
template <typename T, int KB>
__device__ __forceinline__ double p2_rounds(const T *Xs, int P, int N, const uint8_t *ord, int32_t *mrow, int lane) {
  const int OP = p2_ord_pitch(N);
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
    ccol[cc] = act[cc] ? (int)ord[i * OP] : 0;
    cur[cc] = act[cc] ? Xs[i * P + ccol[cc]] : (T)-3;
  }
  for (int round = 0; round < N; round++) {
    T bv = (T)0;
    int brow = 0x7fffffff;
#pragma unroll
    for (int cc = 0; cc < KB; cc++)
      if (act[cc] && (brow == 0x7fffffff || cur[cc] > bv)) { bv = cur[cc]; brow = lane + 32 * cc; }
    const unsigned long long b = (brow == 0x7fffffff) ? 0ull : big_bits(bv);  // X > 0: bits order values
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    brow = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)brow : 0x7fffffffu);
    int mycol = 0;
#pragma unroll
    for (int cc = 0; cc < KB; cc++)
      if (cc == (brow >> 5)) mycol = ccol[cc];
    const int bcol = __shfl_sync(0xffffffffu, mycol, brow & 31);
    if (lane == 0) mrow[brow] = bcol;
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
          col = ord[i * OP + p];
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
  double wsum = 0.0;
  if (lane == 0)
    for (int i = 0; i < N; i++) wsum += (double)Xs[i * P + mrow[i]];
  return wsum;
}

// ---- exact packed keys: (value bits | 6-bit column field), comparable across
// rows.  fp64: (exponent - emin_pair) in 6 bits | 52-bit mantissa; needs the
// pair's exponent span < 64 (else the value-sort path is used).  fp32: the
// 31 value bits.  X > 0 (teleport floor), so bit order is value order.
template <typename T>
__device__ __forceinline__ unsigned long long p2_key(T v, int col, int emin) {
  if (sizeof(T) == 8) {
    const unsigned long long b = (unsigned long long)__double_as_longlong((double)v);
    return ((((b >> 52) & 0x7ff) - (unsigned long long)emin) << 58) | ((b & ((1ull << 52) - 1)) << 6) |
           (unsigned long long)(63 - col);
  } else {
    return ((unsigned long long)__float_as_uint((float)v) << 6) | (unsigned long long)(63 - col);
  }
}
// X is stored as packed keys when they are exact: always for fp32 (the float
// bits themselves), for fp64 when the pair's exponent span fits the 6-bit
// field; otherwise as values (p2_sort_row's value path)
template <typename T>
__device__ __forceinline__ bool p2_use_keys(int emin, int emax) {
  return sizeof(T) == 4 || (emax - emin < 64);
}
template <typename T>
__device__ __forceinline__ double p2_key_value(unsigned long long k, int emin) {
  if (sizeof(T) == 8)
    return __longlong_as_double((long long)((((k >> 58) + (unsigned long long)emin) << 52) | ((k >> 6) & ((1ull << 52) - 1))));
  return (double)__uint_as_float((unsigned)(k >> 6));
}

// Bitonic sort (descending) of n = 32 KB 32-bit keys held by one thread.
template <int KB>
__device__ __forceinline__ void p2_sort_u32(uint32_t (&v)[32 * KB]) {
  constexpr int n = 32 * KB;
#pragma unroll
  for (int k = 2; k <= n; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < n; i++) {
        const int l = i ^ j;
        if (l > i) {
          const uint32_t a = v[i], b = v[l];
          const uint32_t hi = max(a, b), lo = min(a, b);
          if ((i & k) == 0) { v[i] = hi; v[l] = lo; } else { v[i] = lo; v[l] = hi; }
        }
      }
}

// One row's order by one thread: 32-bit keys (top 26 value bits | column
// field) sorted in registers; adjacent entries whose 26-bit prefixes tie but
// whose exact keys differ are re-ordered by an insertion pass on the exact
// 64-bit keys (rare: near-ties within ~1e-6 relative).
template <typename T, int KB>
__device__ __forceinline__ void p2_row_order(const unsigned long long *Krow, int N, uint8_t *ord) {
  constexpr int VB = sizeof(T) == 8 ? 58 : 31;  // value bits above the column field
  uint32_t v[32 * KB];
#pragma unroll
  for (int q = 0; q < 32 * KB; q++)
    v[q] = (q < N) ? (uint32_t)((((Krow[q] >> 6) >> (VB - 26)) << 6) | (Krow[q] & 63ull)) : 0u;  // padding last
  p2_sort_u32<KB>(v);
  // orders as packed 32-bit words (ord is 4-byte aligned, pitch p2_ord_pitch)
#pragma unroll
  for (int w = 0; w < 8 * KB; w++)
    if (4 * w < N)
      reinterpret_cast<uint32_t *>(ord)[w] = (63u - (v[4 * w] & 63u)) | ((63u - (v[4 * w + 1] & 63u)) << 8) |
                                              ((63u - (v[4 * w + 2] & 63u)) << 16) | ((63u - (v[4 * w + 3] & 63u)) << 24);
  // neighbours with equal 26-bit prefixes are looked up exactly (no key loads
  // unless some prefix ties)
  uint32_t tie = 0u;
#pragma unroll
  for (int q = 0; q + 1 < 32 * KB; q++)
    if (q + 1 < N && (v[q] >> 6) == (v[q + 1] >> 6)) tie |= 1u << (q & 31);
  bool coll = false;
  if (tie) {
#pragma unroll
    for (int q = 0; q + 1 < 32 * KB; q++)
      if (((tie >> (q & 31)) & 1u) && (Krow[63 - (v[q] & 63u)] >> 6) != (Krow[63 - (v[q + 1] & 63u)] >> 6))
        coll = true;
  }
  if (coll) {
    for (int p = 1; p < N; p++) {
      const uint8_t cp = ord[p];
      const unsigned long long kp = Krow[cp];
      int q = p - 1;
      while (q >= 0 && Krow[ord[q]] < kp) {  // exact key order: value desc, column asc
        ord[q + 1] = ord[q];
        q--;
      }
      ord[q + 1] = cp;
    }
  }
}

// Same order for 32 < N <= 64 with two threads per row (adjacent lanes: half 0
// sorts positions 0..31 descending, half 1 positions 32..63 ascending; a
// shuffle exchange makes both halves bitonic, an in-register merge finishes).
template <typename T>
__device__ __forceinline__ void p2_row_order_pair(const unsigned long long *Krow, int N, uint8_t *ord, int half,
                                                  bool act) {
  constexpr int VB = sizeof(T) == 8 ? 58 : 31;
  uint32_t v[32];
  // half 1 sorts the complemented keys descending, i.e. its keys ascending:
  // one compile-time network for both halves (no per-exchange direction select)
  const uint32_t flip = half ? 0xffffffffu : 0u;
#pragma unroll
  for (int q = 0; q < 32; q++) {
    const int j = half * 32 + q;
    v[q] = ((act && j < N) ? (uint32_t)((((Krow[j] >> 6) >> (VB - 26)) << 6) | (Krow[j] & 63ull)) : 0u) ^ flip;
  }
  // sort half 0 descending, half 1 ascending (padding 0 ends up last overall)
  p2_sort_u32<1>(v);
#pragma unroll
  for (int q = 0; q < 32; q++) v[q] ^= flip;
#pragma unroll
  for (int q = 0; q < 32; q++) {  // half 0 keeps the larger 32, half 1 the smaller
    const uint32_t o = __shfl_xor_sync(0xffffffffu, v[q], 1);
    v[q] = half == 0 ? max(v[q], o) : min(v[q], o);
  }
#pragma unroll
  for (int j = 16; j > 0; j >>= 1)
#pragma unroll
    for (int i = 0; i < 32; i++) {
      const int l = i ^ j;
      if (l > i) {
        const uint32_t a = v[i], b = v[l];
        v[i] = max(a, b);
        v[l] = min(a, b);
      }
    }
  // orders as packed 32-bit words (rows 4-byte aligned at pitch
  // p2_ord_pitch(N) >= N: a word starting below N stays inside the row)
#pragma unroll
  for (int w = 0; w < 8; w++)
    if (act && half * 32 + 4 * w < N)
      reinterpret_cast<uint32_t *>(ord + half * 32)[w] =
          (63u - (v[4 * w] & 63u)) | ((63u - (v[4 * w + 1] & 63u)) << 8) | ((63u - (v[4 * w + 2] & 63u)) << 16) |
          ((63u - (v[4 * w + 3] & 63u)) << 24);
  // neighbours with equal 26-bit prefixes are looked up exactly (no key loads
  // unless some prefix ties)
  const uint32_t first1 = __shfl_down_sync(0xffffffffu, v[0], 1);  // half 1's first, seen by half 0
  uint32_t tie = 0u;
#pragma unroll
  for (int q = 0; q < 32; q++) {
    const uint32_t nx = q + 1 < 32 ? v[q + 1] : first1;
    const bool in = q + 1 < 32 ? half * 32 + q + 1 < N : (half == 0 && 32 < N);
    if (act && in && (v[q] >> 6) == (nx >> 6)) tie |= 1u << q;
  }
  bool coll = false;
  if (tie) {
#pragma unroll
    for (int q = 0; q < 32; q++) {
      const uint32_t nx = q + 1 < 32 ? v[q + 1] : first1;
      if (((tie >> q) & 1u) && (Krow[63 - (v[q] & 63u)] >> 6) != (Krow[63 - (nx & 63u)] >> 6)) coll = true;
    }
  }
  const int other = __shfl_xor_sync(0xffffffffu, coll ? 1 : 0, 1);  // (unconditional: every lane shuffles)
  coll = coll || other != 0;
  __syncwarp();
  if (coll && half == 0) {  // rare: exact insertion pass over the whole row
    for (int p = 1; p < N; p++) {
      const uint8_t cp = ord[p];
      const unsigned long long kp = Krow[cp];
      int q = p - 1;
      while (q >= 0 && Krow[ord[q]] < kp) {
        ord[q + 1] = ord[q];
        q--;
      }
      ord[q + 1] = cp;
    }
  }
}

// Greedy rounds on sorted key rows (pitch PK), one warp: a head's cross-row
// key swaps the column field for (63 - row), so one 64-bit max picks the best
// head with ties to the lowest row — np.argmax's first occurrence.
template <typename T, int KB>
__device__ __forceinline__ double p2_rounds_keys(const unsigned long long *Kr, int PK, const uint8_t *ord, int N, int emin,
                                                 int32_t *mrow, int lane) {
  unsigned long long hk[KB];
  int ptr[KB];
  bool act[KB];
  uint32_t tk[KB];  // taken columns, 32 per word (32-bit tests on the advance path)
  const int OP = p2_ord_pitch(N);
#pragma unroll
  for (int q = 0; q < KB; q++) tk[q] = 0u;
  auto taken_col = [&](int c) { return ((KB > 1 && c >= 32 ? tk[KB - 1] : tk[0]) >> (c & 31)) & 1u; };
#pragma unroll
  for (int cc = 0; cc < KB; cc++) {
    const int i = lane + 32 * cc;
    act[cc] = i < N;
    ptr[cc] = 0;
    hk[cc] = act[cc] ? Kr[i * PK + ord[i * OP]] : 0ull;
  }
  double wsum = 0.0;
  for (int round = 0; round < N; round++) {
    unsigned long long g = 0ull;
#pragma unroll
    for (int cc = 0; cc < KB; cc++) {
      const unsigned long long gk = (hk[cc] & ~63ull) | (unsigned long long)(63 - (lane + 32 * cc));
      if (act[cc] && gk > g) g = gk;
    }
    const unsigned ghi = __reduce_max_sync(0xffffffffu, (unsigned)(g >> 32));
    const unsigned glo = __reduce_max_sync(0xffffffffu, (unsigned)(g >> 32) == ghi ? (unsigned)g : 0u);
    const int brow = 63 - (int)(glo & 63u);
    unsigned long long mine = hk[0];
#pragma unroll
    for (int cc = 1; cc < KB; cc++)
      if ((brow >> 5) == cc) mine = hk[cc];
    const unsigned long long wk = __shfl_sync(0xffffffffu, mine, brow & 31);
    const int bcol = 63 - (int)(wk & 63ull);
    if (lane == 0) {
      mrow[2 * brow] = (int)(unsigned)(wk >> 32);  // winning key (value bits) for W
      mrow[2 * brow + 1] = (int)(unsigned)wk;
    }
    if (KB > 1 && bcol >= 32) tk[KB - 1] |= 1u << (bcol & 31); else tk[0] |= 1u << (bcol & 31);
    // advance the rows whose head column was taken: the lane's rows'
    // loads are issued side by side (one order load, one key load on the
    // critical path when the next column is free, the common case)
    bool adv[KB];
    int col[KB];
#pragma unroll
    for (int cc = 0; cc < KB; cc++) {
      if (lane + 32 * cc == brow) act[cc] = false;
      adv[cc] = act[cc] && 63 - (int)(hk[cc] & 63ull) == bcol;
      col[cc] = adv[cc] ? (int)ord[(lane + 32 * cc) * OP + (++ptr[cc])] : 0;
    }
#pragma unroll
    for (int cc = 0; cc < KB; cc++)
      if (adv[cc])
        while (taken_col(col[cc])) col[cc] = ord[(lane + 32 * cc) * OP + (++ptr[cc])];
#pragma unroll
    for (int cc = 0; cc < KB; cc++)
      if (adv[cc]) hk[cc] = Kr[(lane + 32 * cc) * PK + col[cc]];
  }
  __syncwarp();
  if (lane == 0)  // similarity.py:150: Python's sum, row order
    for (int i = 0; i < N; i++) {
      const unsigned long long k = ((unsigned long long)(unsigned)mrow[2 * i] << 32) | (unsigned)mrow[2 * i + 1];
      wsum += p2_key_value<T>(k, emin);
    }
  return wsum;
}

template <typename T, int KB, int AR, int BC, int PW, int MINB>
__global__ void __launch_bounds__(32 * (PW + 1), MINB)
    isorank_pair2_kernel(const int32_t *n_nodes, PairWork work, PairOut out, Pair2Params prm, const T *useq,
                         const double *dseq, const int64_t *uoff, unsigned long long *counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = prm.N, P = N | 1;
  const P2Smem L = p2_smem_layout(N, sizeof(T), prm.kcap);
  P2Meta *meta = (P2Meta *)(smem_raw + L.meta);
  double *red = (double *)(smem_raw + L.red);
  uint32_t *amb = (uint32_t *)(smem_raw + L.amb);
  int64_t *s_item = (int64_t *)(smem_raw + L.item);
  int32_t *s_first = (int32_t *)(smem_raw + L.first);
  constexpr int NP = 32 * PW;       // producer threads
  constexpr int NALL = NP + 32;     // producers + consumer warp
  constexpr int BAR_P = 1, BAR_FULL = 2, BAR_EMPTY = 4;  // named barriers (ids 2,3 / 4,5 per buffer)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double inv_nn = 1.0 / (double)((long long)N * N);

  if (warp == PW) {
    // ---------------- consumer: greedy rounds of the pairs in order
    // (a second consumer warp owning one buffer each measured 2% slower)
    int32_t *mrow = (int32_t *)(smem_raw + L.mrow);
    unsigned long long ph_t = 0;
    int ph_last = -1;
    for (int it = 0;; it++) {
      const int s = it & 1;
      P2_PHASE(8);  // wait for a full buffer
      nbar_sync(BAR_FULL + s, NALL);
      P2_PHASE(9);  // greedy rounds + outputs
      const P2Meta mt = meta[s];
      if (!mt.valid) { P2_PHASE(15); break; }
      const T *Xs = (const T *)(smem_raw + L.x[s]);
      const double wsum =
          mt.keys ? p2_rounds_keys<T, KB>((const unsigned long long *)Xs, 32 * KB + 1, smem_raw + L.ord[s], N, mt.emin,
                                          mrow, lane)
                  : p2_rounds<T, KB>(Xs, P, N, smem_raw + L.ord[s], mrow, lane);
      if (lane == 0) {
        if (out.d) out.d[mt.slot] = isorank_distance_of(wsum, N);
        if (out.W) out.W[mt.slot] = wsum;
        if (out.iters) out.iters[mt.slot] = mt.K;
        if (out.conv) out.conv[mt.slot] = mt.conv;
      }
      __syncwarp();
      nbar_arrive(BAR_EMPTY + s, NALL);
    }
    return;
  }

  // ---------------- producers
  const double invN = 1.0 / (double)N;
  const double c = (1.0 - prm.alpha) * inv_nn;
  const int mmax = prm.max_iter < prm.kcap ? prm.max_iter : prm.kcap;
  double *apw = (double *)(smem_raw + L.tab);
  for (int m = tid; m <= prm.kcap + 1; m += NP) apw[m] = prm.apow[m];  // alpha^m, once per CTA
  nbar_sync(BAR_P, NP);
  const int NPt = seq_pitch<T>(N);                      // history row pitch
  const int SPD = p2_stage_pitch(NPt, (int)sizeof(T));  // staged row pitch (conflict-free fragment loads)
  unsigned long long ph_t = 0;
  int ph_last = -1;
  // items are claimed one pair ahead (thread 0 holds the claim in a register
  // while the current pair runs), so the global atomic's round trip is not
  // on the producers' path; every claimed item below n_items is processed
  unsigned long long claim = tid == 0 ? atomicAdd(counter, 1ull) : 0ull;
  for (int it = 0;; it++) {
    const int s = it & 1;
    P2_PHASE(0);  // claim an item + wait for the free buffer
    if (tid == 0) {
      *s_item = (int64_t)claim;
      claim = atomicAdd(counter, 1ull);
      s_first[0] = 0x7fffffff;
      s_first[1] = 0x7fffffff;
      s_first[2] = -1;
    }
    for (int q = tid; q <= (prm.kcap >> 5); q += NP) amb[q] = 0u;
    nbar_sync(BAR_P, NP);
    const int64_t item = *s_item;
    if (it >= 2) nbar_sync(BAR_EMPTY + s, NALL);  // buffer s released by the consumer (pair it-2)
    if (item >= work.n_items) {
      if (tid == 0) meta[s].valid = 0;
      nbar_arrive(BAR_FULL + s, NALL);
      if (it >= 1) nbar_sync(BAR_EMPTY + (s ^ 1), NALL);  // match the consumer's last release
      break;
    }
    T *Xs = (T *)(smem_raw + L.x[s]);
    T *stg = Xs;
    uint8_t *ord = smem_raw + L.ord[s];
    int64_t slot, ca, cb;
    if (work.mode == WORK_RECT) {
      // (query, corpus) rectangle in size-sorted positions; A = the query
      int lo = 0, hi = work.nrect - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (work.rect_start[mid] <= item) lo = mid; else hi = mid - 1;
      }
      const int32_t *R = work.rect + 4 * lo;
      const int64_t loc = item - work.rect_start[lo];
      const int w = R[3] - R[2];
      const int q = R[0] + (int)(loc / w), cc = R[2] + (int)(loc % w);
      slot = (int64_t)(work.qperm[q] - work.qbase) * work.ld + (work.cperm[cc] - work.cbase);
      ca = prm.cbase + q;
      cb = prm.cbase2 + cc;
    } else {
      // triangle unit -> sorted rows a <= b; the alignment runs in the caller's
      // (lower graph index, higher graph index) direction
      // row a of unit uu: row_start[a] = a K - a (a - 1) / 2 <= uu, in closed form
      const int64_t uu = work.u0 + item;
      const int64_t Kt = work.K;
      const double bq = 2.0 * (double)Kt + 1.0;
      int64_t a = (int64_t)((bq - sqrt(bq * bq - 8.0 * (double)uu)) * 0.5);
      auto rstart = [&](int64_t x) { return x * Kt - x * (x - 1) / 2; };
      if (a < 0) a = 0;
      if (a > Kt - 1) a = Kt - 1;
      while (a > 0 && rstart(a) > uu) a--;
      while (a + 1 < Kt && rstart(a + 1) <= uu) a++;
      const int b = (int)(a + (uu - rstart(a)));
      int pa = (int)a, pb = b;
      if (work.perm[pa] > work.perm[pb]) { const int t = pa; pa = pb; pb = t; }
      slot = uu - work.out_base;
      ca = prm.cbase + pa;
      cb = prm.cbase + pb;
    }
    const T *UA = useq + uoff[ca];
    const T *UB = useq + uoff[cb];
    const double *DA = dseq + ca * (int64_t)(prm.kcap + 1);
    const double *DB = dseq + cb * (int64_t)(prm.kcap + 1);
    P2_PHASE(1);  // bracket scan + exact deltas

    // ---- stopping sweep K (similarity.py:139-146): every sweep's bracket in
    // parallel (alpha^m from the host's table, the same sequential products),
    // then exact delta only for the ambiguous sweeps before the first
    // certain stop, in order
    for (int m = tid + 1; m <= mmax; m += NP) {
      const double ak = apw[m];
      const double da = DA[m], db = DB[m];
      const double hiB = ak * invN * (da + db) * (1.0 + prm.eps);
      const double loB = ak * invN * fmax(da, db) * (1.0 - prm.eps);
      if (hiB < prm.tol) atomicMin(s_first, m);
      else if (loB < prm.tol) atomicOr(amb + (m >> 5), 1u << (m & 31));
    }
    nbar_sync(BAR_P, NP);
    int K = mmax;
    bool conv = false;
    {
      const int first = *s_first;
      if (first != 0x7fffffff) { K = first; conv = true; }
      const int lim = first == 0x7fffffff ? mmax : first - 1;
      for (int wd = 0; wd <= (lim >> 5); wd++) {
        uint32_t bits = amb[wd];
        while (bits) {
          const int m = wd * 32 + __ffs(bits) - 1;
          bits &= bits - 1;
          if (m > lim) break;
          // exact delta_m = alpha^m/N^2 sum_ij |u_m[i] v_m[j] - u_{m-1}[i] v_{m-1}[j]|
          const T *un = UA + (size_t)m * NPt, *uo = UA + (size_t)(m - 1) * NPt;
          const T *vn = UB + (size_t)m * NPt, *vo = UB + (size_t)(m - 1) * NPt;
          double dl = 0.0;
          for (int e = tid; e < N * N; e += NP) {
            const int i = e / N, j = e - (e / N) * N;
            dl += fabs((double)fma(-uo[i], vo[j], un[i] * vn[j]));
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) dl += __shfl_xor_sync(0xffffffffu, dl, o);
          if (lane == 0) red[warp] = dl;
          nbar_sync(BAR_P, NP);
          double S = 0.0;
          for (int q = 0; q < PW; q++) S += red[q];
          nbar_sync(BAR_P, NP);  // red is rewritten by the next exact pass
          if (apw[m] * inv_nn * S < prm.tol) {  // similarity.py:144
            K = m;
            conv = true;
            wd = prm.kcap;  // ends the scan
            break;
          }
        }
      }
    }

    // ---- X_K = sum_{m<K} (c alpha^m) u_m v_m^T + (alpha^K/N^2) u_K v_K^T, the
    // u/v rows staged through shared memory in chunks of P2_KC sweeps
    // (16-byte cp.async; rows past K zero-filled up to the chunk's end)
    P2_PHASE(2);  // staging + rank-K product + key build
    const int nch = (K + 1 + P2_KC - 1) / P2_KC;  // rows m = 0..K
    // staging assignment: copy q (16 bytes) of rows mm0, mm0 + sstep, ...
    constexpr int EPU = 16 / sizeof(T);  // elements per 16-byte copy
    const int upr = NPt / EPU, w2 = 2 * upr;
    const int sstep = NP / w2, sq = tid % w2, smm0 = tid / w2;
    const int sside = sq >= upr, sr = (sq - sside * upr) * EPU;
    const T *ssrc = (sside ? UB : UA) + sr;
    // a P2_NS-deep ring: chunk ch lives in buffer ch % P2_NS; two chunks
    // are in flight while one is multiplied, one producer barrier per chunk
    auto stage = [&](int ch) {
      if (ch < nch && smm0 < sstep) {
        T *dst = stg + (ch % P2_NS) * P2_KC * SPD + sside * NPt + sr;
        const int m0 = ch * P2_KC;
        for (int mm = smm0; mm < P2_KC; mm += sstep) {
          const bool ok = m0 + mm <= K;
          big_cp_async_zfill<16>(dst + mm * SPD, ssrc + (size_t)(ok ? m0 + mm : 0) * NPt, ok);
        }
      }
      big_cp_async_commit();  // (empty groups past the last chunk keep the wait counts uniform)
    };
#pragma unroll
    for (int q = 0; q + 1 < P2_NS; q++) stage(q);
    int emn = 0x7fffffff, emx = -1;
    int emin = 0;
    bool keys = true;
    constexpr int PK = 32 * KB + 1;
    unsigned long long *Kr = (unsigned long long *)Xs;
    {
      // fp64 tensor cores: mma.m8n8k4 accumulates each 8x8 tile as the fma
      // chain over k in order (bitwise equal to the scalar chain, probed on
      // B200: tools/probes/dmma_probe.cu), so X is the same as the m-ascending
      // fma accumulation of the low-rank kernel.  Warp tile grid WR x WC,
      // TR x TC 8x8 tiles per warp covering BC x BC tiles (N <= 8 BC: the
      // host launches the BC = 6 instance for N <= 48, so the mma work there
      // is 36 tiles instead of 64; predicated mma.sync measured slower).
      constexpr int WR = 2, WC = PW / 2, TR = BC / WR, TC = BC / WC;
      static_assert(TR * WR == BC && TC * WC == BC && 8 * BC <= 32 * KB, "tile grid");
      const int wr = warp % WR, wc = warp / WR;
      const int lr = lane >> 2, lk = lane & 3;
      double acc[TR][TC][2];
#pragma unroll
      for (int x = 0; x < TR; x++)
#pragma unroll
        for (int y = 0; y < TC; y++) acc[x][y][0] = acc[x][y][1] = 0.0;
      for (int ch = 0; ch < nch; ch++) {
        big_cp_async_wait_group<P2_NS - 2>();  // this thread's copies of chunk ch have landed
        nbar_sync(BAR_P, NP);                  // everyone's have; everyone is done with chunk ch - 1
        stage(ch + P2_NS - 1);                 // into chunk ch - 1's buffer
        const T *buf = stg + (ch % P2_NS) * P2_KC * SPD;  // (fp32 mode: rows promoted to fp64 for the mma)
        const int m0 = ch * P2_KC;
#pragma unroll
        for (int k0 = 0; k0 < P2_KC; k0 += 4) {
          const int m = m0 + k0 + lk;  // this lane's k
          if (m0 + k0 > K) break;
          // c alpha^m (the low-rank kernel's cak) / alpha^K / N^2 (its sc), rounded to T
          const double cf = (m < K) ? (double)(T)(c * apw[m]) : (m == K ? (double)(T)(apw[m] * inv_nn) : 0.0);
          const T *row = buf + (k0 + lk) * SPD;
          double af[TR], bf[TC];
#pragma unroll
          for (int x = 0; x < TR; x++) {
            const int i = (wr * TR + x) * 8 + lr;
            af[x] = cf * (i < N ? (double)row[i] : 0.0);
          }
#pragma unroll
          for (int y = 0; y < TC; y++) {
            const int j = (wc * TC + y) * 8 + lr;
            bf[y] = j < N ? (double)row[NPt + j] : 0.0;
          }
#pragma unroll
          for (int x = 0; x < TR; x++)
#pragma unroll
            for (int y = 0; y < TC; y++)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                           : "+d"(acc[x][y][0]), "+d"(acc[x][y][1])
                           : "d"(af[x]), "d"(bf[y]));
        }
      }
      P2_PHASE(5);  // exponent range + key build
      big_cp_async_wait_group<0>();  // (only empty groups remain; the producer barrier below the
                                     // exponent reduction orders the key writes after every read)
#pragma unroll
      for (int x = 0; x < TR; x++)
#pragma unroll
        for (int y = 0; y < TC; y++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int i = (wr * TR + x) * 8 + lr, j = (wc * TC + y) * 8 + 2 * lk + h;
            if (i < N && j < N) {
              const int e = big_exponent(acc[x][y][h]);
              emn = min(emn, e);
              emx = max(emx, e);
            }
          }
      emn = __reduce_min_sync(0xffffffffu, emn);
      emx = __reduce_max_sync(0xffffffffu, emx);
      if (lane == 0) {
        atomicMin(s_first + 1, emn);
        atomicMax(s_first + 2, emx);
      }
      nbar_sync(BAR_P, NP);
      emin = s_first[1];
      keys = p2_use_keys<T>(emin, s_first[2]);  // the same predicate as the readers below
#pragma unroll
      for (int x = 0; x < TR; x++)
#pragma unroll
        for (int y = 0; y < TC; y++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int i = (wr * TR + x) * 8 + lr, j = (wc * TC + y) * 8 + 2 * lk + h;
            if (i < N && j < N) {
              if (keys) Kr[i * PK + j] = p2_key<T>((T)acc[x][y][h], j, emin);
              else Xs[i * P + j] = (T)acc[x][y][h];
            }
          }
    }
    nbar_sync(BAR_P, NP);
    P2_PHASE(3);  // row orders
    // (emin / keys were read before this barrier: thread 0 rewrites s_first
    // for the next pair as soon as it passes it)
    if (keys) {
      // ---- row orders: one thread per row, 32-bit prefix keys in registers
      if constexpr (KB == 2) {  // two adjacent lanes per row
        const int row = tid >> 1, half = tid & 1;
        const bool act = row < N;
        p2_row_order_pair<T>(Kr + (act ? row : 0) * PK, N, ord + (act ? row : 0) * p2_ord_pitch(N), half, act);
      } else {
        if (tid < N) p2_row_order<T, KB>(Kr + tid * PK, N, ord + tid * p2_ord_pitch(N));
      }
    } else {
      for (int i = warp; i < N; i += PW) p2_sort_row<T, KB>(Xs + i * P, N, ord + i * p2_ord_pitch(N), lane);
    }
    if (tid == 0) {
      meta[s].slot = slot;
      meta[s].K = K;
      meta[s].conv = conv ? 1 : 0;
      meta[s].valid = 1;
      meta[s].keys = keys ? 1 : 0;
      meta[s].emin = emin;
    }
    nbar_arrive(BAR_FULL + s, NALL);  // publishes X, ord, meta (bar.arrive orders prior smem writes)
    P2_PHASE(4);
  }
  P2_PHASE(15);
}

}  // namespace cfgsim
