// Low-rank IsoRank pair kernel for sm_100a (start vector = uniform).
//
// The reference iterates (similarity.py:139-146)
//     x <- (alpha K^T x + (1-alpha) h) / sum(.),   K = kron(A', B'),
// from x0 = h = 1/N^2.  A' and B' are row-stochastic, so sum(.) == 1 in exact
// arithmetic and the map is affine; with X = x as an N x N matrix the iterates
// have the closed form
//     X_k = c * sum_{m<k} alpha^m u_m v_m^T + (alpha^k / N^2) u_k v_k^T,
//     u_m = (A'^T)^m 1,  v_m = (B'^T)^m 1,  c = (1-alpha)/N^2,
// and the L1 change the stopping rule tests is a rank-2 norm
//     delta_k = (alpha^k / N^2) * sum_ij | u_k[i] v_k[j] - u_{k-1}[i] v_{k-1}[j] |.
// So a sweep costs two sparse mat-vecs on N-vectors plus ~4 fp64 operations
// per matrix entry, with no shared-memory traffic per entry:
//   * u_k, v_k live in shared memory (3-deep rings);
//   * each thread owns an AR x BC block of entries (rows ty + TY*a, columns
//     tx + TX*b) and keeps the accumulated P_k = c sum_{m<k} alpha^m u_m v_m^T
//     for them in registers;
//   * per sweep: delta_k partials over the owned block, P += c alpha^{k-1}
//     u_{k-1} v_{k-1}^T, and the next mat-vecs u_{k+1} = A'^T u_k,
//     v_{k+1} = B'^T v_k (one thread per output entry), then ONE CTA barrier
//     and a fixed-order reduction of delta_k (deterministic, no atomics).
// At the stop k = K the alignment matrix X_K = P_K + (alpha^K/N^2) u_K v_K^T is
// written to shared memory for the greedy matching epilogue (greedy_match).
//
// Parity: identical iteration counts and d within ~1e-16 of the reference on
// every golden vector and on 3,000 config-2 pairs vs the pinned oracle (the
// closed form only changes floating-point summation order, like the
// two-product restatement).  A caller-supplied start vector is
// not rank-1 and runs on the general kernel (isorank.cuh).
#pragma once
#include "isorank.cuh"

namespace cfgsim {

struct LRParams {
  double alpha;
  double tol;
  int32_t max_iter;
  int32_t cap;    // list entries per side
  int32_t nlim;   // max N of this launch
  int32_t np;     // padded vector length (>= TY*AR, TX*BC)
  int32_t ty, tx; // thread grid of the entry blocks (ty * tx <= blockDim.x)
  // large N: the dense scratch (and, for dense-bound reruns, the lists) live
  // in a per-CTA global-memory slab instead of shared memory
  unsigned char *gslab;
  int64_t gslab_bytes;  // per CTA
  int32_t lists_global;
};

// Offsets of every array; those flagged global are offsets into the CTA's
// global slab, the others into dynamic shared memory.
struct LRSmem {
  size_t dense, idxA, wA, idxB, wB, toffA, toffB, zA, zB, u, v, lo, fr, zflag, red, misc, total, gtotal;
};

template <typename T>
__host__ __device__ inline LRSmem lr_smem_layout(int nlim, int cap, int np, bool dense_global, bool lists_global) {
  LRSmem s;
  size_t o = 0, g = 0;
  auto take = [&](size_t bytes, bool glob = false) {
    size_t &cur = glob ? g : o;
    size_t at = cur;
    cur += (bytes + 15) & ~size_t(15);
    return at;
  };
  const int pitch = nlim | 1;
  // prologue scratch (dense fp64 operator, N x (N|1)) / epilogue X (pitch
  // N|1) plus the greedy-matching scratch behind it
  size_t dbytes = sizeof(double) * (size_t)nlim * pitch;
  const size_t ebytes = sizeof(T) * (size_t)nlim * pitch + 16 + (size_t)nlim * nlim + 8 * (size_t)nlim + 64;
  if (ebytes > dbytes) dbytes = ebytes;
  s.dense = take(dbytes, dense_global);
  s.idxA = take(sizeof(int32_t) * (size_t)cap, lists_global);
  s.wA = take(sizeof(T) * (size_t)cap, lists_global);
  s.idxB = take(sizeof(int32_t) * (size_t)cap, lists_global);
  s.wB = take(sizeof(T) * (size_t)cap, lists_global);
  s.toffA = take(sizeof(int32_t) * (nlim + 1));
  s.toffB = take(sizeof(int32_t) * (nlim + 1));
  s.zA = take(sizeof(int32_t) * (nlim + 1));
  s.zB = take(sizeof(int32_t) * (nlim + 1));
  s.u = take(sizeof(T) * 3 * (size_t)np);
  s.v = take(sizeof(T) * 3 * (size_t)np);
  s.lo = take(sizeof(int32_t) * (nlim + 1));
  s.fr = take(sizeof(double) * (nlim + 1));
  s.zflag = take(sizeof(uint8_t) * (nlim + 1));
  s.red = take(sizeof(double) * 32);
  s.misc = take(64);
  s.total = o;
  s.gtotal = g;
  return s;
}

// y[t] = (M^T x)[t] = sum_{e in column t} w_e x[i_e] + (1/N) sum_{i in z} x[i]
template <typename T>
__device__ __forceinline__ T lr_matvec_entry(const int32_t *__restrict__ toff, const int32_t *__restrict__ idx,
                                             const T *__restrict__ w, const int32_t *__restrict__ z, int nz,
                                             const T *__restrict__ x, int t, T invN) {
  // two independent chains each (fixed order: deterministic)
  T z0 = 0, z1 = 0;
  int e = 0;
  for (; e + 1 < nz; e += 2) {
    z0 += x[z[e]];
    z1 += x[z[e + 1]];
  }
  if (e < nz) z0 += x[z[e]];
  T a0 = (z0 + z1) * invN, a1 = 0;
  const int e1 = toff[t + 1];
  e = toff[t];
  for (; e + 1 < e1; e += 2) {
    a0 = fma(w[e], x[idx[e]], a0);
    a1 = fma(w[e + 1], x[idx[e + 1]], a1);
  }
  if (e < e1) a0 = fma(w[e], x[idx[e]], a0);
  return a0 + a1;
}

template <typename T, int KB, int AR, int BC, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
    isorank_lowrank_kernel(DevCorpus CA, DevCorpus CB, PairWork work, PairOut out, LRParams prm,
                           unsigned long long *counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const bool dglob = prm.gslab != nullptr, lglob = prm.lists_global != 0;
  const LRSmem L = lr_smem_layout<T>(prm.nlim, prm.cap, prm.np, dglob, lglob);
  unsigned char *gbase = dglob ? prm.gslab + (size_t)blockIdx.x * prm.gslab_bytes : nullptr;
  double *dense = (double *)((dglob ? gbase : smem_raw) + L.dense);
  T *Xs = (T *)dense;  // epilogue alignment matrix (aliases the scratch)
  unsigned char *lbase = lglob ? gbase : smem_raw;
  int32_t *idxA = (int32_t *)(lbase + L.idxA);
  T *wA = (T *)(lbase + L.wA);
  int32_t *idxB = (int32_t *)(lbase + L.idxB);
  T *wB = (T *)(lbase + L.wB);
  int32_t *toffA = (int32_t *)(smem_raw + L.toffA);
  int32_t *toffB = (int32_t *)(smem_raw + L.toffB);
  int32_t *zA = (int32_t *)(smem_raw + L.zA);
  int32_t *zB = (int32_t *)(smem_raw + L.zB);
  T *uR = (T *)(smem_raw + L.u);
  T *vR = (T *)(smem_raw + L.v);
  int32_t *lo_s = (int32_t *)(smem_raw + L.lo);
  double *fr_s = (double *)(smem_raw + L.fr);
  uint8_t *zflag = (uint8_t *)(smem_raw + L.zflag);
  double *red = (double *)(smem_raw + L.red);
  int32_t *misc = (int32_t *)(smem_raw + L.misc);
  int64_t *s_item = (int64_t *)(misc + 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  const int np = prm.np, TY = prm.ty, TX = prm.tx;
  const bool owner = tid < TY * TX;
  const int ty = owner ? tid / TX : 0, tx = owner ? tid - (tid / TX) * TX : 0;

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
      const DevCorpus &C1 = dir ? CB : CA;
      const DevCorpus &C2 = dir ? CA : CB;
      const int na = C1.n_nodes[g1], nb = C2.n_nodes[g2];
      const int N = na > nb ? na : nb;
      const int P = N | 1;

      // ---- prologue: column lists of both row-normalised operators
      int32_t *nzA = misc + 1, *nzB = misc + 2;
      bool ok = build_side<T, KB, 1, false>(C1, g1, N, P, dense, lo_s, fr_s, zflag, zA, nzA, toffA, nullptr,
                                            idxA, wA, prm.cap, false, misc);
      if (ok)
        ok = build_side<T, KB, 1, false>(C2, g2, N, P, dense, lo_s, fr_s, zflag, zB, nzB, toffB, nullptr,
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
      const T invN = (T)(1.0 / (double)N);

      // ---- u_0 = v_0 = 1 (zero padding up to np), u_1 = A'^T 1, v_1 = B'^T 1
      for (int q = tid; q < 3 * np; q += NT) {
        const T one = ((q % np) < N && q < np) ? (T)1 : (T)0;
        uR[q] = one;
        vR[q] = one;
      }
      __syncthreads();
      for (int q = tid; q < 2 * N; q += NT) {
        if (q < N)
          uR[np + q] = lr_matvec_entry(toffA, idxA, wA, zA, nzAv, uR, q, invN);
        else
          vR[np + q - N] = lr_matvec_entry(toffB, idxB, wB, zB, nzBv, vR, q - N, invN);
      }
      __syncthreads();

      const double c = (1.0 - prm.alpha) * (1.0 / (double)((long long)N * N));  // (1-alpha)*uniform, :140
      const double inv_nn = 1.0 / (double)((long long)N * N);
      T Pacc[AR][BC];
#pragma unroll
      for (int a = 0; a < AR; a++)
#pragma unroll
        for (int b = 0; b < BC; b++) Pacc[a][b] = 0;
      double ak1 = 1.0;  // alpha^(k-1)
      int it_done = prm.max_iter;
      bool converged = false;
      int k = 1;
      for (;; k++) {
        const T *uo = uR + ((k - 1) % 3) * np, *un = uR + (k % 3) * np;
        const T *vo = vR + ((k - 1) % 3) * np, *vn = vR + (k % 3) * np;
        // delta_k partial and P += c alpha^(k-1) u_{k-1} v_{k-1}^T on the owned block
        T dl = 0;
        if (owner) {
          const T cak = (T)(c * ak1);
          T uoa[AR], una[AR], cua[AR];
#pragma unroll
          for (int a = 0; a < AR; a++) {
            const int i = ty + TY * a;
            uoa[a] = uo[i];
            una[a] = un[i];
            cua[a] = cak * uoa[a];
          }
#pragma unroll
          for (int b = 0; b < BC; b++) {
            const int j = tx + TX * b;
            const T vob = vo[j], vnb = vn[j];
#pragma unroll
            for (int a = 0; a < AR; a++) {
              const T d = fma(-uoa[a], vob, una[a] * vnb);
              dl += fabs(d);
              Pacc[a][b] = fma(cua[a], vob, Pacc[a][b]);
            }
          }
        }
        // next mat-vecs u_{k+1}, v_{k+1} (harmless extra work after the last sweep)
        if (k < prm.max_iter) {
          T *uw = uR + ((k + 1) % 3) * np, *vw = vR + ((k + 1) % 3) * np;
          for (int q = tid; q < 2 * N; q += NT) {
            if (q < N)
              uw[q] = lr_matvec_entry(toffA, idxA, wA, zA, nzAv, un, q, invN);
            else
              vw[q - N] = lr_matvec_entry(toffB, idxB, wB, zB, nzBv, vn, q - N, invN);
          }
        }
        double ds = (double)dl;
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) ds += __shfl_xor_sync(0xffffffffu, ds, m);
        if (lane == 0) red[((k & 1) << 4) + warp] = ds;  // double-buffered partials
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < NW; w++) tot += red[((k & 1) << 4) + w];
        const double ak = ak1 * prm.alpha;
        const double delta = ak * inv_nn * tot;  // sum |fresh - x|, :142
        if (delta < prm.tol) {                   // :144
          it_done = k;
          converged = true;
          break;
        }
        if (k >= prm.max_iter) break;
        ak1 = ak;
      }

      // ---- X_K = P_K + alpha^K / N^2 u_K v_K^T  ->  shared memory (pitch P)
      {
        const double akK = ak1 * prm.alpha;
        const T *uK = uR + (k % 3) * np, *vK = vR + (k % 3) * np;
        if (owner) {
          const T sc = (T)(akK * inv_nn);
#pragma unroll
          for (int a = 0; a < AR; a++) {
            const int i = ty + TY * a;
            const T su = sc * uK[i];
#pragma unroll
            for (int b = 0; b < BC; b++) {
              const int j = tx + TX * b;
              if (i < N && j < N) Xs[i * P + j] = fma(su, vK[j], Pacc[a][b]);
            }
          }
        }
      }
      __syncthreads();
      {
        uint8_t *scr = (uint8_t *)Xs + ((sizeof(T) * (size_t)N * P + 15) & ~(size_t)15);
        const double wsum = greedy_match<T, KB>(Xs, P, N, scr, lane, warp, NW, out.match);
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
