// cfgsim C ABI (include/cfgsim.h): corpus upload, tier scheduling, launches.
//
// Replaces the reference's per-pair Python loop (similarity.py:240-246) and
// measure_distance ISO branch (similarity.py:176-189).  All arithmetic of
// the pair path runs in isorank.cuh on sm_100a; this file only moves data,
// buckets pairs into on-chip tiers by N = max(n_a, n_b), and launches
// persistent kernels that pull pairs from an atomic work counter (pair cost
// varies ~8x with the data-dependent iteration count).
#include <cuda_runtime.h>
#include <sched.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cfgsim.h"
#include <nvtx3/nvToolsExt.h>
#include "isorank.cuh"
#include "tiers.h"
#include "isorank_lr.cuh"
#include "flat.cuh"
#include "ward.cuh"
#include "isorank_start.cuh"
#include "cost_model.h"

using namespace cfgsim;

// NVTX ranges (SURVEY §5 tracing): pack / stage 1 / stage 2 / large-N /
// gather show up as named ranges under nsys or ncu --nvtx
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
#define CFGSIM_NVTX(name) NvtxRange nvtx_range_(name)

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(e_ == cudaErrorMemoryAllocation ? CFGSIM_ERR_NOMEM : CFGSIM_ERR_CUDA, \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                 \
  } while (0)

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// page-locked host memory (cudaHostAlloc / registered): D2H lands there directly
bool is_pinned_host_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// cudaFuncSetAttribute + occupancy query, cached per (device, kernel, block,
// smem): both are host round trips into the driver, and a C2 step launches
// ~50 stage-2 / stage-1 kernels
cudaError_t cached_occupancy(const void *fn, int threads, size_t smem, int *occ) {
  struct Key {
    int dev;
    const void *fn;
    int threads;
    size_t smem;
    bool operator<(const Key &o) const {
      return std::tie(dev, fn, threads, smem) < std::tie(o.dev, o.fn, o.threads, o.smem);
    }
  };
  static std::mutex mu;
  static std::map<Key, int> cache;
  static std::map<std::pair<int, const void *>, size_t> attr;  // max dynamic smem already set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  const Key k{dev, fn, threads, smem};
  auto it = cache.find(k);
  if (it != cache.end()) {
    *occ = it->second;
    return cudaSuccess;
  }
  size_t &cur = attr[{dev, fn}];
  if (smem > cur) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cur = smem;
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, threads, smem);
  if (e == cudaSuccess) cache[k] = *occ;
  return e;
}

// RAII device buffer
struct DBuf {
  void *p = nullptr;
  size_t n = 0;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t bytes) {
    if (p) cudaFree(p);
    p = nullptr;
    n = bytes;
    return bytes ? cudaMalloc(&p, bytes) : cudaSuccess;
  }
  template <typename T>
  T *as() const {
    return (T *)p;
  }
};

// Pinned host buffer, grow-only (staging of host outputs and corpus uploads).
struct PinBuf {
  void *p = nullptr;
  size_t n = 0;
  ~PinBuf() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t grow(size_t bytes) {
    if (n >= bytes) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocDefault);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
};

}  // namespace

// A packed corpus in one device allocation: CSR, CSC, graph sizes, the
// size-sorted permutation and the triangle row starts, uploaded with one
// copy from pinned staging (include/cfgsim.h "Packed corpus").
struct cfgsim_corpus {
  int device = 0;
  int32_t K = 0;
  int32_t max_nodes = 0;
  std::vector<int32_t> n_nodes;   // graph order
  std::vector<int32_t> perm;      // sorted position -> graph (n desc, index asc)
  std::vector<int32_t> n_sorted;  // n of perm[a]
  std::vector<int64_t> row_start; // triangle units: K+1
  DBuf d_all;                     // every device array below lives in here
  const int32_t *d_n = nullptr, *d_rowptr = nullptr, *d_col = nullptr, *d_perm = nullptr;
  const int64_t *d_rp_off = nullptr, *d_nz_off = nullptr, *d_row_start = nullptr;
  const double *d_val = nullptr;
  const int32_t *d_cscp = nullptr, *d_csc_row = nullptr;  // transposed copy (large-N kernel)
  const double *d_csc_val = nullptr;
  int64_t bytes = 0;
  DevCorpus dev() const {
    DevCorpus c;
    c.n_graphs = K;
    c.n_nodes = d_n;
    c.rp_off = d_rp_off;
    c.rowptr = d_rowptr;
    c.nz_off = d_nz_off;
    c.col = d_col;
    c.val = d_val;
    c.cscp = d_cscp;
    c.csc_row = d_csc_row;
    c.csc_val = d_csc_val;
    return c;
  }
};

namespace {

// ---------------------------------------------------------------- tiers
// A tier is one kernel instantiation.  nmax is the largest N it can hold
// on-chip (phase A handles column N = 32*KB with an extra uniform pass).  occ is the CTAs/SM the
// tier is tuned for (register-limited); the list capacity is whatever
// shared memory is left at that occupancy, capped by the dense bound.
struct Tier {
  int nmax;
  int kb, nw, r, occ;
  size_t entry_bytes;
  const void *fn;
  size_t (*smem)(int nlim, int cap);
};

template <typename T, int KB, int NW, int R, int MINB>
Tier make_tier() {
  Tier t;
  t.nmax = 32 * KB;
  t.kb = KB;
  t.nw = NW;
  t.r = R;
  t.occ = MINB;
  t.entry_bytes = sizeof(int32_t) + R * sizeof(T);
  t.fn = (const void *)isorank_pair_kernel<T, KB, NW, R, MINB>;
  t.smem = [](int nlim, int cap) { return smem_layout<T, R>(nlim, cap).total; };
  return t;
}

const std::vector<Tier> &tiers(int precision) {
  // R = 4 row/column tiles (measured faster than R = 2 on config-2 corpora)
  static std::vector<Tier> t64 = {make_tier<double, 1, 4, 4, 6>(), make_tier<double, 2, 8, 4, 3>(),
                                  make_tier<double, 4, 16, 4, 1>()};
  static std::vector<Tier> t32 = {make_tier<float, 1, 4, 4, 6>(), make_tier<float, 2, 8, 4, 3>(),
                                  make_tier<float, 4, 16, 4, 1>()};
  return precision == CFGSIM_FP32 ? t32 : t64;
}

constexpr size_t kMaxSmem = 227 * 1024;   // per CTA
constexpr size_t kSmemPerSM = 228 * 1024; // per SM, incl. 1 KB reserved per CTA

int dense_cap(int nlim, int r) { return ((nlim + r - 1) / r) * nlim; }

// CTAs/SM a tier can reach with no dynamic smem (register / warp limits)
int occ_limit(const Tier &T) {
  static std::mutex mu;
  static std::vector<std::pair<const void *, int>> cache;
  std::lock_guard<std::mutex> lk(mu);
  for (auto &e : cache)
    if (e.first == T.fn) return e.second;
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, T.fn, T.nw * 32, 0) != cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
  occ = std::max(1, occ);
  cache.push_back({T.fn, occ});
  return occ;
}

struct Plan {
  int ti = -1, cap = 0, occ = 0;
  bool same_launch(const Plan &o) const { return ti == o.ti && occ == o.occ; }
};

// Tier, list capacity and target CTAs/SM for pairs of size N.  Typical CFG
// operators need <= ~5N list entries per side (measured on config-2
// corpora); the capacity is whatever fits at the highest reachable
// occupancy.  Pairs that still overflow are re-run with the dense bound.
Plan plan_for(int precision, int N, bool dense) {
  const auto &ts = tiers(precision);
  for (size_t i = 0; i < ts.size(); i++) {
    const Tier &T = ts[i];
    if (N > T.nmax) continue;
    const int dc = dense_cap(N, T.r);
    const int need = dense ? dc : std::min(dc, 5 * N + 16);
    const size_t base = T.smem(N, 0) + 64;
    for (int occ = occ_limit(T); occ >= 1; occ--) {
      const size_t budget = std::min(kMaxSmem, kSmemPerSM / occ - 1024);
      if (base >= budget) continue;
      const int fit = (int)((budget - base) / (2 * T.entry_bytes)) - 8;
      if (fit >= need) {
        Plan pl;
        pl.ti = (int)i;
        pl.cap = std::min(fit, dc);
        pl.occ = occ;
        return pl;
      }
    }
  }
  return Plan{};
}

// capacity for a launch sized for nlim at the plan's occupancy
int cap_for(int precision, const Plan &pl, int nlim, bool dense) {
  const Tier &T = tiers(precision)[pl.ti];
  const int dc = dense_cap(nlim, T.r);
  if (dense) return dc;
  const size_t base = T.smem(nlim, 0) + 64;
  const size_t budget = std::min(kMaxSmem, kSmemPerSM / pl.occ - 1024);
  if (base >= budget) return std::min(dc, 5 * nlim + 16);
  return std::max(1, std::min(dc, (int)((budget - base) / (2 * T.entry_bytes)) - 8));
}

// Per-device scratch shared by every corpus handle on that device (work
// counters, overflow lists, large-N slabs, two-stage combo tables).  Calls
// that use it are serialised per device (DeviceGuard below): a recursive
// mutex for host threads, and an event recorded on the previous user's stream
// that the next user's stream waits on, so async calls on different streams
// never overlap on the shared buffers.
struct Scratch {
  DBuf counters, ovf_count, ovf_list, gslab, status;
  DBuf seq_u, seq_d, seq_g, seq_n, seq_off, seq_st, seq_list, seq_apow;  // two-stage combos
  std::string seq_key;  // identity of the combo tables currently uploaded ("" = none)
  int64_t ovf_cap = 0;
  DBuf pool_lin, pool_it, pool_out[4];  // per-call outputs, grow-only (no cudaMalloc/cudaFree per call)
  PinBuf pin_out[4], pin_in;            // pinned staging of host outputs / corpus uploads
  std::recursive_mutex mu;
  // device buffers of destroyed corpora, reused by the next corpus of a
  // similar size (no cudaMalloc / cudaFree — which synchronises — per call)
  std::vector<std::pair<size_t, void *>> corpus_free;
  cudaEvent_t done = nullptr;  // recorded at the end of the last call's stream work
  int depth = 0;               // nesting of guards on the owning thread
};

Scratch &scratch_for(int device) {
  static std::mutex mu;
  static std::vector<Scratch *> per_dev(64, nullptr);
  std::lock_guard<std::mutex> lk(mu);
  if (!per_dev[device]) per_dev[device] = new Scratch();
  return *per_dev[device];
}

// Serialises one ABI call's use of the device's Scratch (see Scratch).  While
// a stream is being captured into a CUDA graph the event wait/record is
// skipped (graph replays are ordered by the capturing stream itself).
class DeviceGuard {
 public:
  DeviceGuard(int device, cudaStream_t st) : S_(scratch_for(device)), st_(st), lk_(S_.mu) {
    if (S_.depth++ > 0) return;  // nested call: the outermost guard orders the stream
    capturing_ = is_capturing(st);
    if (!S_.done && cudaEventCreateWithFlags(&S_.done, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      S_.done = nullptr;
    }
    if (S_.done && !capturing_) cudaStreamWaitEvent(st_, S_.done, 0);
  }
  ~DeviceGuard() {
    if (--S_.depth > 0) return;
    if (S_.done && !capturing_) cudaEventRecord(S_.done, st_);
  }
  DeviceGuard(const DeviceGuard &) = delete;
  DeviceGuard &operator=(const DeviceGuard &) = delete;

 private:
  static bool is_capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return cs != cudaStreamCaptureStatusNone;
  }
  Scratch &S_;
  cudaStream_t st_;
  std::lock_guard<std::recursive_mutex> lk_;
  bool capturing_ = false;
};

// Launch one tier over `work` (persistent grid, atomic work counter).
int launch_tier(int precision, int ti, int nlim, int cap, const DevCorpus &A, const DevCorpus &B,
                const PairWork &work, const PairOut &out, const cfgsim_params *p,
                unsigned long long *counter, cudaStream_t st, int force_m = 0) {
  const Tier &T = tiers(precision)[ti];
  const size_t smem = T.smem(nlim, cap);
  if (smem > kMaxSmem) return fail(CFGSIM_ERR_ARG, "tier shared memory exceeds 227 KB");
  int dev;
  CU(cudaGetDevice(&dev));
  int sms = 0, occ = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CU(cached_occupancy((const void *)T.fn, T.nw * 32, smem, &occ));
  if (occ < 1) return fail(CFGSIM_ERR_CUDA, "tier kernel cannot be resident (occupancy 0)");
  int64_t grid = (int64_t)sms * occ;
  if (grid > work.n_items) grid = work.n_items;
  if (grid < 1) return CFGSIM_OK;
  PairParams prm;
  prm.alpha = p->alpha;
  prm.tol = (precision == CFGSIM_FP32) ? std::max(p->tol, p->tol_fp32) : p->tol;
  prm.max_iter = p->max_iter;
  prm.cap = cap;
  prm.nlim = nlim;
  static const int env_force_m = [] {  // CFGSIM_FORCE_M=1: exact delta every sweep (testing)
    const char *e = getenv("CFGSIM_FORCE_M");
    return (e && atoi(e) != 0) ? 1 : 0;
  }();
  prm.force_m = force_m | env_force_m;
  CU(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st));
  void *args[] = {(void *)&A, (void *)&B, (void *)&work, (void *)&out, (void *)&prm, (void *)&counter};
  CU(cudaLaunchKernel(T.fn, dim3((unsigned)grid), dim3(T.nw * 32), args, smem, st));
  g_launches++;
  return CFGSIM_OK;
}

// ---------------------------------------------------------------- low-rank tiers
// isorank_lowrank_kernel instantiations (isorank_lr.cuh): KB row chunks for
// the prologue/epilogue, AR x BC entries per thread.  Launches are per exact
// N, so the thread grid (TY x TX) and the vector padding fit N tightly.
struct LRTier {
  int nmax, kb, ar, bc;
  const void *fn;
};

const std::vector<LRTier> &lr_tiers(int precision) {
  static std::vector<LRTier> t64 = {
      {32, 1, 4, 4, (const void *)isorank_lowrank_kernel<double, 1, 4, 4, 64, 10>},
      {64, 2, 4, 8, (const void *)isorank_lowrank_kernel<double, 2, 4, 8, 128, 4>},
      {128, 4, 4, 8, (const void *)isorank_lowrank_kernel<double, 4, 4, 8, 512, 1>}};
  static std::vector<LRTier> t32 = {
      {32, 1, 4, 4, (const void *)isorank_lowrank_kernel<float, 1, 4, 4, 64, 10>},
      {64, 2, 4, 8, (const void *)isorank_lowrank_kernel<float, 2, 4, 8, 128, 5>},
      {128, 4, 4, 8, (const void *)isorank_lowrank_kernel<float, 4, 4, 8, 512, 1>}};
  return precision == CFGSIM_FP32 ? t32 : t64;
}

// CFGSIM_ALGO=dense selects the general two-product kernel for every pair
// (A/B validation); default is the low-rank kernel whenever x0 is uniform.
bool use_lowrank() {
  static const bool lr = [] {
    const char *e = getenv("CFGSIM_ALGO");
    return !(e && std::string(e) == "dense");
  }();
  return lr;
}

bool lr_supported(int precision, int N) { return N <= lr_tiers(precision).back().nmax; }
// Pairs with N above this go to the large-N kernel even where a low-rank tier
// exists: measured per-unit cost (tools/calibrate_split.py) low-rank 2.39 /
// 2.89 / 3.16 us at N = 96 / 112 / 128 vs large-N 2.35 us at N = 129.
// CFGSIM_BIG_MIN overrides (A/B).
int big_min() {
  static const int v = [] {
    const char *e = getenv("CFGSIM_BIG_MIN");
    return e ? atoi(e) : 96;
  }();
  return v;
}
bool lr_tier(int precision, int N) { return lr_supported(precision, N) && N <= big_min(); }

int lr_launch(int precision, int nlim, bool dense_lists, const DevCorpus &A, const DevCorpus &B,
              const PairWork &work, const PairOut &out, const cfgsim_params *p, unsigned long long *counter,
              cudaStream_t st) {
  const auto &ts = lr_tiers(precision);
  size_t ti = 0;
  while (ti < ts.size() && nlim > ts[ti].nmax) ti++;
  if (ti == ts.size()) return fail(CFGSIM_ERR_ARG, "pair size N=" + std::to_string(nlim) + " exceeds the low-rank tiers");
  const LRTier &T = ts[ti];
  LRParams prm;
  prm.alpha = p->alpha;
  prm.tol = (precision == CFGSIM_FP32) ? std::max(p->tol, p->tol_fp32) : p->tol;
  prm.max_iter = p->max_iter;
  prm.nlim = nlim;
  prm.ty = (nlim + T.ar - 1) / T.ar;
  prm.tx = (nlim + T.bc - 1) / T.bc;
  const int maxt = T.nmax <= 32 ? 64 : (T.nmax <= 64 ? 128 : 512);  // __launch_bounds__ of the tier
  int nt = std::min(maxt, std::max(64, ((prm.ty * prm.tx + 31) / 32) * 32));
  prm.np = (std::max(std::max(nlim, prm.ty * T.ar), prm.tx * T.bc) + 1) & ~1;
  const int dc = nlim * nlim;
  prm.cap = dense_lists ? dc : std::min(dc, 14 * nlim + 16);
  // scratch placement: dense N x N operator/alignment in global memory for
  // N > 64 (keeps several CTAs per SM); lists in global memory if they would
  // not fit in shared memory (dense-bound reruns of large N)
  const bool dglob = nlim > 64;
  auto layout = [&](bool lg) {
    return precision == CFGSIM_FP32 ? lr_smem_layout<float>(nlim, prm.cap, prm.np, dglob, lg)
                                    : lr_smem_layout<double>(nlim, prm.cap, prm.np, dglob, lg);
  };
  bool lglob = false;
  LRSmem L = layout(false);
  if (L.total > kMaxSmem) {
    if (!dglob) return fail(CFGSIM_ERR_ARG, "low-rank kernel shared memory exceeds 227 KB (N=" + std::to_string(nlim) + ")");
    lglob = true;
    L = layout(true);
  }
  prm.lists_global = lglob ? 1 : 0;
  const size_t smem = L.total;
  prm.gslab = nullptr;
  prm.gslab_bytes = (int64_t)L.gtotal;
  int dev, sms = 0, occ = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CU(cached_occupancy((const void *)T.fn, nt, smem, &occ));
  if (occ < 1) return fail(CFGSIM_ERR_CUDA, "low-rank kernel cannot be resident (occupancy 0)");
  int64_t grid = std::min<int64_t>((int64_t)sms * occ, work.n_items);
  if (grid < 1) return CFGSIM_OK;
  if (dglob) {
    Scratch &S = scratch_for(dev);
    const size_t need = (size_t)grid * L.gtotal;
    if (S.gslab.n < need) {
      CU(cudaStreamSynchronize(st));  // a previous launch may still use the old slab
      CU(S.gslab.alloc(need));
    }
    prm.gslab = S.gslab.as<unsigned char>();
  }
  CU(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st));
  void *args[] = {(void *)&A, (void *)&B, (void *)&work, (void *)&out, (void *)&prm, (void *)&counter};
  CU(cudaLaunchKernel(T.fn, dim3((unsigned)grid), dim3(nt), args, smem, st));
  g_launches++;
  return CFGSIM_OK;
}

// ---------------------------------------------------------------- large-N kernel
// isorank_big_kernel (isorank_big.cuh) for 128 < N <= 1024: one launch per
// sort class (N <= 32 KB), slab per CTA sized for the launch's largest N.
constexpr int kBigNmax = 1024;
constexpr int kBigKey = 1 << 20;  // bucket keys above any N

int big_kb(int N) { return N <= 256 ? 8 : (N <= 512 ? 16 : 32); }

const void *big_fn(int precision, int kb) {
  if (precision == CFGSIM_FP32)
    return kb == 8 ? (const void *)isorank_big_kernel<float, 8>
                   : (kb == 16 ? (const void *)isorank_big_kernel<float, 16> : (const void *)isorank_big_kernel<float, 32>);
  return kb == 8 ? (const void *)isorank_big_kernel<double, 8>
                 : (kb == 16 ? (const void *)isorank_big_kernel<double, 16> : (const void *)isorank_big_kernel<double, 32>);
}

// Iterations after which the delta bracket (isorank_big.cuh) certainly stops:
// delta_k <= 4 alpha^k (1 + eps).
int big_kcap(double alpha, double tol, int max_iter) {
  double a = 1.0;
  for (int k = 1; k <= max_iter; k++) {
    a *= alpha;
    if (4.01 * a < tol) return std::min(max_iter, k + 1);
  }
  return max_iter;
}

int big_launch(int precision, int nlim, const DevCorpus &A, const DevCorpus &B, const PairWork &work,
               const PairOut &out, const cfgsim_params *p, unsigned long long *counter, cudaStream_t st,
               const double *xg = nullptr, int kg = 0, int convg = 0, const BigParams *hist = nullptr) {
  CFGSIM_NVTX("cfgsim.large_n");
  if (nlim > kBigNmax) return fail(CFGSIM_ERR_ARG, "pair size N=" + std::to_string(nlim) + " exceeds 1024");
  const int kb = big_kb(nlim);
  const void *fn = big_fn(precision, kb);
  BigParams prm{};
  prm.xg = xg;  // given-X mode (fp64 only): sort + match an X computed outside
  prm.kg = kg;
  prm.convg = convg;
  if (hist) {  // history mode (fp64 all-pairs): precomputed per-(graph, N) sequences
    prm.hu = hist->hu;
    prm.hd = hist->hd;
    prm.hstride = hist->hstride;
    prm.hcbase = hist->hcbase;
    prm.hapow = hist->hapow;
  }
  prm.alpha = p->alpha;
  prm.tol = (precision == CFGSIM_FP32) ? std::max(p->tol, p->tol_fp32) : p->tol;
  prm.eps = (precision == CFGSIM_FP32) ? 0.02 : 1e-6;
  prm.max_iter = p->max_iter;
  prm.kcap = big_kcap(p->alpha, prm.tol, p->max_iter);
  prm.nlim = nlim;
  const size_t smem = precision == CFGSIM_FP32 ? big_smem_layout<float>(nlim).total : big_smem_layout<double>(nlim).total;
  const size_t slab = precision == CFGSIM_FP32 ? big_slab_layout<float>(nlim, prm.kcap).total
                                               : big_slab_layout<double>(nlim, prm.kcap).total;
  if (smem > kMaxSmem) return fail(CFGSIM_ERR_ARG, "large-N kernel shared memory exceeds 227 KB");
  int dev, sms = 0, occ = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CU(cached_occupancy((const void *)fn, BIG_THREADS, smem, &occ));
  if (occ < 1) return fail(CFGSIM_ERR_CUDA, "large-N kernel cannot be resident (occupancy 0)");
  const int64_t grid = std::min<int64_t>((int64_t)sms * occ, work.n_items);
  if (grid < 1) return CFGSIM_OK;
  Scratch &S = scratch_for(dev);
  const size_t need = (size_t)grid * slab;
  if (S.gslab.n < need) {
    CU(cudaStreamSynchronize(st));  // a previous launch may still use the old slab
    CU(S.gslab.alloc(need));
  }
  if (!S.status.p) {
    CU(S.status.alloc(sizeof(int32_t)));
    CU(cudaMemset(S.status.p, 0, sizeof(int32_t)));
  }
  prm.slab = S.gslab.as<unsigned char>();
  prm.slab_bytes = (int64_t)slab;
  prm.status = S.status.as<int32_t>();
  static const bool phases = [] {
    const char *e = getenv("CFGSIM_PHASES");
    return e && atoi(e) != 0;
  }();
  static DBuf phase_buf;
  prm.phase = nullptr;
  if (phases) {
    if (!phase_buf.p) CU(phase_buf.alloc(8 * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(phase_buf.p, 0, 8 * sizeof(unsigned long long), st));
    prm.phase = phase_buf.as<unsigned long long>();
  }
  CU(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st));
  void *args[] = {(void *)&A, (void *)&B, (void *)&work, (void *)&out, (void *)&prm, (void *)&counter};
  CU(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(BIG_THREADS), args, smem, st));
  g_launches++;
  if (prm.phase) {
    unsigned long long ph[8];
    CU(cudaMemcpyAsync(ph, prm.phase, sizeof(ph), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    double tot = 0;
    for (int k = 0; k < 5; k++) tot += (double)ph[k];
    fprintf(stderr, "[cfgsim big N<=%d] phase cycles (sum over CTAs): operators %.1f%% sweeps %.1f%% gemm %.1f%% "
            "sort %.1f%% greedy %.1f%% total %.3e | sum N %llu advances %llu deep %llu\n", nlim, 100 * ph[0] / tot,
            100 * ph[1] / tot, 100 * ph[2] / tot, 100 * ph[3] / tot, 100 * ph[4] / tot, tot, ph[7], ph[5], ph[6]);
  }
  return CFGSIM_OK;
}

// internal-error flag of the large-N kernel (synchronises the stream)
bool stream_capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

int big_status(Scratch &S, cudaStream_t st) {
  if (!S.status.p) return CFGSIM_OK;
  // (a CUDA-graph capture cannot read it back; the flag is an internal
  // assertion the bracket makes unreachable, checked on every eager call)
  if (stream_capturing(st)) return CFGSIM_OK;
  int32_t v = 0;
  CU(cudaMemcpyAsync(&v, S.status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (v) {
    CU(cudaMemset(S.status.p, 0, sizeof(int32_t)));
    return fail(CFGSIM_ERR_CUDA, "internal: large-N kernel iteration history overflow");
  }
  return CFGSIM_OK;
}

// ---------------------------------------------------------------- two-stage small N
// isorank_seq.cuh: per (graph, N) combo sequences (stage 1), then per-pair
// rank-K products (stage 2).  Used for unordered all-pairs units with N <= 64
// (CFGSIM_TWOSTAGE=0 selects the per-pair low-rank kernel instead).
constexpr int kSeqNmax = 64;

bool use_twostage() {
  static const bool on = [] {
    const char *e = getenv("CFGSIM_TWOSTAGE");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// Combo table of one two-stage run (host side).
struct SeqTable {
  std::vector<int32_t> g, n;
  std::vector<int64_t> uoff;
  int64_t utot = 0;
  template <typename T>
  void add(int32_t graph, int N, int kcap) {
    g.push_back(graph);
    n.push_back(N);
    uoff.push_back(utot);
    utot += (int64_t)(kcap + 1) * seq_pitch<T>(N);
  }
};

cudaError_t grow_buf(DBuf &b, size_t bytes, cudaStream_t st) {
  if (b.n >= bytes) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(st);  // a previous launch may still read the old buffer
  if (e != cudaSuccess) return e;
  return b.alloc(bytes);
}

struct SeqRun {
  double tol, eps;
  int kcap;
};

template <typename T>
SeqRun seq_run_params(const cfgsim_params *p) {
  SeqRun r;
  r.tol = sizeof(T) == 4 ? std::max(p->tol, p->tol_fp32) : p->tol;
  r.eps = sizeof(T) == 4 ? 0.02 : 1e-6;
  r.kcap = big_kcap(p->alpha, r.tol, p->max_iter);
  return r;
}

// Upload a combo table and the alpha^m table.
template <typename T>
int seq_upload(Scratch &S, const SeqTable &tb, const SeqRun &rr, const cfgsim_params *p, cudaStream_t st) {
  const int64_t nc = (int64_t)tb.g.size();
  CU(grow_buf(S.seq_u, sizeof(T) * (size_t)std::max<int64_t>(tb.utot, 1), st));
  CU(grow_buf(S.seq_d, sizeof(double) * (size_t)std::max<int64_t>(nc, 1) * (rr.kcap + 1), st));
  CU(grow_buf(S.seq_g, sizeof(int32_t) * std::max<int64_t>(nc, 1), st));
  CU(grow_buf(S.seq_n, sizeof(int32_t) * std::max<int64_t>(nc, 1), st));
  CU(grow_buf(S.seq_off, sizeof(int64_t) * std::max<int64_t>(nc, 1), st));
  CU(grow_buf(S.seq_st, sizeof(int32_t) * std::max<int64_t>(nc, 1), st));
  CU(cudaMemcpyAsync(S.seq_g.p, tb.g.data(), sizeof(int32_t) * nc, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(S.seq_n.p, tb.n.data(), sizeof(int32_t) * nc, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(S.seq_off.p, tb.uoff.data(), sizeof(int64_t) * nc, cudaMemcpyHostToDevice, st));
  std::vector<double> apow(rr.kcap + 2);  // alpha^m by sequential products (the pair kernels' order)
  apow[0] = 1.0;
  for (int m = 1; m <= rr.kcap + 1; m++) apow[m] = apow[m - 1] * p->alpha;
  CU(grow_buf(S.seq_apow, sizeof(double) * apow.size(), st));
  CU(cudaMemcpyAsync(S.seq_apow.p, apow.data(), sizeof(double) * apow.size(), cudaMemcpyHostToDevice, st));
  return CFGSIM_OK;
}

// Stage 1 for combos [id0, id0 + n), all graphs of corpus C; combos whose
// operator lists overflow are re-run with dense-bound lists.
template <typename T>
int seq_stage1(const cfgsim_corpus *C, int64_t id0, int64_t n, const SeqRun &rr, const cfgsim_params *p, Scratch &S,
               cudaStream_t st, bool single = false) {
  CFGSIM_NVTX("cfgsim.stage1");
  if (n <= 0) return CFGSIM_OK;
  int dev, sms = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SeqParams sp;
  sp.alpha = p->alpha;
  sp.tol = rr.tol;
  sp.eps = rr.eps;
  sp.max_iter = p->max_iter;
  sp.kcap = rr.kcap;
  sp.nlim = kSeqNmax;
  SeqCombos cb;
  cb.n = n;
  cb.id0 = id0;
  cb.list = nullptr;
  cb.g = S.seq_g.as<int32_t>();
  cb.nn = S.seq_n.as<int32_t>();
  cb.uoff = S.seq_off.as<int64_t>();
  cb.status = S.seq_st.as<int32_t>();
  const void *f1 = (const void *)isorank_seq_kernel<T, 2>;
  DevCorpus dc = C->dev();
  T *useq = S.seq_u.as<T>();
  double *dseq = S.seq_d.as<double>();
  // pass 0: typical list capacity; pass 1 re-runs only the combos that
  // overflowed it (status 1) with dense-bound lists — decided on the device,
  // so no host synchronisation sits between the stages
  // single: every combo through the one-combo-per-CTA kernel with dense-bound
  // lists (A/B and debugging; CFGSIM_SEQ_SINGLE=1)
  for (int pass = single ? 1 : 0; pass < 2; pass++) {
    // pass 0: four combos per CTA, warp-synchronous recurrences; pass 1: the
    // one-combo-per-CTA kernel re-runs flagged combos with dense-bound lists
    sp.cap = pass == 0 ? 10 * kSeqNmax + 16 : kSeqNmax * kSeqNmax;  // 10N+16: 2 CTAs/SM
    cb.redo = single ? 0 : pass;
    const void *fk = pass == 0 ? (const void *)isorank_seq4_kernel<T, 2> : f1;
    const int nthr = pass == 0 ? 32 * SEQ4 : 128;
    const size_t smem = pass == 0 ? seq4_smem_layout<T>(kSeqNmax, sp.cap).total : seq_smem_layout<T>(kSeqNmax, sp.cap).total;
    int occ = 0;
    CU(cached_occupancy((const void *)fk, nthr, smem, &occ));
    if (occ < 1) return fail(CFGSIM_ERR_CUDA, "stage-1 kernel cannot be resident");
    const int64_t units = pass == 0 ? (cb.n + SEQ4 - 1) / SEQ4 : cb.n;
    const int64_t grid = std::min<int64_t>((int64_t)sms * occ, units);
    void *args[] = {(void *)&dc, (void *)&cb, (void *)&sp, (void *)&useq, (void *)&dseq};
    CU(cudaLaunchKernel(fk, dim3((unsigned)grid), dim3(nthr), args, smem, st));
    g_launches++;
  }
  return CFGSIM_OK;
}

// Stage 2 over `w` (triangle units or query x corpus rectangles) of one N.
template <typename T>
int seq_stage2(int N, int64_t cbase, int64_t cbase2, const PairWork &w, const PairOut &o, const SeqRun &rr,
               const cfgsim_params *p, Scratch &S, int &launch_no, cudaStream_t st) {
  CFGSIM_NVTX("cfgsim.stage2");
  if (w.n_items <= 0) return CFGSIM_OK;
  int dev, sms = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const bool small = N <= 32;
  const int ar = 4, bc = small ? 4 : 8, pw = small ? 2 : 4;  // producer warps (+1 consumer warp)
  Pair2Params pp;
  pp.alpha = p->alpha;
  pp.tol = rr.tol;
  pp.eps = rr.eps;
  pp.max_iter = p->max_iter;
  pp.kcap = rr.kcap;
  pp.N = N;
  pp.ty = (N + ar - 1) / ar;
  pp.tx = (N + bc - 1) / bc;
  pp.cbase = cbase;
  pp.cbase2 = cbase2;
  pp.apow = S.seq_apow.as<double>();
  static const int minb_env = [] {  // CFGSIM_P2_OCC=2|3: CTAs/SM the stage-2 kernel is compiled for
    const char *e = getenv("CFGSIM_P2_OCC");
    return e ? atoi(e) : 3;
  }();
  const int nt = 32 * (pw + 1);
  const size_t smem = p2_smem_bytes(N, sizeof(T), rr.kcap);
  const void *f2 = small ? (minb_env == 2 ? (const void *)isorank_pair2_kernel<T, 1, 4, 4, 2, 4>
                                          : (const void *)isorank_pair2_kernel<T, 1, 4, 4, 2, 6>)
                         : (minb_env == 2 ? (const void *)isorank_pair2_kernel<T, 2, 4, 8, 4, 2>
                            : N <= 48     ? (const void *)isorank_pair2_kernel<T, 2, 4, 6, 4, 3>  // 6 x 6 mma tiles
                                          : (const void *)isorank_pair2_kernel<T, 2, 4, 8, 4, 3>);
  int occ = 0;
  CU(cached_occupancy((const void *)f2, nt, smem, &occ));
  if (occ < 1) return fail(CFGSIM_ERR_CUDA, "stage-2 kernel cannot be resident");
  const int64_t grid = std::min<int64_t>((int64_t)sms * occ, w.n_items);
  unsigned long long *ctr = S.counters.as<unsigned long long>() + (launch_no++ % 64);
  CU(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
  const int32_t *nn = nullptr;
  const T *useq = S.seq_u.as<T>();
  const double *dseq = S.seq_d.as<double>();
  const int64_t *uo = S.seq_off.as<int64_t>();
  static const bool phases = [] {
    const char *e = getenv("CFGSIM_PHASES");
    return e && atoi(e) != 0;
  }();
  static DBuf phase_buf;
  pp.phase = nullptr;
  if (phases) {
    if (!phase_buf.p) CU(phase_buf.alloc(16 * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(phase_buf.p, 0, 16 * sizeof(unsigned long long), st));
    pp.phase = phase_buf.as<unsigned long long>();
  }
  void *args[] = {(void *)&nn, (void *)&w, (void *)&o, (void *)&pp, (void *)&useq, (void *)&dseq, (void *)&uo,
                  (void *)&ctr};
  CU(cudaLaunchKernel(f2, dim3((unsigned)grid), dim3(nt), args, smem, st));
  g_launches++;
  if (pp.phase) {
    unsigned long long ph[16];
    CU(cudaMemcpyAsync(ph, pp.phase, sizeof(ph), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    double tp = 0, tc = 0;
    for (int k = 0; k < 6; k++) tp += (double)ph[k];
    for (int k = 8; k < 10; k++) tc += (double)ph[k];
    fprintf(stderr, "[cfgsim pair2 N=%d items=%lld grid=%lld] producer: wait/claim %.1f%% bracket+delta %.1f%% "
            "stage+mma+keys %.1f%% row-orders %.1f%% tail %.1f%% (%.3e cyc) | consumer: wait %.1f%% rounds %.1f%% "
            "(%.3e cyc) | of which keys %.1f%%\n", N, (long long)w.n_items, (long long)grid, 100 * ph[0] / tp,
            100 * ph[1] / tp, 100 * (ph[2] + ph[5]) / tp, 100 * ph[3] / tp, 100 * ph[4] / tp, tp, 100 * ph[8] / tc,
            100 * ph[9] / tc, tc, 100 * ph[5] / tp);
  }
  return CFGSIM_OK;
}

template <typename T>
int seq_allpairs_t(const cfgsim_corpus *c, int64_t us, int64_t ue, const cfgsim_params *p, double *d_lin,
                   int32_t *iters_lin, int64_t out_base, int &launch_no, cudaStream_t st) {
  Scratch &S = scratch_for(c->device);
  const SeqRun rr = seq_run_params<T>(p);
  const auto &rs = c->row_start;
  const int a0 = (int)(std::upper_bound(rs.begin(), rs.end(), us) - rs.begin()) - 1;
  const int a1 = (int)(std::upper_bound(rs.begin(), rs.end(), ue - 1) - rs.begin()) - 1;
  // groups of equal N among rows a0..a1; combos (perm[b], N) for b >= the group's first row
  struct Grp { int N, ra, rb; int64_t cbase; };
  std::vector<Grp> grps;
  int64_t ncombo = 0;
  for (int a = a0; a <= a1;) {
    const int N = c->n_sorted[a];
    int b = a;
    while (b + 1 <= a1 && c->n_sorted[b + 1] == N) b++;
    grps.push_back({N, a, b, ncombo - a});
    ncombo += c->K - a;
    a = b + 1;
  }
  // the combo tables depend only on (corpus, unit range, kcap, alpha, T):
  // repeated calls reuse the uploaded tables (a plan, not results — stage 1
  // and stage 2 still run on every call)
  char key[256];
  snprintf(key, sizeof(key), "%p/%lld/%lld/%d/%.17g/%d", (const void *)c, (long long)us, (long long)ue, rr.kcap,
           p->alpha, (int)sizeof(T));
  if (S.seq_key != key) {
    SeqTable tb;
    for (const Grp &gp : grps)
      for (int q = gp.ra; q < c->K; q++) tb.add<T>(c->perm[q], gp.N, rr.kcap);
    S.seq_key.clear();
    if (int rc = seq_upload<T>(S, tb, rr, p, st)) return rc;
    S.seq_key = key;
  }
  if (int rc = seq_stage1<T>(c, 0, ncombo, rr, p, S, st)) return rc;
  for (const Grp &gp : grps) {
    const int64_t gu0 = std::max(us, rs[gp.ra]), gu1 = std::min(ue, rs[gp.rb + 1]);
    if (gu1 <= gu0) continue;
    PairWork w{};
    w.mode = WORK_TRIANGLE;
    w.ordered = 0;
    w.n_items = gu1 - gu0;
    w.u0 = gu0;
    w.out_base = out_base;
    w.row_start = c->d_row_start;
    w.perm = c->d_perm;
    w.K = c->K;
    PairOut o{};
    o.d = d_lin;
    o.iters = iters_lin;
    if (int rc = seq_stage2<T>(gp.N, gp.cbase, 0, w, o, rr, p, S, launch_no, st)) return rc;
  }
  return CFGSIM_OK;
}

// Query-vs-corpus block through the two-stage path: for each N <= 64 the
// combos of queries and corpus graphs with n <= N, then the rectangles
// {n_q == N} x {n_c <= N} and {n_q < N} x {n_c == N} (sorted positions).
template <typename T>
int seq_nearest_t(const cfgsim_corpus *Q, const cfgsim_corpus *C, const std::vector<int32_t> &qs,
                  const std::vector<int32_t> &cs, const int32_t *dqs, const int32_t *dcs, int32_t q0, int32_t c0,
                  int32_t nc, const std::vector<int> &ns, const cfgsim_params *p, double *dm, int &launch_no,
                  cudaStream_t st) {
  Scratch &S = scratch_for(Q->device);
  S.seq_key.clear();  // the shared combo buffers are rewritten below
  const SeqRun rr = seq_run_params<T>(p);
  auto cnt = [](const std::vector<int32_t> &v, const cfgsim_corpus *X, int n, bool le) {
    return (int32_t)((le ? std::upper_bound(v.begin(), v.end(), n, [&](int t, int x) { return t < X->n_nodes[x]; })
                         : std::lower_bound(v.begin(), v.end(), n, [&](int x, int t) { return X->n_nodes[x] < t; })) -
                     v.begin());
  };
  // every size's rectangles and their prefix sums, uploaded once (no host
  // synchronisation between the sizes: the combo tables of the next size are
  // rewritten in stream order after the previous size's kernels)
  std::vector<int32_t> all_rects;
  std::vector<int64_t> all_rsum;
  std::vector<size_t> at_rect(ns.size()), at_rsum(ns.size());
  std::vector<int> nrs(ns.size(), 0);
  for (size_t gi = 0; gi < ns.size(); gi++) {
    const int N = ns[gi];
    const int32_t qlt = cnt(qs, Q, N, false), qle = cnt(qs, Q, N, true);
    const int32_t clt = cnt(cs, C, N, false), cle = cnt(cs, C, N, true);
    at_rect[gi] = all_rects.size();
    at_rsum[gi] = all_rsum.size();
    if (qle > qlt && cle > 0) all_rects.insert(all_rects.end(), {qlt, qle, 0, cle});
    if (qlt > 0 && cle > clt) all_rects.insert(all_rects.end(), {0, qlt, clt, cle});
    const int nr = (int)(all_rects.size() - at_rect[gi]) / 4;
    nrs[gi] = nr;
    int64_t acc = 0;
    all_rsum.push_back(0);
    for (int r = 0; r < nr; r++) {
      const int32_t *R = all_rects.data() + at_rect[gi] + 4 * r;
      acc += (int64_t)(R[1] - R[0]) * (R[3] - R[2]);
      all_rsum.push_back(acc);
    }
  }
  DBuf drs, drect;
  CU(drs.alloc(sizeof(int64_t) * std::max<size_t>(all_rsum.size(), 1)));
  CU(drect.alloc(sizeof(int32_t) * std::max<size_t>(all_rects.size(), 1)));
  if (!all_rsum.empty())
    CU(cudaMemcpyAsync(drs.p, all_rsum.data(), sizeof(int64_t) * all_rsum.size(), cudaMemcpyHostToDevice, st));
  if (!all_rects.empty())
    CU(cudaMemcpyAsync(drect.p, all_rects.data(), sizeof(int32_t) * all_rects.size(), cudaMemcpyHostToDevice, st));
  for (size_t gi = 0; gi < ns.size(); gi++) {
    const int N = ns[gi];
    const int nr = nrs[gi];
    if (nr == 0) continue;
    const int32_t qle = cnt(qs, Q, N, true), cle = cnt(cs, C, N, true);
    SeqTable tb;  // [queries with n <= N | corpus graphs with n <= N], sorted positions
    for (int32_t q = 0; q < qle; q++) tb.add<T>(qs[q], N, rr.kcap);
    for (int32_t x = 0; x < cle; x++) tb.add<T>(cs[x], N, rr.kcap);
    if (int rc = seq_upload<T>(S, tb, rr, p, st)) return rc;
    if (int rc = seq_stage1<T>(Q, 0, qle, rr, p, S, st)) return rc;
    if (int rc = seq_stage1<T>(C, qle, cle, rr, p, S, st)) return rc;
    PairWork w{};
    w.mode = WORK_RECT;
    w.n_items = all_rsum[at_rsum[gi] + nr];
    w.nrect = nr;
    w.rect_start = drs.as<int64_t>() + at_rsum[gi];
    w.rect = drect.as<int32_t>() + at_rect[gi];
    w.qperm = dqs;
    w.cperm = dcs;
    w.qbase = q0;
    w.cbase = c0;
    w.ld = nc;
    PairOut o{};
    o.d = dm;
    if (int rc = seq_stage2<T>(N, 0, qle, w, o, rr, p, S, launch_no, st)) return rc;
  }
  CU(cudaStreamSynchronize(st));  // (drs / drect are freed on return)
  return CFGSIM_OK;
}

int seq_allpairs(const cfgsim_corpus *c, int64_t us, int64_t ue, const cfgsim_params *p, double *d_lin,
                 int32_t *iters_lin, int64_t out_base, int &launch_no, cudaStream_t st) {
  if (ue <= us) return CFGSIM_OK;
  return p->precision == CFGSIM_FP32 ? seq_allpairs_t<float>(c, us, ue, p, d_lin, iters_lin, out_base, launch_no, st)
                                     : seq_allpairs_t<double>(c, us, ue, p, d_lin, iters_lin, out_base, launch_no, st);
}

int check_params(const cfgsim_params *p) {
  if (!p) return fail(CFGSIM_ERR_ARG, "params is NULL");
  if (!(p->alpha > 0.0 && p->alpha < 1.0))
    return fail(CFGSIM_ERR_ARG, "alpha must be in (0, 1)");  // similarity.py:129-130
  if (!(p->tol > 0.0)) return fail(CFGSIM_ERR_ARG, "tol must be positive");
  if (p->max_iter < 1) return fail(CFGSIM_ERR_ARG, "max_iter must be >= 1");
  if (p->precision != CFGSIM_FP64 && p->precision != CFGSIM_FP32)
    return fail(CFGSIM_ERR_ARG, "precision must be CFGSIM_FP64 or CFGSIM_FP32");
  return CFGSIM_OK;
}

int set_device(int dev) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(CFGSIM_ERR_NODEVICE, "no CUDA device: cfgsim has no CPU path");
  }
  if (dev < 0 || dev >= n) return fail(CFGSIM_ERR_ARG, "device index out of range");
  CU(cudaSetDevice(dev));
  cudaDeviceProp pr;
  CU(cudaGetDeviceProperties(&pr, dev));
  if (pr.major != 10) return fail(CFGSIM_ERR_NODEVICE, "cfgsim is built for sm_100a only");
  return CFGSIM_OK;
}

// Host copy of a large buffer on several threads (pinned staging -> user memory).
void parallel_memcpy(void *dst, const void *src, size_t n) {
  const size_t kChunk = 4u << 20;
  const int nt = (int)std::min<size_t>(std::min<size_t>(8, std::max(1u, std::thread::hardware_concurrency())),
                                       (n + kChunk - 1) / kChunk);
  if (nt <= 1) {
    memcpy(dst, src, n);
    return;
  }
  const size_t per = (n + nt - 1) / nt;
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; t++) {
    const size_t a = per * t, b = std::min(n, a + per);
    if (a < b) pool.emplace_back([=] { memcpy((char *)dst + a, (const char *)src + a, b - a); });
  }
  memcpy(dst, src, std::min(n, per));
  for (auto &th : pool) th.join();
}

// Output staging: device pointers are used in place; host pointers get a
// device buffer (pooled in the device's Scratch when the caller passes one)
// and, from 1 MB up, a pinned host buffer the D2H copy lands in (then one
// multi-threaded memcpy into the caller's memory after the stream sync).
struct OutStage {
  void *user = nullptr;
  size_t bytes = 0;
  DBuf own;
  void *dev = nullptr;
  bool host = false;
  PinBuf *pin = nullptr;
  cudaError_t prepare(void *u, size_t b, cudaStream_t st = 0, DBuf *pool = nullptr, PinBuf *pinb = nullptr) {
    user = u;
    bytes = b;
    if (!u) return cudaSuccess;
    if (is_device_ptr(u)) {
      dev = u;
      return cudaSuccess;
    }
    host = true;
    cudaError_t e;
    if (pool) {
      e = grow_buf(*pool, std::max<size_t>(b, 16), st);
      dev = pool->p;
    } else {
      e = own.alloc(b);
      dev = own.p;
    }
    if (e == cudaSuccess && pinb && b >= (1u << 20) && !is_pinned_host_ptr(u)) {
      e = pinb->grow(b);  // (the previous user of this buffer synchronised before returning)
      if (e == cudaSuccess) pin = pinb;
    }  // (a page-locked caller buffer receives the D2H directly: no staging copy)
    return e;
  }
  cudaError_t finish(cudaStream_t st) {
    if (user && host) return cudaMemcpyAsync(pin ? pin->p : user, dev, bytes, cudaMemcpyDeviceToHost, st);
    return cudaSuccess;
  }
  void complete() {  // after the stream synchronised
    if (user && host && pin) parallel_memcpy(user, pin->p, bytes);
  }
};

// Pair-list execution shared by isorank_pairs / nearest / overflow reruns.
// ia/ib/slot are host arrays.  Outputs are device arrays indexed by slot.
int run_list(const cfgsim_corpus *A, const cfgsim_corpus *B, const std::vector<int32_t> &ia,
             const std::vector<int32_t> &ib, const std::vector<int64_t> &slot, const cfgsim_params *p,
             double *d, double *W, int32_t *iters, uint8_t *conv, double *X, int32_t *match,
             const double *x0, cudaStream_t st, int mode = 0);  // mode: 1 dense lists, 2 force_m

int handle_overflow(const cfgsim_corpus *A, const cfgsim_corpus *B, const PairWork &work,
                    const cfgsim_params *p, double *d, double *W, int32_t *iters, uint8_t *conv,
                    Scratch &S, cudaStream_t st) {
  int32_t cnt = 0;
  CU(cudaMemcpyAsync(&cnt, S.ovf_count.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (cnt == 0) return CFGSIM_OK;
  if (cnt > S.ovf_cap) return fail(CFGSIM_ERR_CUDA, "overflow list capacity exceeded");
  std::vector<int64_t> recs(cnt);
  CU(cudaMemcpy(recs.data(), S.ovf_list.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost));
  // kind 0: list overflow -> dense-bound lists; kind 1: ambiguous stop -> force_m
  std::vector<int32_t> ia[2], ib[2];
  std::vector<int64_t> sl[2];
  for (int64_t rec : recs) {
    const int kind = (int)(rec & 1);
    const int dir = (int)((rec >> 1) & 1);
    if (work.mode == WORK_LIST)
      return fail(CFGSIM_ERR_CUDA, "internal: list overflow must be handled by run_list");
    const int64_t u = rec >> 2;  // absolute unit
    const auto &rs = A->row_start;
    const int a = (int)(std::upper_bound(rs.begin(), rs.end(), u) - rs.begin()) - 1;
    const int b = a + (int)(u - rs[a]);
    int g1 = A->perm[a], g2 = A->perm[b];
    if (work.ordered ? dir != 0 : g1 > g2) std::swap(g1, g2);
    ia[kind].push_back(g1);
    ib[kind].push_back(g2);
    sl[kind].push_back(work.ordered ? 2 * (u - work.out_base) + dir : (u - work.out_base));
  }
  CU(cudaMemsetAsync(S.ovf_count.p, 0, sizeof(int32_t), st));
  for (int kind = 0; kind < 2; kind++)
    if (int rc = run_list(A, B, ia[kind], ib[kind], sl[kind], p, d, W, iters, conv, nullptr, nullptr,
                          nullptr, st, kind == 0 ? 1 : 2))
      return rc;
  return CFGSIM_OK;
}

int ensure_scratch(Scratch &S, int64_t ovf_cap) {
  if (!S.counters.p) {
    CU(S.counters.alloc(sizeof(unsigned long long) * 64));
    CU(S.ovf_count.alloc(sizeof(int32_t)));
    CU(cudaMemset(S.ovf_count.p, 0, sizeof(int32_t)));
  }
  if (S.ovf_cap < ovf_cap) {
    CU(S.ovf_list.alloc(sizeof(int64_t) * ovf_cap));
    S.ovf_cap = ovf_cap;
  }
  return CFGSIM_OK;
}

int run_list(const cfgsim_corpus *A, const cfgsim_corpus *B, const std::vector<int32_t> &ia,
             const std::vector<int32_t> &ib, const std::vector<int64_t> &slot, const cfgsim_params *p,
             double *d, double *W, int32_t *iters, uint8_t *conv, double *X, int32_t *match,
             const double *x0, cudaStream_t st, int mode) {
  const bool dense_lists = (mode & 1) != 0;
  const int64_t n = (int64_t)ia.size();
  if (n == 0) return CFGSIM_OK;
  Scratch &S = scratch_for(A->device);
  if (int rc = ensure_scratch(S, 1 << 16)) return rc;
  // bucket by launch plan: low-rank kernel -> one launch per exact N;
  // general kernel -> per (tier, occupancy), within a bucket by descending N
  const bool lr = (x0 == nullptr) && use_lowrank();
  std::vector<Plan> plans;
  std::vector<std::vector<int64_t>> bucket;
  for (int64_t q = 0; q < n; q++) {
    const int N = std::max(A->n_nodes[ia[q]], B->n_nodes[ib[q]]);
    Plan pl;
    if (lr) {
      if (lr_tier(p->precision, N)) {
        pl.ti = N;  // bucket key: one low-rank launch per exact N
      } else if (N <= kBigNmax) {
        pl.ti = kBigKey + big_kb(N);  // large-N kernel, one launch per sort class
      } else {
        return fail(CFGSIM_ERR_ARG, "pair size N=" + std::to_string(N) + " exceeds 1024");
      }
      pl.occ = 0;
    } else {
      pl = plan_for(p->precision, N, dense_lists);
    }
    if (pl.ti < 0)
      return fail(CFGSIM_ERR_ARG, "pair size N=" + std::to_string(N) +
                                      " exceeds the on-chip tiers of this build");
    size_t bi = 0;
    while (bi < plans.size() && !plans[bi].same_launch(pl)) bi++;
    if (bi == plans.size()) {
      plans.push_back(pl);
      bucket.emplace_back();
    }
    bucket[bi].push_back(q);
  }
  for (size_t bi = 0; bi < bucket.size(); bi++) {
    auto &bk = bucket[bi];
    const int ti = plans[bi].ti;
    std::stable_sort(bk.begin(), bk.end(), [&](int64_t x, int64_t y) {
      return std::max(A->n_nodes[ia[x]], B->n_nodes[ib[x]]) >
             std::max(A->n_nodes[ia[y]], B->n_nodes[ib[y]]);
    });
    int nlim = 0;
    std::vector<int32_t> hia(bk.size()), hib(bk.size());
    std::vector<int64_t> hsl(bk.size());
    for (size_t q = 0; q < bk.size(); q++) {
      hia[q] = ia[bk[q]];
      hib[q] = ib[bk[q]];
      hsl[q] = slot[bk[q]];
      nlim = std::max(nlim, std::max(A->n_nodes[hia[q]], B->n_nodes[hib[q]]));
    }
    DBuf dia, dib, dsl;
    CU(dia.alloc(sizeof(int32_t) * bk.size()));
    CU(dib.alloc(sizeof(int32_t) * bk.size()));
    CU(dsl.alloc(sizeof(int64_t) * bk.size()));
    CU(cudaMemcpyAsync(dia.p, hia.data(), sizeof(int32_t) * bk.size(), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dib.p, hib.data(), sizeof(int32_t) * bk.size(), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dsl.p, hsl.data(), sizeof(int64_t) * bk.size(), cudaMemcpyHostToDevice, st));
    PairWork w{};
    w.mode = WORK_LIST;
    w.n_items = (int64_t)bk.size();
    w.ia = dia.as<int32_t>();
    w.ib = dib.as<int32_t>();
    w.slot = dsl.as<int64_t>();
    PairOut o{};
    o.d = d;
    o.W = W;
    o.iters = iters;
    o.conv = conv;
    o.X = X;
    o.match = match;
    o.x0 = x0;
    o.ovf_count = S.ovf_count.as<int32_t>();
    o.ovf_list = S.ovf_list.as<int64_t>();
    o.ovf_cap = (int32_t)S.ovf_cap;
    if (lr && ti >= kBigKey) {
      if (int rc = big_launch(p->precision, nlim, A->dev(), B->dev(), w, o, p,
                              S.counters.as<unsigned long long>() + (bi % 32), st))
        return rc;
      if (int rc = big_status(S, st)) return rc;
    } else if (lr) {
      if (int rc = lr_launch(p->precision, nlim, dense_lists, A->dev(), B->dev(), w, o, p,
                             S.counters.as<unsigned long long>() + (bi % 32), st))
        return rc;
    } else {
      const int cap2 = cap_for(p->precision, plans[bi], nlim, dense_lists);
      if (int rc = launch_tier(p->precision, ti, nlim, cap2, A->dev(), B->dev(), w, o, p,
                               S.counters.as<unsigned long long>() + (bi % 32), st, (mode & 2) ? 1 : 0))
        return rc;
    }
    // overflowed / ambiguous items are re-run (dense-bound lists / force_m)
    int32_t cnt = 0;
    CU(cudaMemcpyAsync(&cnt, S.ovf_count.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (cnt > 0) {
      if (cnt > S.ovf_cap) return fail(CFGSIM_ERR_CUDA, "overflow list capacity exceeded");
      std::vector<int64_t> recs(cnt);
      CU(cudaMemcpy(recs.data(), S.ovf_list.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost));
      CU(cudaMemset(S.ovf_count.p, 0, sizeof(int32_t)));
      std::vector<int32_t> ra[2], rb[2];
      std::vector<int64_t> rs[2];
      for (int64_t rec : recs) {
        const int kind = (int)(rec & 1);
        const int64_t item = rec >> 2;
        ra[kind].push_back(hia[item]);
        rb[kind].push_back(hib[item]);
        rs[kind].push_back(hsl[item]);
      }
      if (!ra[0].empty() && dense_lists) return fail(CFGSIM_ERR_CUDA, "internal: dense-bound lists overflowed");
      if (!ra[1].empty() && (mode & 2)) return fail(CFGSIM_ERR_CUDA, "internal: ambiguous stop with force_m");
      if (int rc = run_list(A, B, ra[0], rb[0], rs[0], p, d, W, iters, conv, X, match, x0, st, mode | 1)) return rc;
      if (int rc = run_list(A, B, ra[1], rb[1], rs[1], p, d, W, iters, conv, X, match, x0, st, mode | 2)) return rc;
    }
  }
  return CFGSIM_OK;
}

__global__ void scatter_kernel(int64_t n_units, int32_t K, const int64_t *row_start,
                               const int32_t *perm, int32_t ordered, const double *d_lin,
                               const int32_t *it_lin, double *d_mat, int32_t *it_mat) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n_units;
       u += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = K - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (row_start[mid] <= u) lo = mid; else hi = mid - 1;
    }
    const int a = lo, b = a + (int)(u - row_start[a]);
    const int64_t ga = perm[a], gb = perm[b];
    const double d0 = ordered ? d_lin[2 * u] : d_lin[u];
    const double d1 = (ordered && a != b) ? d_lin[2 * u + 1] : d0;
    d_mat[ga * K + gb] = d0;
    d_mat[gb * K + ga] = d1;
    if (it_mat && it_lin) {
      const int32_t i0 = ordered ? it_lin[2 * u] : it_lin[u];
      const int32_t i1 = (ordered && a != b) ? it_lin[2 * u + 1] : i0;
      it_mat[ga * K + gb] = i0;
      it_mat[gb * K + ga] = i1;
    }
  }
}

// argmin over each row of a (nq x nc) distance block, ties -> lowest column.
__global__ void rowmin_kernel(int32_t nq, int32_t nc, const double *dmat, int64_t col0,
                              double *best_d, int64_t *best_i) {
  const int q = blockIdx.x;
  if (q >= nq) return;
  double bv = INFINITY;
  int64_t bi = INT64_MAX;
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    const double v = dmat[(int64_t)q * nc + c];
    if (v < bv) { bv = v; bi = c; }  // NaN never wins (np.argmin would; pairs never fail here)
  }
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  for (int m = 16; m > 0; m >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, m);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, m);
    if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++)
      if (sv[w] < bv || (sv[w] == bv && si[w] < bi)) { bv = sv[w]; bi = si[w]; }
    best_d[q] = bv;
    best_i[q] = (bi == INT64_MAX) ? -1 : bi + col0;
  }
}

// interpolate_to on the device (matrix.py:74-106), bit-exact.
__global__ void interp_kernel(int n, const double *src, int N, double *dst) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N * N; e += gridDim.x * blockDim.x) {
    const int p = e / N, q = e % N;
    if (n == N) { dst[e] = src[e]; continue; }
    if (n == 1) { dst[e] = src[0]; continue; }
    auto lof = [&](int t, int &l, double &f) {
      const double pos = __ddiv_rn((double)((long long)t * (n - 1)), (double)(N - 1));
      l = (int)floor(pos);
      if (l > n - 2) l = n - 2;
      f = __dsub_rn(pos, (double)l);
    };
    int lp, lq;
    double fp, fq;
    lof(p, lp, fp);
    lof(q, lq, fq);
    const double v00 = src[lp * n + lq], v01 = src[lp * n + lq + 1];
    const double v10 = src[(lp + 1) * n + lq], v11 = src[(lp + 1) * n + lq + 1];
    const double omc = __dsub_rn(1.0, fq);
    const double top = __dadd_rn(__dmul_rn(omc, v00), __dmul_rn(fq, v01));
    const double bot = __dadd_rn(__dmul_rn(omc, v10), __dmul_rn(fq, v11));
    dst[e] = __dadd_rn(__dmul_rn(__dsub_rn(1.0, fp), top), __dmul_rn(fp, bot));
  }
}

int corpus_from_dense(int device, int n, const double *M, cfgsim_corpus **out) {
  std::vector<int32_t> rp(n + 1, 0), col;
  std::vector<double> val;
  for (int r = 0; r < n; r++) {
    for (int c = 0; c < n; c++) {
      const double v = M[(size_t)r * n + c];
      if (v != 0.0) {
        col.push_back(c);
        val.push_back(v);
      }
    }
    rp[r + 1] = (int32_t)col.size();
  }
  const int32_t nn = n;
  const int64_t rpo = 0, nzo = 0;
  return cfgsim_corpus_create(device, 1, &nn, &rpo, rp.data(), &nzo, col.data(), val.data(), out);
}

}  // namespace

namespace {
// Flat-measure launch over a pair list or the upper triangle of one corpus.
int flat_launch(const cfgsim_corpus *A, const cfgsim_corpus *B, FlatWork w, double *out, cudaStream_t st) {
  if (w.n_items <= 0) return CFGSIM_OK;
  w.nlim = std::max(A->max_nodes, B->max_nodes);
  const size_t smem = sizeof(double) * 4 * (size_t)w.nlim;
  if (smem > kMaxSmem) return fail(CFGSIM_ERR_ARG, "flat measures: graph too large for the row buffers");
  CU(cudaFuncSetAttribute((const void *)flat_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev, sms = 0, occ = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)flat_pair_kernel, FLAT_THREADS, smem));
  const int64_t grid = std::min<int64_t>((int64_t)sms * std::max(occ, 1), w.n_items);
  flat_pair_kernel<<<(unsigned)grid, FLAT_THREADS, smem, st>>>(A->dev(), B->dev(), w, out);
  g_launches++;
  CU(cudaGetLastError());
  return CFGSIM_OK;
}

int check_flat(int32_t measure, double p) {
  if (measure < CFGSIM_EUC || measure > CFGSIM_COS) return fail(CFGSIM_ERR_ARG, "unknown flat measure");
  if (measure == CFGSIM_MIN && !(p >= 1.0))
    return fail(CFGSIM_ERR_ORDER, "order p must be >= 1");  // similarity.py:46-47 (BadOrder)
  return CFGSIM_OK;
}
}  // namespace

// ====================================================================== C ABI
namespace {
// Persistent host worker pool for the graph-parallel packing passes (thread
// creation per pass cost ~3-5 ms on a C2-sized corpus, several passes per
// corpus).  One job at a time; the caller participates.
class HostPool {
 public:
  static HostPool &get() {
    static HostPool pool;
    return pool;
  }
  int size() const { return (int)th_.size() + 1; }
  void run(const std::function<void()> &work) {
    std::lock_guard<std::mutex> serial(run_mu_);
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = &work;
      active_ = (int)th_.size();
      gen_++;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return active_ == 0; });
    job_ = nullptr;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : th_) t.join();
  }

 private:
  HostPool() {
    // host packing threads (CFGSIM_HOST_THREADS; default: the CPUs this
    // process may run on, at most 8 — packing a corpus is a few ms of work,
    // and a burst of more threads than the container's CPU quota gets the
    // whole process throttled for a scheduler period)
    const char *e = getenv("CFGSIM_HOST_THREADS");
    int avail = (int)std::thread::hardware_concurrency();
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) avail = CPU_COUNT(&set);
    const int n = e && atoi(e) > 0 ? atoi(e) : std::max(1, std::min(8, avail));
    for (int t = 1; t < n; t++) th_.emplace_back([this] { loop(); });
  }
  void loop() {
    int seen = 0;
    for (;;) {
      const std::function<void()> *j;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        j = job_;
      }
      (*j)();
      std::lock_guard<std::mutex> lk(m_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_, run_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void()> *job_ = nullptr;
  int gen_ = 0, active_ = 0;
  bool stop_ = false;
};

// run f(g) for g in [0, n) on the host cores (graph-parallel packing)
template <typename F>
void parallel_graphs(int n, F f) {
  if (n < 64) {
    for (int g = 0; g < n; g++) f(g);
    return;
  }
  std::atomic<int> next{0};
  const std::function<void()> work = [&]() {
    for (int g0; (g0 = next.fetch_add(32)) < n;)
      for (int g = g0; g < std::min(n, g0 + 32); g++) f(g);
  };
  HostPool::get().run(work);
}

// CSC of every graph (rows ascending within a column), same offsets as the
// CSR; false if a column index is out of range
bool build_csc(int32_t n_graphs, const int32_t *n_nodes, const int64_t *rp_off, const int32_t *rowptr,
               const int64_t *nz_off, const int32_t *col, const double *val, int32_t *cscp, int32_t *crow,
               double *cval, int &bad_graph) {
  std::atomic<int> bad{-1};
  parallel_graphs(n_graphs, [&](int g) {
    const int n = n_nodes[g];
    const int32_t *rp = rowptr + rp_off[g];
    int32_t *cp = cscp + rp_off[g];
    for (int k = 0; k <= n; k++) cp[k] = 0;
    for (int r = 0; r < n; r++)
      for (int32_t q = rp[r]; q < rp[r + 1]; q++) {
        const int cc = col[nz_off[g] + q];
        if (cc < 0 || cc >= n) {
          int e = -1;
          bad.compare_exchange_strong(e, g);
          return;
        }
        cp[cc + 1]++;
      }
    for (int k = 0; k < n; k++) cp[k + 1] += cp[k];
    std::vector<int32_t> fill(cp, cp + n);
    for (int r = 0; r < n; r++)
      for (int32_t q = rp[r]; q < rp[r + 1]; q++) {
        const int cc = col[nz_off[g] + q];
        const int32_t at = fill[cc]++;
        crow[nz_off[g] + at] = r;
        cval[nz_off[g] + at] = val[nz_off[g] + q];
      }
  });
  bad_graph = bad.load();
  return bad_graph < 0;
}

int corpus_create_impl(int32_t device, int32_t n_graphs, const int32_t *n_nodes, const int64_t *rp_off,
                       const int32_t *rowptr, const int64_t *nz_off, const int32_t *col, const double *val,
                       const int32_t *cscp_in, const int32_t *crow_in, const double *cval_in, cfgsim_corpus **out) {
  CFGSIM_NVTX("cfgsim.pack");
  if (!out || n_graphs < 1 || !n_nodes || !rp_off || !rowptr || !nz_off)
    return fail(CFGSIM_ERR_ARG, "bad corpus arguments");
  if (int rc = set_device(device)) return rc;
  auto *c = new cfgsim_corpus();
  c->device = device;
  c->K = n_graphs;
  c->n_nodes.assign(n_nodes, n_nodes + n_graphs);
  int64_t rp_total = 0, nz_total = 0;
  for (int g = 0; g < n_graphs; g++) {
    const int n = n_nodes[g];
    if (n < 1) {
      delete c;
      return fail(CFGSIM_ERR_ARG, "graph with no nodes (EmptyGraph)");
    }
    c->max_nodes = std::max(c->max_nodes, n);
    rp_total = std::max(rp_total, rp_off[g] + n + 1);
    nz_total = std::max(nz_total, nz_off[g] + (int64_t)rowptr[rp_off[g] + n]);
  }
  c->perm.resize(n_graphs);
  std::iota(c->perm.begin(), c->perm.end(), 0);
  std::stable_sort(c->perm.begin(), c->perm.end(),
                   [&](int x, int y) { return n_nodes[x] > n_nodes[y]; });
  c->n_sorted.resize(n_graphs);
  for (int a = 0; a < n_graphs; a++) c->n_sorted[a] = n_nodes[c->perm[a]];
  c->row_start.resize(n_graphs + 1);
  c->row_start[0] = 0;
  for (int a = 0; a < n_graphs; a++) c->row_start[a + 1] = c->row_start[a] + (n_graphs - a);

  // host-side CSC unless the dense packer built it
  std::vector<int32_t> cscp_v, crow_v;
  std::vector<double> cval_v;
  if (!cscp_in) {
    cscp_v.assign(rp_total, 0);
    crow_v.assign(nz_total, 0);
    cval_v.assign(nz_total, 0.0);
    int bad = -1;
    if (!build_csc(n_graphs, n_nodes, rp_off, rowptr, nz_off, col, val, cscp_v.data(), crow_v.data(), cval_v.data(),
                   bad)) {
      delete c;
      return fail(CFGSIM_ERR_ARG, "column index out of range in graph " + std::to_string(bad));
    }
    cscp_in = cscp_v.data();
    crow_in = crow_v.data();
    cval_in = cval_v.data();
  }
  // one allocation, 256-byte aligned sub-arrays, one H2D copy from pinned staging
  struct Part { const void *src; size_t bytes; size_t at; };
  std::vector<Part> parts = {
      {n_nodes, sizeof(int32_t) * n_graphs, 0},          {rp_off, sizeof(int64_t) * n_graphs, 0},
      {rowptr, sizeof(int32_t) * rp_total, 0},           {nz_off, sizeof(int64_t) * n_graphs, 0},
      {col, sizeof(int32_t) * nz_total, 0},              {val, sizeof(double) * nz_total, 0},
      {cscp_in, sizeof(int32_t) * rp_total, 0},          {crow_in, sizeof(int32_t) * nz_total, 0},
      {cval_in, sizeof(double) * nz_total, 0},           {c->perm.data(), sizeof(int32_t) * n_graphs, 0},
      {c->row_start.data(), sizeof(int64_t) * (n_graphs + 1), 0}};
  size_t total = 0;
  for (Part &pt : parts) {
    pt.at = total;
    total += (pt.bytes + 255) & ~size_t(255);
  }
  Scratch &S = scratch_for(device);
  cudaError_t e = cudaSuccess;
  {
    std::lock_guard<std::recursive_mutex> lk(S.mu);
    const size_t want = std::max<size_t>(total, 256);
    int best = -1;
    for (int q = 0; q < (int)S.corpus_free.size(); q++)
      if (S.corpus_free[q].first >= want && S.corpus_free[q].first <= 2 * want + (1u << 20) &&
          (best < 0 || S.corpus_free[q].first < S.corpus_free[best].first))
        best = q;
    if (best >= 0) {
      c->d_all.p = S.corpus_free[best].second;
      c->d_all.n = S.corpus_free[best].first;
      S.corpus_free.erase(S.corpus_free.begin() + best);
    } else {
      e = c->d_all.alloc(want);
    }
  }
  if (e == cudaSuccess) {
    std::lock_guard<std::recursive_mutex> lk(S.mu);
    e = S.pin_in.grow(total);
    if (e == cudaSuccess) {
      unsigned char *h = (unsigned char *)S.pin_in.p;
      for (const Part &pt : parts)
        if (pt.bytes) memcpy(h + pt.at, pt.src, pt.bytes);
      e = cudaMemcpy(c->d_all.p, h, total, cudaMemcpyHostToDevice);
    }
  }
  if (e != cudaSuccess) {
    delete c;
    return fail(e == cudaErrorMemoryAllocation ? CFGSIM_ERR_NOMEM : CFGSIM_ERR_CUDA,
                std::string("corpus upload: ") + cudaGetErrorString(e));
  }
  unsigned char *base = (unsigned char *)c->d_all.p;
  c->d_n = (const int32_t *)(base + parts[0].at);
  c->d_rp_off = (const int64_t *)(base + parts[1].at);
  c->d_rowptr = (const int32_t *)(base + parts[2].at);
  c->d_nz_off = (const int64_t *)(base + parts[3].at);
  c->d_col = (const int32_t *)(base + parts[4].at);
  c->d_val = (const double *)(base + parts[5].at);
  c->d_cscp = (const int32_t *)(base + parts[6].at);
  c->d_csc_row = (const int32_t *)(base + parts[7].at);
  c->d_csc_val = (const double *)(base + parts[8].at);
  c->d_perm = (const int32_t *)(base + parts[9].at);
  c->d_row_start = (const int64_t *)(base + parts[10].at);
  for (const Part &pt : parts) c->bytes += (int64_t)pt.bytes;
  *out = c;
  return CFGSIM_OK;
}

}  // namespace

extern "C" {

const char *cfgsim_last_error(void) { return g_err.c_str(); }
int cfgsim_version(void) { return 100; }
int64_t cfgsim_launch_count(void) { return g_launches.load(); }

int cfgsim_device_count(int32_t *n) {
  if (!n) return fail(CFGSIM_ERR_ARG, "n is NULL");
  *n = 0;
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return CFGSIM_OK;
  }
  for (int i = 0; i < c; i++) {
    cudaDeviceProp pr;
    if (cudaGetDeviceProperties(&pr, i) == cudaSuccess && pr.major == 10) (*n)++;
  }
  return CFGSIM_OK;
}

int cfgsim_corpus_create(int32_t device, int32_t n_graphs, const int32_t *n_nodes,
                         const int64_t *rp_off, const int32_t *rowptr, const int64_t *nz_off,
                         const int32_t *col, const double *val, cfgsim_corpus **out) {
  return corpus_create_impl(device, n_graphs, n_nodes, rp_off, rowptr, nz_off, col, val, nullptr, nullptr, nullptr,
                            out);
}

int cfgsim_corpus_create_dense(int32_t device, int32_t n_graphs, const int32_t *n_nodes, const double *const *mats,
                               cfgsim_corpus **out) {
  if (!out || n_graphs < 1 || !n_nodes || !mats) return fail(CFGSIM_ERR_ARG, "bad corpus arguments");
  for (int g = 0; g < n_graphs; g++)
    if (n_nodes[g] < 1 || !mats[g]) return fail(CFGSIM_ERR_ARG, "graph with no nodes (EmptyGraph)");
  // graph-parallel packing: nonzero counts, offsets, then CSR and CSC fills
  std::vector<int64_t> nnz(n_graphs), rp_off(n_graphs), nz_off(n_graphs);
  parallel_graphs(n_graphs, [&](int g) {
    const int n = n_nodes[g];
    const double *m = mats[g];
    int64_t k = 0;
    for (size_t e = 0; e < (size_t)n * n; e++) k += m[e] != 0.0;
    nnz[g] = k;
  });
  int64_t rp_at = 0, nz_at = 0;
  for (int g = 0; g < n_graphs; g++) {
    rp_off[g] = rp_at;
    nz_off[g] = nz_at;
    rp_at += n_nodes[g] + 1;
    nz_at += nnz[g];
  }
  std::vector<int32_t> rowptr(rp_at), col(nz_at), cscp(rp_at), crow(nz_at);
  std::vector<double> val(nz_at), cval(nz_at);
  parallel_graphs(n_graphs, [&](int g) {
    const int n = n_nodes[g];
    const double *m = mats[g];
    int32_t *rp = rowptr.data() + rp_off[g];
    int32_t *cl = col.data() + nz_off[g];
    double *vl = val.data() + nz_off[g];
    int32_t k = 0;
    rp[0] = 0;
    for (int r = 0; r < n; r++) {
      for (int q = 0; q < n; q++) {
        const double v = m[(size_t)r * n + q];
        if (v != 0.0) {
          cl[k] = q;
          vl[k++] = v;
        }
      }
      rp[r + 1] = k;
    }
  });
  int bad = -1;
  build_csc(n_graphs, n_nodes, rp_off.data(), rowptr.data(), nz_off.data(), col.data(), val.data(), cscp.data(),
            crow.data(), cval.data(), bad);
  return corpus_create_impl(device, n_graphs, n_nodes, rp_off.data(), rowptr.data(), nz_off.data(), col.data(),
                            val.data(), cscp.data(), crow.data(), cval.data(), out);
}

int cfgsim_corpus_destroy(cfgsim_corpus *c) {
  if (c) {
    cudaSetDevice(c->device);
    Scratch &S = scratch_for(c->device);
    std::lock_guard<std::recursive_mutex> lk(S.mu);
    S.seq_key.clear();  // a new corpus may reuse this address
    if (c->d_all.p && S.corpus_free.size() < 4) {  // keep the buffer for the next corpus
      S.corpus_free.push_back({c->d_all.n, c->d_all.p});
      c->d_all.p = nullptr;
    }
    delete c;
  }
  return CFGSIM_OK;
}

int cfgsim_corpus_info(const cfgsim_corpus *c, int32_t *n_graphs, int32_t *max_nodes,
                       int64_t *device_bytes) {
  if (!c) return fail(CFGSIM_ERR_ARG, "corpus is NULL");
  if (n_graphs) *n_graphs = c->K;
  if (max_nodes) *max_nodes = c->max_nodes;
  if (device_bytes) *device_bytes = c->bytes;
  return CFGSIM_OK;
}

int cfgsim_isorank_pairs(const cfgsim_corpus *A, const cfgsim_corpus *B, int64_t n_pairs,
                         const int32_t *ia, const int32_t *ib, const cfgsim_params *p, double *d,
                         double *W, int32_t *iters, uint8_t *converged, void *cuda_stream) {
  CFGSIM_NVTX("cfgsim.isorank_pairs");
  if (!A || !B || n_pairs < 0 || (n_pairs && (!ia || !ib)))
    return fail(CFGSIM_ERR_ARG, "bad pair arguments");
  if (int rc = check_params(p)) return rc;
  if (A->device != B->device) return fail(CFGSIM_ERR_ARG, "corpora live on different devices");
  if (int rc = set_device(A->device)) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  DeviceGuard guard(A->device, st);
  std::vector<int32_t> ha(n_pairs), hb(n_pairs);
  if (n_pairs) {
    CU(cudaMemcpyAsync(ha.data(), ia, sizeof(int32_t) * n_pairs, cudaMemcpyDefault, st));
    CU(cudaMemcpyAsync(hb.data(), ib, sizeof(int32_t) * n_pairs, cudaMemcpyDefault, st));
    CU(cudaStreamSynchronize(st));
  }
  for (int64_t q = 0; q < n_pairs; q++)
    if (ha[q] < 0 || ha[q] >= A->K || hb[q] < 0 || hb[q] >= B->K)
      return fail(CFGSIM_ERR_ARG, "pair index out of range");
  std::vector<int64_t> slot(n_pairs);
  std::iota(slot.begin(), slot.end(), 0);
  Scratch &S = scratch_for(A->device);
  OutStage sd, sw, si, sc;
  CU(sd.prepare(d, sizeof(double) * n_pairs, st, &S.pool_out[0], &S.pin_out[0]));
  CU(sw.prepare(W, sizeof(double) * n_pairs, st, &S.pool_out[1], &S.pin_out[1]));
  CU(si.prepare(iters, sizeof(int32_t) * n_pairs, st, &S.pool_out[2], &S.pin_out[2]));
  CU(sc.prepare(converged, sizeof(uint8_t) * n_pairs, st, &S.pool_out[3], &S.pin_out[3]));
  if (int rc = run_list(A, B, ha, hb, slot, p, (double *)sd.dev, (double *)sw.dev,
                        (int32_t *)si.dev, (uint8_t *)sc.dev, nullptr, nullptr, nullptr, st))
    return rc;
  CU(cudaGetLastError());
  CU(sd.finish(st));
  CU(sw.finish(st));
  CU(si.finish(st));
  CU(sc.finish(st));
  CU(cudaStreamSynchronize(st));
  sd.complete();
  sw.complete();
  si.complete();
  sc.complete();
  return CFGSIM_OK;
}

namespace {
// alpha^m by sequential products (the large-N sweeps' ak), m = 0..kmax
__global__ void big_apow_kernel(double alpha, int kmax, double *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double a = 1.0;
    for (int m = 0; m <= kmax; m++) {
      out[m] = a;
      a *= alpha;
    }
  }
}

int big_hist_min_rows() {  // CFGSIM_BIG_HIST_ROWS: rows a size group needs for history mode
  static const int v = [] {
    const char *e = getenv("CFGSIM_BIG_HIST_ROWS");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  return v;
}

bool use_bighist() {  // CFGSIM_BIG_HIST=0: per-pair sweeps in the large-N kernel (A/B)
  static const bool on = [] {
    const char *e = getenv("CFGSIM_BIG_HIST");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// One size group of large-N rows (rows ra.. of size N) over units [u0, u1):
// the sequences of every partner graph (sorted positions ra .. K-1) at size
// N once (isorank_seqbig_kernel), then the pair kernel in history mode.
// Device-resident tables, no host round trip (capturable).
int bighist_group(const cfgsim_corpus *c, int ra, int N, int64_t u0, int64_t u1, PairWork w, const PairOut &o,
                  const cfgsim_params *p, Scratch &S, unsigned long long *ctr, cudaStream_t st) {
  const int64_t ncombo = c->K - ra;
  const double tol = p->tol;
  const int kcap = big_kcap(p->alpha, tol, p->max_iter);
  const int64_t stride = (int64_t)(kcap + 1) * big_hpitch(N);
  CU(grow_buf(S.seq_u, sizeof(double) * (size_t)(ncombo * stride), st));
  CU(grow_buf(S.seq_d, sizeof(double) * (size_t)(ncombo * (kcap + 1)), st));
  CU(grow_buf(S.seq_apow, sizeof(double) * (size_t)(kcap + 2), st));
  S.seq_key.clear();  // the shared combo buffers are rewritten
  big_apow_kernel<<<1, 32, 0, st>>>(p->alpha, kcap + 1, S.seq_apow.as<double>());
  g_launches++;
  // stage: the group's sequences
  BigParams sp{};
  sp.alpha = p->alpha;
  sp.tol = tol;
  sp.eps = 1e-6;
  sp.max_iter = p->max_iter;
  sp.kcap = kcap;
  sp.nlim = N;
  SeqBigCombos cb{};
  cb.n = ncombo;
  cb.N = N;
  cb.g = c->d_perm + ra;
  cb.stride = stride;
  cb.hu = S.seq_u.as<double>();
  cb.hd = S.seq_d.as<double>();
  const size_t smem = big_smem_layout<double>(N).total;
  const void *fk = (const void *)isorank_seqbig_kernel<8>;
  int dev, sms = 0, occ = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CU(cached_occupancy(fk, BIG_THREADS, smem, &occ));
  if (occ < 1) return fail(CFGSIM_ERR_CUDA, "sequence kernel cannot be resident");
  const int64_t grid = std::min<int64_t>((int64_t)sms * occ, ncombo);
  DevCorpus dc = c->dev();
  void *args[] = {(void *)&dc, (void *)&cb, (void *)&sp};
  CU(cudaLaunchKernel(fk, dim3((unsigned)grid), dim3(BIG_THREADS), args, smem, st));
  g_launches++;
  // the group's pairs: the large-N kernel in history mode
  w.u0 = u0;
  w.n_items = u1 - u0;
  BigParams hist{};
  hist.hu = S.seq_u.as<double>();
  hist.hd = S.seq_d.as<double>();
  hist.hstride = stride;
  hist.hcbase = -(int64_t)ra;
  hist.hapow = S.seq_apow.as<double>();
  return big_launch(CFGSIM_FP64, N, dc, dc, w, o, p, ctr, st, nullptr, 0, 0, &hist);
}
}  // namespace

int cfgsim_allpairs_units(const cfgsim_corpus *c, int64_t *n_units) {
  if (!c || !n_units) return fail(CFGSIM_ERR_ARG, "bad arguments");
  *n_units = c->row_start[c->K];
  return CFGSIM_OK;
}

int cfgsim_allpairs_split(const cfgsim_corpus *c, int32_t world, int64_t *bounds) {
  if (!c || world < 1 || !bounds) return fail(CFGSIM_ERR_ARG, "bad arguments");
  // cost of unit (a, b >= a) = unit_cost_us(N), N = n_sorted[a] (rows sorted
  // by n desc): the measured per-tier cost model of cost_model.h
  std::vector<double> cum(c->K + 1, 0.0);
  for (int a = 0; a < c->K; a++) cum[a + 1] = cum[a] + (double)(c->K - a) * unit_cost_us(c->n_sorted[a]);
  const double total = cum[c->K];
  bounds[0] = 0;
  for (int r = 1; r < world; r++) {
    const double target = total * r / world;
    const int a = (int)(std::upper_bound(cum.begin(), cum.end(), target) - cum.begin()) - 1;
    const double per = unit_cost_us(c->n_sorted[std::min(a, c->K - 1)]);
    int64_t u = c->row_start[a] + (int64_t)std::ceil((target - cum[a]) / per);
    u = std::min<int64_t>(u, c->row_start[std::min(a + 1, c->K)]);
    bounds[r] = std::max(u, bounds[r - 1]);
  }
  bounds[world] = c->row_start[c->K];
  return CFGSIM_OK;
}

int cfgsim_allpairs_range(const cfgsim_corpus *c, int64_t u0, int64_t u1, int32_t ordered,
                          const cfgsim_params *p, double *d_lin, int32_t *iters_lin,
                          void *cuda_stream) {
  CFGSIM_NVTX("cfgsim.allpairs_range");
  if (!c || u0 < 0 || u1 < u0 || u1 > c->row_start[c->K])
    return fail(CFGSIM_ERR_ARG, "bad unit range");
  if (int rc = check_params(p)) return rc;
  if (int rc = set_device(c->device)) return rc;
  if (u1 == u0) return CFGSIM_OK;
  cudaGetLastError();  // (a stale non-sticky error of an unrelated earlier call is not this call's)
  if ((d_lin && !is_device_ptr(d_lin)) || (iters_lin && !is_device_ptr(iters_lin)))
    return fail(CFGSIM_ERR_ARG, "allpairs_range outputs must be device pointers");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  DeviceGuard guard(c->device, st);
  Scratch &S = scratch_for(c->device);
  if (int rc = ensure_scratch(S, 1 << 16)) return rc;
  const bool lr = use_lowrank();
  // rows of the size-sorted corpus are contiguous per N: split the unit range
  // into runs of rows with one launch plan (low-rank: one N per launch).
  int a = (int)(std::upper_bound(c->row_start.begin(), c->row_start.end(), u0) -
                c->row_start.begin()) - 1;
  int64_t u = u0;
  int launch_no = 0;
  PairWork w{};
  w.mode = WORK_TRIANGLE;
  w.ordered = ordered;
  w.out_base = u0;
  w.row_start = c->d_row_start;
  w.perm = c->d_perm;
  w.K = c->K;
  PairOut o{};
  o.d = d_lin;
  o.iters = iters_lin;
  o.ovf_count = S.ovf_count.as<int32_t>();
  o.ovf_list = S.ovf_list.as<int64_t>();
  o.ovf_cap = (int32_t)S.ovf_cap;
  // unordered units of rows with N <= 64 (a suffix of the size-sorted rows):
  // two-stage path; the loop below covers the rest
  int64_t u_end = u1;
  const double tol_eff = p->precision == CFGSIM_FP32 ? std::max(p->tol, p->tol_fp32) : p->tol;
  if (lr && !ordered && use_twostage() && big_kcap(p->alpha, tol_eff, p->max_iter) <= 512) {
    int as = a;
    while (as < c->K && c->n_sorted[as] > kSeqNmax) as++;
    const int64_t us = std::max(u0, as < c->K ? c->row_start[as] : u1);
    if (us < u1) {
      if (int rc = seq_allpairs(c, us, u1, p, d_lin, iters_lin, u0, launch_no, st)) return rc;
      u_end = us;
    }
  }
  while (u < u_end) {
    const int N = c->n_sorted[a];
    int a_end = a;
    Plan pl;
    const bool big = lr && !lr_tier(p->precision, N);
    if (big) {
      if (N > kBigNmax) return fail(CFGSIM_ERR_ARG, "pair size N=" + std::to_string(N) + " exceeds 1024");
      while (a_end + 1 < c->K && !lr_tier(p->precision, c->n_sorted[a_end + 1]) &&
             big_kb(c->n_sorted[a_end + 1]) == big_kb(N))
        a_end++;
    } else if (lr) {
      while (a_end + 1 < c->K && c->n_sorted[a_end + 1] == N) a_end++;
    } else {
      pl = plan_for(p->precision, N, false);
      if (pl.ti < 0)
        return fail(CFGSIM_ERR_ARG, "pair size N=" + std::to_string(N) +
                                        " exceeds the on-chip tiers of this build");
      while (a_end + 1 < c->K && plan_for(p->precision, c->n_sorted[a_end + 1], false).same_launch(pl))
        a_end++;
    }
    const int64_t seg_end = std::min(u_end, c->row_start[a_end + 1]);
    w.n_items = seg_end - u;
    w.u0 = u;
    unsigned long long *ctr = S.counters.as<unsigned long long>() + (launch_no % 64);
    if (big && p->precision == CFGSIM_FP64 && !ordered && use_bighist()) {
      // size groups with many rows share per-(graph, N) sequences (history
      // mode); runs of small groups go through the per-pair kernel as one
      // launch (a group's sequences cost about as much as its rows' own
      // sweeps until it has several rows)
      int64_t pu0 = -1, pu1 = -1;  // pending per-pair unit range
      auto flush = [&]() -> int {
        if (pu1 > pu0 && pu0 >= 0) {
          PairWork w2 = w;
          w2.u0 = pu0;
          w2.n_items = pu1 - pu0;
          unsigned long long *pctr = S.counters.as<unsigned long long>() + (launch_no++ % 64);
          const int nl = c->n_sorted[std::upper_bound(c->row_start.begin(), c->row_start.end(), pu0) -
                                     c->row_start.begin() - 1];
          if (int rc = big_launch(p->precision, nl, c->dev(), c->dev(), w2, o, p, pctr, st)) return rc;
        }
        pu0 = pu1 = -1;
        return CFGSIM_OK;
      };
      for (int ga = a; ga <= a_end;) {
        int gb = ga;
        while (gb + 1 <= a_end && c->n_sorted[gb + 1] == c->n_sorted[ga]) gb++;
        const int64_t gu0 = std::max(u, c->row_start[ga]), gu1 = std::min(seg_end, c->row_start[gb + 1]);
        if (gu1 > gu0) {
          if (gb - ga + 1 >= big_hist_min_rows()) {
            if (int rc = flush()) return rc;
            unsigned long long *gctr = S.counters.as<unsigned long long>() + (launch_no++ % 64);
            if (int rc = bighist_group(c, ga, c->n_sorted[ga], gu0, gu1, w, o, p, S, gctr, st)) return rc;
          } else {
            if (pu0 < 0) pu0 = gu0;
            pu1 = gu1;
          }
        }
        ga = gb + 1;
      }
      if (int rc = flush()) return rc;
    } else if (big) {
      if (int rc = big_launch(p->precision, N, c->dev(), c->dev(), w, o, p, ctr, st)) return rc;
    } else {
      // per-pair kernels with operator lists: records of overflowed /
      // ambiguous pairs, handled after every launch so that the list never
      // needs more than one launch's units (a full C5 rank range has
      // millions of mid-N pairs)
      if (stream_capturing(st))  // overflow records need a host round trip per launch
        return fail(CFGSIM_ERR_ARG, "allpairs_range: N=" + std::to_string(N) +
                                        " rows use list kernels, which cannot be captured into a CUDA graph");
      if (S.ovf_cap < w.n_items) {
        CU(cudaStreamSynchronize(st));
        if (int rc = ensure_scratch(S, w.n_items)) return rc;
        o.ovf_list = S.ovf_list.as<int64_t>();
        o.ovf_cap = (int32_t)std::min<int64_t>(S.ovf_cap, INT32_MAX);
      }
      if (lr) {
        if (int rc = lr_launch(p->precision, N, false, c->dev(), c->dev(), w, o, p, ctr, st)) return rc;
      } else if (int rc = launch_tier(p->precision, pl.ti, N, cap_for(p->precision, pl, N, false), c->dev(),
                                      c->dev(), w, o, p, ctr, st)) {
        return rc;
      }
      if (int rc = handle_overflow(c, c, w, p, d_lin, nullptr, iters_lin, nullptr, S, st)) return rc;
    }
    launch_no++;
    u = seg_end;
    a = a_end + 1;
  }
  // overflowed / ambiguous pairs of the per-pair kernels (records hold
  // absolute units); the two-stage path alone needs no host round trip
  if (u_end > u0) {
    // (under capture only large-N kernels ran — list kernels refuse it — and
    // they leave no overflow records)
    if (!stream_capturing(st))
      if (int rc = handle_overflow(c, c, w, p, d_lin, nullptr, iters_lin, nullptr, S, st)) return rc;
    if (int rc = big_status(S, st)) return rc;
  }
  CU(cudaGetLastError());
  return CFGSIM_OK;
}

int cfgsim_allpairs_scatter(const cfgsim_corpus *c, int32_t ordered, const double *d_lin,
                            const int32_t *iters_lin, double *d_mat, int32_t *iters_mat,
                            void *cuda_stream) {
  CFGSIM_NVTX("cfgsim.gather");
  if (!c || !d_lin || !d_mat) return fail(CFGSIM_ERR_ARG, "bad arguments");
  if (int rc = set_device(c->device)) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int64_t nu = c->row_start[c->K];
  g_launches++;
  scatter_kernel<<<1184, 256, 0, st>>>(nu, c->K, c->d_row_start,
                                       c->d_perm, ordered, d_lin, iters_lin, d_mat,
                                       iters_mat);
  CU(cudaGetLastError());
  return CFGSIM_OK;
}

int cfgsim_allpairs(const cfgsim_corpus *c, int32_t ordered, const cfgsim_params *p,
                    double *d_mat, int32_t *iters_mat, void *cuda_stream) {
  CFGSIM_NVTX("cfgsim.allpairs");
  if (!c || !d_mat) return fail(CFGSIM_ERR_ARG, "bad arguments");
  if (int rc = check_params(p)) return rc;
  if (int rc = set_device(c->device)) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  DeviceGuard guard(c->device, st);
  const int64_t nu = c->row_start[c->K];
  const int64_t slots = ordered ? 2 * nu : nu;
  Scratch &S = scratch_for(c->device);
  CU(grow_buf(S.pool_lin, sizeof(double) * slots, st));
  if (iters_mat) CU(grow_buf(S.pool_it, sizeof(int32_t) * slots, st));
  double *dl = S.pool_lin.as<double>();
  int32_t *il = iters_mat ? S.pool_it.as<int32_t>() : nullptr;
  const size_t KK = (size_t)c->K * c->K;
  OutStage sd, si;
  CU(sd.prepare(d_mat, sizeof(double) * KK, st, &S.pool_out[0], &S.pin_out[0]));
  CU(si.prepare(iters_mat, sizeof(int32_t) * KK, st, &S.pool_out[1], &S.pin_out[1]));
  if (int rc = cfgsim_allpairs_range(c, 0, nu, ordered, p, dl, il, st)) return rc;
  if (int rc = cfgsim_allpairs_scatter(c, ordered, dl, il, (double *)sd.dev, (int32_t *)si.dev, st)) return rc;
  CU(sd.finish(st));
  CU(si.finish(st));
  CU(cudaStreamSynchronize(st));
  sd.complete();
  si.complete();
  return CFGSIM_OK;
}

// isorank_align(start=...) beyond the on-chip general kernel (N <= 1024):
// the reference iteration with X in HBM (isorank_start.cuh), then the
// large-N kernel's sort + matching on the final X.  fp64.
int start_big_single(const cfgsim_corpus *ca, const cfgsim_corpus *cb, int N, const cfgsim_params *p,
                     const double *dx0, double *dd, double *dw, int32_t *di, uint8_t *dc, double *dX, int32_t *dm) {
  CFGSIM_NVTX("cfgsim.start_large_n");
  if (N > kBigNmax) return fail(CFGSIM_ERR_ARG, "pair size N=" + std::to_string(N) + " exceeds 1024");
  const int64_t nn = (int64_t)N * N;
  const int64_t chunk = 8192;
  const int nparts = (int)((nn + chunk - 1) / chunk);
  DBuf opA, opB, xa, fb, tb, part, dpart, dlt, dia, dib, dsl;
  CU(opA.alloc(sizeof(double) * nn));
  CU(opB.alloc(sizeof(double) * nn));
  CU(xa.alloc(sizeof(double) * nn));
  CU(fb.alloc(sizeof(double) * nn));
  CU(tb.alloc(sizeof(double) * nn));
  CU(part.alloc(sizeof(double) * nparts));
  CU(dpart.alloc(sizeof(double) * nparts));
  CU(dlt.alloc(sizeof(double)));
  cudaStream_t st = 0;
  const DevCorpus A = ca->dev(), B = cb->dev();
  start_dense_op_kernel<<<(N + 7) / 8, 256, 0, st>>>(A, 0, N, opA.as<double>());
  start_dense_op_kernel<<<(N + 7) / 8, 256, 0, st>>>(B, 0, N, opB.as<double>());
  g_launches += 2;
  CU(cudaMemcpyAsync(xa.p, dx0, sizeof(double) * nn, cudaMemcpyDeviceToDevice, st));
  const dim3 gg((N + SG_T - 1) / SG_T, (N + SG_T - 1) / SG_T);
  const double u = 1.0 / (double)nn;  // np.full(n * n, 1.0 / (n * n))
  int k = 0, conv = 0;
  for (k = 1; k <= p->max_iter; k++) {
    start_gemm_kernel<<<gg, 256, 0, st>>>(opA.as<double>(), xa.as<double>(), tb.as<double>(), N, 1);  // A'^T X
    start_gemm_kernel<<<gg, 256, 0, st>>>(tb.as<double>(), opB.as<double>(), fb.as<double>(), N, 0);  // (.) B'
    start_update_kernel<<<nparts, SR_T, 0, st>>>(fb.as<double>(), nn, p->alpha, u, chunk, part.as<double>());
    start_norm_kernel<<<nparts, SR_T, 0, st>>>(fb.as<double>(), xa.as<double>(), nn, chunk, part.as<double>(), nparts,
                                               dpart.as<double>());
    start_delta_kernel<<<1, 32, 0, st>>>(dpart.as<double>(), nparts, dlt.as<double>());
    g_launches += 5;
    CU(cudaGetLastError());
    double delta = 0.0;
    CU(cudaMemcpyAsync(&delta, dlt.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    std::swap(xa.p, fb.p);  // x = fresh (similarity.py:143)
    if (delta < p->tol) {   // :144
      conv = 1;
      break;
    }
  }
  if (k > p->max_iter) k = p->max_iter;
  if (dX) CU(cudaMemcpyAsync(dX, xa.p, sizeof(double) * nn, cudaMemcpyDeviceToDevice, st));
  int32_t zero = 0;
  int64_t zslot = 0;
  CU(dia.alloc(sizeof(int32_t)));
  CU(dib.alloc(sizeof(int32_t)));
  CU(dsl.alloc(sizeof(int64_t)));
  CU(cudaMemcpyAsync(dia.p, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dib.p, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dsl.p, &zslot, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  PairWork w{};
  w.mode = WORK_LIST;
  w.n_items = 1;
  w.ia = dia.as<int32_t>();
  w.ib = dib.as<int32_t>();
  w.slot = dsl.as<int64_t>();
  PairOut o{};
  o.d = dd;
  o.W = dw;
  o.iters = di;
  o.conv = dc;
  o.match = dm;
  Scratch &S = scratch_for(ca->device);
  if (int rc = ensure_scratch(S, 1 << 16)) return rc;
  cfgsim_params p64 = *p;
  p64.precision = CFGSIM_FP64;
  if (int rc = big_launch(CFGSIM_FP64, N, A, B, w, o, &p64, S.counters.as<unsigned long long>(), st, xa.as<double>(), k,
                          conv))
    return rc;
  if (int rc = big_status(S, st)) return rc;
  CU(cudaStreamSynchronize(st));
  return CFGSIM_OK;
}

int cfgsim_isorank_single(int32_t device, int32_t na, const double *A, int32_t nb,
                          const double *B, const cfgsim_params *p, const double *x0,
                          double *X_out, int32_t *match_out, double *d, double *W,
                          int32_t *iters, uint8_t *converged) {
  CFGSIM_NVTX("cfgsim.isorank_single");
  if (na < 1 || nb < 1 || !A || !B) return fail(CFGSIM_ERR_ARG, "bad matrices");
  if (int rc = check_params(p)) return rc;
  if (int rc = set_device(device)) return rc;
  DeviceGuard guard(device, 0);
  cfgsim_corpus *ca = nullptr, *cb = nullptr;
  if (int rc = corpus_from_dense(device, na, A, &ca)) return rc;
  if (int rc = corpus_from_dense(device, nb, B, &cb)) {
    cfgsim_corpus_destroy(ca);
    return rc;
  }
  const int N = std::max(na, nb);
  DBuf dd, dw, di, dc, dX, dm, dx0;
  int rc = CFGSIM_OK;
  auto cu = [&](cudaError_t e) {
    if (e != cudaSuccess && rc == CFGSIM_OK)
      rc = fail(CFGSIM_ERR_CUDA, std::string("single: ") + cudaGetErrorString(e));
    return e == cudaSuccess;
  };
  cu(dd.alloc(8));
  cu(dw.alloc(8));
  cu(di.alloc(4));
  cu(dc.alloc(1));
  cu(dX.alloc(sizeof(double) * N * N));
  cu(dm.alloc(sizeof(int32_t) * N));
  if (x0) {
    cu(dx0.alloc(sizeof(double) * N * N));
    cu(cudaMemcpy(dx0.p, x0, sizeof(double) * N * N, cudaMemcpyHostToDevice));
  }
  if (rc == CFGSIM_OK && x0 && plan_for(p->precision, N, false).ti < 0) {
    // a start vector beyond the on-chip general kernel's tiers
    rc = start_big_single(ca, cb, N, p, dx0.as<double>(), dd.as<double>(), dw.as<double>(), di.as<int32_t>(),
                          dc.as<uint8_t>(), dX.as<double>(), dm.as<int32_t>());
  } else if (rc == CFGSIM_OK) {
    std::vector<int32_t> ia{0}, ib{0};
    std::vector<int64_t> sl{0};
    rc = run_list(ca, cb, ia, ib, sl, p, dd.as<double>(), dw.as<double>(), di.as<int32_t>(),
                  dc.as<uint8_t>(), dX.as<double>(), dm.as<int32_t>(), dx0.as<double>(), 0);
  }
  if (rc == CFGSIM_OK) cu(cudaDeviceSynchronize());
  if (rc == CFGSIM_OK) {
    if (d) cu(cudaMemcpy(d, dd.p, 8, cudaMemcpyDeviceToHost));
    if (W) cu(cudaMemcpy(W, dw.p, 8, cudaMemcpyDeviceToHost));
    if (iters) cu(cudaMemcpy(iters, di.p, 4, cudaMemcpyDeviceToHost));
    if (converged) cu(cudaMemcpy(converged, dc.p, 1, cudaMemcpyDeviceToHost));
    if (X_out) cu(cudaMemcpy(X_out, dX.p, sizeof(double) * N * N, cudaMemcpyDeviceToHost));
    if (match_out) cu(cudaMemcpy(match_out, dm.p, sizeof(int32_t) * N, cudaMemcpyDeviceToHost));
  }
  cfgsim_corpus_destroy(ca);
  cfgsim_corpus_destroy(cb);
  return rc;
}

int cfgsim_nearest(const cfgsim_corpus *Q, const cfgsim_corpus *C, int32_t c0, int32_t c1,
                   const cfgsim_params *p, double *best_d, int64_t *best_idx, void *cuda_stream) {
  CFGSIM_NVTX("cfgsim.nearest");
  if (!Q || !C || c0 < 0 || c1 > C->K || c1 <= c0 || !best_d || !best_idx)
    return fail(CFGSIM_ERR_ARG, "bad nearest arguments");
  if (int rc = check_params(p)) return rc;
  if (Q->device != C->device) return fail(CFGSIM_ERR_ARG, "corpora live on different devices");
  if (int rc = set_device(Q->device)) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  DeviceGuard guard(Q->device, st);
  const int32_t nq = Q->K, nc = c1 - c0;
  Scratch &S = scratch_for(Q->device);
  OutStage sd, si;
  CU(sd.prepare(best_d, sizeof(double) * nq, st, &S.pool_out[0], &S.pin_out[0]));
  CU(si.prepare(best_idx, sizeof(int64_t) * nq, st, &S.pool_out[1], &S.pin_out[1]));
  if (int rc = ensure_scratch(S, 1 << 16)) return rc;
  // corpus range in ascending node count (stable): pairs are enumerated as
  // rectangles of equal N = max(n_q, n_c) (two per distinct N) in these orders
  std::vector<int32_t> cs(nc);
  std::iota(cs.begin(), cs.end(), c0);
  std::stable_sort(cs.begin(), cs.end(), [&](int x, int y) { return C->n_nodes[x] < C->n_nodes[y]; });
  DBuf dcs;
  CU(dcs.alloc(sizeof(int32_t) * nc));
  CU(cudaMemcpyAsync(dcs.p, cs.data(), sizeof(int32_t) * nc, cudaMemcpyHostToDevice, st));
  // query blocks: one block's distance matrix stays <= 2^28 entries (2 GiB)
  const int64_t per_block = std::max<int64_t>(1, ((int64_t)1 << 28) / nc);
  DBuf dqs;
  CU(grow_buf(S.pool_lin, sizeof(double) * std::min<int64_t>(nq, per_block) * nc, st));  // the distance block
  double *const dmp = S.pool_lin.as<double>();
  CU(dqs.alloc(sizeof(int32_t) * std::min<int64_t>(nq, per_block)));
  const bool lr = use_lowrank();
  for (int32_t q0 = 0; q0 < nq; q0 += (int32_t)per_block) {
    const int32_t q1 = (int32_t)std::min<int64_t>(nq, q0 + per_block);
    const int32_t bq = q1 - q0;
    std::vector<int32_t> qs(bq);
    std::iota(qs.begin(), qs.end(), q0);
    std::stable_sort(qs.begin(), qs.end(), [&](int x, int y) { return Q->n_nodes[x] < Q->n_nodes[y]; });
    CU(cudaMemcpyAsync(dqs.p, qs.data(), sizeof(int32_t) * bq, cudaMemcpyHostToDevice, st));
    // launches: one per exact N (low-rank kernel) / per sort class (large-N kernel)
    struct Launch { int key, nlim; std::vector<int32_t> rects; };
    std::vector<Launch> launches;
    std::vector<int> ns;
    for (int x : qs) ns.push_back(Q->n_nodes[x]);
    for (int x : cs) ns.push_back(C->n_nodes[x]);
    std::sort(ns.begin(), ns.end());
    ns.erase(std::unique(ns.begin(), ns.end()), ns.end());
    auto qcount = [&](int n, bool le) {  // queries with n_q < n (le: <= n)
      return (int32_t)((le ? std::upper_bound(qs.begin(), qs.end(), n, [&](int v, int x) { return v < Q->n_nodes[x]; })
                           : std::lower_bound(qs.begin(), qs.end(), n, [&](int x, int v) { return Q->n_nodes[x] < v; })) -
                       qs.begin());
    };
    auto ccount = [&](int n, bool le) {
      return (int32_t)((le ? std::upper_bound(cs.begin(), cs.end(), n, [&](int v, int x) { return v < C->n_nodes[x]; })
                           : std::lower_bound(cs.begin(), cs.end(), n, [&](int x, int v) { return C->n_nodes[x] < v; })) -
                       cs.begin());
    };
    // N <= 64: two-stage path (per-(graph, N) sequences, then per-pair rank-K products)
    const double tol_eff = p->precision == CFGSIM_FP32 ? std::max(p->tol, p->tol_fp32) : p->tol;
    const bool two = lr && use_twostage() && big_kcap(p->alpha, tol_eff, p->max_iter) <= 512;
    int launch_no2 = 0;
    if (two) {
      std::vector<int> small;
      for (int N : ns)
        if (N <= kSeqNmax) small.push_back(N);
      const int rc = p->precision == CFGSIM_FP32
                         ? seq_nearest_t<float>(Q, C, qs, cs, dqs.as<int32_t>(), dcs.as<int32_t>(), q0, c0, nc, small,
                                                p, dmp, launch_no2, st)
                         : seq_nearest_t<double>(Q, C, qs, cs, dqs.as<int32_t>(), dcs.as<int32_t>(), q0, c0, nc, small,
                                                 p, dmp, launch_no2, st);
      if (rc) return rc;
    }
    for (int N : ns) {
      if (two && N <= kSeqNmax) continue;
      if (N > kBigNmax) return fail(CFGSIM_ERR_ARG, "pair size N=" + std::to_string(N) + " exceeds 1024");
      const int key = (!lr || lr_tier(p->precision, N)) ? N : kBigKey + big_kb(N);
      if (launches.empty() || launches.back().key != key) launches.push_back({key, N, {}});
      Launch &L = launches.back();
      L.nlim = std::max(L.nlim, N);
      const int32_t qlt = qcount(N, false), qle = qcount(N, true);
      const int32_t clt = ccount(N, false), cle = ccount(N, true);
      if (qle > qlt && cle > 0) L.rects.insert(L.rects.end(), {qlt, qle, 0, cle});   // n_q == N, n_c <= N
      if (qlt > 0 && cle > clt) L.rects.insert(L.rects.end(), {0, qlt, clt, cle});   // n_q < N, n_c == N
    }
    for (size_t li = 0; li < launches.size(); li++) {
      Launch &L = launches[li];
      const int nr = (int)L.rects.size() / 4;
      if (nr == 0) continue;
      std::vector<int64_t> rs(nr + 1, 0);
      for (int r = 0; r < nr; r++)
        rs[r + 1] = rs[r] + (int64_t)(L.rects[4 * r + 1] - L.rects[4 * r]) * (L.rects[4 * r + 3] - L.rects[4 * r + 2]);
      DBuf drs, drect;
      CU(drs.alloc(sizeof(int64_t) * (nr + 1)));
      CU(drect.alloc(sizeof(int32_t) * 4 * nr));
      CU(cudaMemcpyAsync(drs.p, rs.data(), sizeof(int64_t) * (nr + 1), cudaMemcpyHostToDevice, st));
      CU(cudaMemcpyAsync(drect.p, L.rects.data(), sizeof(int32_t) * 4 * nr, cudaMemcpyHostToDevice, st));
      PairWork w{};
      w.mode = WORK_RECT;
      w.n_items = rs[nr];
      w.nrect = nr;
      w.rect_start = drs.as<int64_t>();
      w.rect = drect.as<int32_t>();
      w.qperm = dqs.as<int32_t>();
      w.cperm = dcs.as<int32_t>();
      w.qbase = q0;
      w.cbase = c0;
      w.ld = nc;
      PairOut o{};
      o.d = dmp;
      o.ovf_count = S.ovf_count.as<int32_t>();
      o.ovf_list = S.ovf_list.as<int64_t>();
      o.ovf_cap = (int32_t)S.ovf_cap;
      unsigned long long *ctr = S.counters.as<unsigned long long>() + (li % 64);
      if (L.key >= kBigKey) {
        if (int rc = big_launch(p->precision, L.nlim, Q->dev(), C->dev(), w, o, p, ctr, st)) return rc;
      } else if (lr) {
        if (int rc = lr_launch(p->precision, L.nlim, false, Q->dev(), C->dev(), w, o, p, ctr, st)) return rc;
      } else {
        const Plan pl = plan_for(p->precision, L.nlim, false);
        if (pl.ti < 0) return fail(CFGSIM_ERR_ARG, "pair size N=" + std::to_string(L.nlim) + " exceeds the on-chip tiers");
        if (int rc = launch_tier(p->precision, pl.ti, L.nlim, cap_for(p->precision, pl, L.nlim, false), Q->dev(),
                                 C->dev(), w, o, p, ctr, st))
          return rc;
      }
      // overflowed / ambiguous items of this launch: re-run as pair lists
      int32_t cnt = 0;
      CU(cudaMemcpyAsync(&cnt, S.ovf_count.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      if (cnt > 0) {
        if (cnt > S.ovf_cap) return fail(CFGSIM_ERR_CUDA, "overflow list capacity exceeded");
        std::vector<int64_t> recs(cnt);
        CU(cudaMemcpy(recs.data(), S.ovf_list.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost));
        CU(cudaMemset(S.ovf_count.p, 0, sizeof(int32_t)));
        std::vector<int32_t> ra[2], rb[2];
        std::vector<int64_t> rsl[2];
        for (int64_t rec : recs) {
          const int kind = (int)(rec & 1);
          const int64_t item = rec >> 2;
          const int r = (int)(std::upper_bound(rs.begin(), rs.end(), item) - rs.begin()) - 1;
          const int32_t *R = L.rects.data() + 4 * r;
          const int64_t loc = item - rs[r];
          const int wdt = R[3] - R[2];
          const int gq = qs[R[0] + (int)(loc / wdt)], gc = cs[R[2] + (int)(loc % wdt)];
          ra[kind].push_back(gq);
          rb[kind].push_back(gc);
          rsl[kind].push_back((int64_t)(gq - q0) * nc + (gc - c0));
        }
        for (int kind = 0; kind < 2; kind++)
          if (int rc = run_list(Q, C, ra[kind], rb[kind], rsl[kind], p, dmp, nullptr, nullptr, nullptr,
                                nullptr, nullptr, nullptr, st, kind == 0 ? 1 : 2))
            return rc;
      }
    }
    if (int rc = big_status(S, st)) return rc;
    rowmin_kernel<<<bq, 256, 0, st>>>(bq, nc, dmp, c0, (double *)sd.dev + q0, (int64_t *)si.dev + q0);
    CU(cudaGetLastError());
  }
  CU(sd.finish(st));
  CU(si.finish(st));
  CU(cudaStreamSynchronize(st));
  sd.complete();
  si.complete();
  return CFGSIM_OK;
}

int cfgsim_interpolate(int32_t device, int32_t n, const double *src, int32_t target, double *dst) {
  if (n < 1 || target < n || !src || !dst) return fail(CFGSIM_ERR_ARG, "bad interpolation arguments");
  if (int rc = set_device(device)) return rc;
  DBuf s, d;
  CU(s.alloc(sizeof(double) * n * n));
  CU(d.alloc(sizeof(double) * target * target));
  CU(cudaMemcpy(s.p, src, sizeof(double) * n * n, cudaMemcpyHostToDevice));
  interp_kernel<<<(target * target + 255) / 256, 256>>>(n, s.as<double>(), target, d.as<double>());
  CU(cudaGetLastError());
  CU(cudaMemcpy(dst, d.p, sizeof(double) * target * target, cudaMemcpyDeviceToHost));
  return CFGSIM_OK;
}

int cfgsim_flat_pairs(const cfgsim_corpus *A, const cfgsim_corpus *B, int64_t n_pairs, const int32_t *ia,
                      const int32_t *ib, int32_t measure, double p, double *out, void *cuda_stream) {
  CFGSIM_NVTX("cfgsim.flat_pairs");
  if (!A || !B || n_pairs < 0 || (n_pairs && (!ia || !ib || !out))) return fail(CFGSIM_ERR_ARG, "bad pair arguments");
  if (A->device != B->device) return fail(CFGSIM_ERR_ARG, "corpora live on different devices");
  if (int rc = set_device(A->device)) return rc;
  const bool bad_order = measure == CFGSIM_MIN && !(p >= 1.0);
  if (!bad_order)
    if (int rc = check_flat(measure, p)) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  std::vector<int32_t> ha(n_pairs), hb(n_pairs);
  if (n_pairs) {
    CU(cudaMemcpyAsync(ha.data(), ia, sizeof(int32_t) * n_pairs, cudaMemcpyDefault, st));
    CU(cudaMemcpyAsync(hb.data(), ib, sizeof(int32_t) * n_pairs, cudaMemcpyDefault, st));
    CU(cudaStreamSynchronize(st));
  }
  for (int64_t q = 0; q < n_pairs; q++)
    if (ha[q] < 0 || ha[q] >= A->K || hb[q] < 0 || hb[q] >= B->K) return fail(CFGSIM_ERR_ARG, "pair index out of range");
  DBuf dia, dib;
  CU(dia.alloc(sizeof(int32_t) * std::max<int64_t>(n_pairs, 1)));
  CU(dib.alloc(sizeof(int32_t) * std::max<int64_t>(n_pairs, 1)));
  CU(cudaMemcpyAsync(dia.p, ha.data(), sizeof(int32_t) * n_pairs, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dib.p, hb.data(), sizeof(int32_t) * n_pairs, cudaMemcpyHostToDevice, st));
  OutStage so;
  CU(so.prepare(out, sizeof(double) * n_pairs));
  FlatWork w{};
  w.mode = 0;
  w.n_items = n_pairs;
  w.ia = dia.as<int32_t>();
  w.ib = dib.as<int32_t>();
  w.measure = measure;
  w.p = p;
  if (int rc = flat_launch(A, B, w, (double *)so.dev, st)) return rc;
  CU(so.finish(st));
  CU(cudaStreamSynchronize(st));
  return CFGSIM_OK;
}

int cfgsim_flat_allpairs(const cfgsim_corpus *c, int32_t measure, double p, double *d_mat, void *cuda_stream) {
  CFGSIM_NVTX("cfgsim.flat_allpairs");
  if (!c || !d_mat) return fail(CFGSIM_ERR_ARG, "bad arguments");
  if (int rc = set_device(c->device)) return rc;
  const bool bad_order = measure == CFGSIM_MIN && !(p >= 1.0);
  if (!bad_order)
    if (int rc = check_flat(measure, p)) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const size_t KK = (size_t)c->K * c->K;
  OutStage so;
  CU(so.prepare(d_mat, sizeof(double) * KK));
  CU(cudaMemsetAsync(so.dev, 0, sizeof(double) * KK, st));  // definitional zero diagonal (similarity.py:248-255)
  FlatWork w{};
  w.mode = 1;
  w.n_items = (int64_t)c->K * (c->K - 1) / 2;
  w.K = c->K;
  w.measure = measure;
  w.p = p;  // p < 1: every pair is NaN (BadOrder caught per pair, :243-246)
  if (int rc = flat_launch(c, c, w, (double *)so.dev, st)) return rc;
  CU(so.finish(st));
  CU(cudaStreamSynchronize(st));
  return CFGSIM_OK;
}

int cfgsim_flat_all_allpairs(const cfgsim_corpus *c, double p, double *d_mats, void *cuda_stream) {
  CFGSIM_NVTX("cfgsim.flat_all_allpairs");
  if (!c || !d_mats) return fail(CFGSIM_ERR_ARG, "bad arguments");
  if (int rc = set_device(c->device)) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const size_t KK = (size_t)c->K * c->K;
  OutStage so;
  CU(so.prepare(d_mats, 5 * sizeof(double) * KK));
  CU(cudaMemsetAsync(so.dev, 0, 5 * sizeof(double) * KK, st));  // definitional zero diagonals (similarity.py:248-255)
  FlatWork w{};
  w.mode = 1;
  w.n_items = (int64_t)c->K * (c->K - 1) / 2;
  w.K = c->K;
  w.measure = FLAT_ALL;
  w.p = p;  // p < 1: the MIN matrix is all NaN (BadOrder caught per pair, :243-246)
  w.out_stride = (int64_t)KK;
  if (int rc = flat_launch(c, c, w, (double *)so.dev, st)) return rc;
  CU(so.finish(st));
  CU(cudaStreamSynchronize(st));
  return CFGSIM_OK;
}

namespace {
// fp64 peak probes (the roofline denominator, measured in the same process
// and at the same clocks as the bench): independent accumulator chains, so
// the pipe, not latency, limits.  Not part of any alignment path.
__global__ void probe_dmma_kernel(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int t = 0; t < 8; t++) c[t][0] = c[t][1] = t;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int t = 0; t < 8; t++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  double s = 0;
  for (int t = 0; t < 8; t++) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void probe_dfma_kernel(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int t = 0; t < 16; t++) c[t] = t;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int t = 0; t < 16; t++) c[t] = fma(a, b, c[t]);
  double s = 0;
  for (int t = 0; t < 16; t++) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

int cfgsim_host_alloc(int64_t bytes, void **ptr) {
  if (!ptr || bytes < 0) return fail(CFGSIM_ERR_ARG, "bad arguments");
  *ptr = nullptr;
  if (bytes == 0) return CFGSIM_OK;
  CU(cudaHostAlloc(ptr, (size_t)bytes, cudaHostAllocPortable));
  return CFGSIM_OK;
}

int cfgsim_host_free(void *ptr) {
  if (ptr) CU(cudaFreeHost(ptr));
  return CFGSIM_OK;
}

int cfgsim_probe_fp64(int32_t device, double *mma_tflops, double *fma_tflops) {
  if (int rc = set_device(device)) return rc;
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int blocks = sms * 8, threads = 256, iters = 2048;
  DBuf out;
  CU(out.alloc(sizeof(double) * blocks * threads));
  cudaStream_t st;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  auto time_it = [&](bool mma, double *res) -> int {
    float best = 1e30f;
    for (int rep = 0; rep < 3; rep++) {
      CU(cudaEventRecord(e0, st));
      if (mma) probe_dmma_kernel<<<blocks, threads, 0, st>>>(out.as<double>(), iters);
      else probe_dfma_kernel<<<blocks, threads, 0, st>>>(out.as<double>(), iters);
      CU(cudaEventRecord(e1, st));
      CU(cudaEventSynchronize(e1));
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    // dmma: 8 mma m8n8k4 (512 flop each) per warp per iteration; dfma: 16 fma (2 flop) per thread
    const double flops = mma ? (double)blocks * (threads / 32) * iters * 8 * 512.0
                             : (double)blocks * threads * iters * 16 * 2.0;
    *res = flops / (best * 1e-3) / 1e12;
    return CFGSIM_OK;
  };
  double m = 0, f = 0;
  int rc = time_it(true, &m);
  if (rc == CFGSIM_OK) rc = time_it(false, &f);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  if (rc) return rc;
  if (mma_tflops) *mma_tflops = m;
  if (fma_tflops) *fma_tflops = f;
  return CFGSIM_OK;
}

int cfgsim_flat_single(int32_t device, int32_t na, const double *A, int32_t nb, const double *B, int32_t measure,
                       double p, double *out) {
  if (na < 1 || nb < 1 || !A || !B || !out) return fail(CFGSIM_ERR_ARG, "bad matrices");
  if (int rc = check_flat(measure, p)) return rc;
  if (int rc = set_device(device)) return rc;
  cfgsim_corpus *ca = nullptr, *cb = nullptr;
  if (int rc = corpus_from_dense(device, na, A, &ca)) return rc;
  if (int rc = corpus_from_dense(device, nb, B, &cb)) {
    cfgsim_corpus_destroy(ca);
    return rc;
  }
  const int32_t zero = 0;
  int rc = cfgsim_flat_pairs(ca, cb, 1, &zero, &zero, measure, p, out, nullptr);
  cfgsim_corpus_destroy(ca);
  cfgsim_corpus_destroy(cb);
  if (rc) return rc;
  if (std::isnan(*out)) return fail(CFGSIM_ERR_DEGENERATE, measure == CFGSIM_JAC
                                                             ? "jaccard undefined for two all-zero matrices"
                                                             : "cosine undefined for an all-zero matrix");
  return CFGSIM_OK;
}

int cfgsim_heatmap_csv(int32_t k, const char *ids, const int64_t *id_off, const double *scores, char *out,
                       int64_t cap, int64_t *len, int32_t threads) {
  // export_heatmap_csv (similarity.py:287-293): header ",id0,id1,...", then
  // per row "id," + cells joined by ",", each "%.6f" or "nan" when not finite;
  // "\n" after every line.  Rows are formatted in parallel, then concatenated.
  if (k < 0 || (k && (!ids || !id_off || !scores)) || !len) return fail(CFGSIM_ERR_ARG, "bad csv arguments");
  const int nt = std::max(1, std::min<int>(threads > 0 ? threads : (int)std::thread::hardware_concurrency(), 256));
  std::vector<std::string> rows(k);
  auto work = [&](int t) {
    char buf[64];
    for (int64_t r = t; r < k; r += nt) {
      std::string &s = rows[r];
      s.reserve((size_t)k * 9 + 32);
      s.append(ids + id_off[r], ids + id_off[r + 1]);
      for (int64_t q = 0; q < k; q++) {
        const double x = scores[r * (int64_t)k + q];
        s.push_back(',');
        if (!std::isfinite(x)) {
          s.append("nan");
        } else {
          const int m = snprintf(buf, sizeof(buf), "%.6f", x);
          s.append(buf, (size_t)m);
        }
      }
      s.push_back('\n');
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; t++) pool.emplace_back(work, t);
  work(0);
  for (auto &th : pool) th.join();
  std::string head = ",";
  for (int64_t r = 0; r < k; r++) {
    if (r) head.push_back(',');
    head.append(ids + id_off[r], ids + id_off[r + 1]);
  }
  head.push_back('\n');
  int64_t total = (int64_t)head.size();
  for (auto &s : rows) total += (int64_t)s.size();
  *len = total;
  if (!out) return CFGSIM_OK;  // size query
  if (cap < total) return fail(CFGSIM_ERR_ARG, "csv buffer too small");
  char *p = out;
  memcpy(p, head.data(), head.size());
  p += head.size();
  for (auto &s : rows) {
    memcpy(p, s.data(), s.size());
    p += s.size();
  }
  return CFGSIM_OK;
}

int cfgsim_ward(int32_t device, int32_t k, int32_t dim, const double *features, int64_t *out_a, int64_t *out_b,
                double *out_d, int64_t *out_size) {
  CFGSIM_NVTX("cfgsim.ward");
  // ward_linkage (cluster.py:88-134) on the GPU: k feature vectors of length
  // dim (row-major host array); k - 1 merges (a < b ids, distance, size).
  if (k < 2 || dim < 0 || (dim && !features) || !out_a || !out_b || !out_d || !out_size)
    return fail(CFGSIM_ERR_ARG, "clustering needs at least 2 vectors");
  if (int rc = set_device(device)) return rc;
  DBuf D, id, sz, rmin, rarg, alive, flag, oa, ob, od, os;
  CU(D.alloc(sizeof(double) * (size_t)k * k));
  CU(id.alloc(sizeof(int64_t) * k));
  CU(sz.alloc(sizeof(int64_t) * k));
  CU(rmin.alloc(sizeof(double) * k));
  CU(rarg.alloc(sizeof(int32_t) * k));
  CU(alive.alloc(k));
  CU(flag.alloc(sizeof(int32_t) * k));
  CU(oa.alloc(sizeof(int64_t) * k));
  CU(ob.alloc(sizeof(int64_t) * k));
  CU(od.alloc(sizeof(double) * k));
  CU(os.alloc(sizeof(int64_t) * k));
  // Initial squared distances exactly as cluster.py:109-113 evaluates them:
  // sum((x - y) ** 2 for ...) — libm pow(d, 2.0) (float ** 2 in CPython; not
  // always the rounded product) summed by Python's sum(): 0 + first term, then
  // Neumaier-compensated addition (CPython >= 3.12).  Host threads; the
  // O(K^2 dim) pass is small next to the merge loop's K^2 updates.
  {
    std::vector<double> Dh((size_t)k * k, 0.0);
    const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), 64));
    auto work = [&](int t) {
      for (int64_t i = t; i < k; i += nt)
        for (int64_t j = i + 1; j < k; j++) {
          const double *x = features + i * dim, *y = features + j * dim;
          double f = 0.0, cmp = 0.0;
          for (int q = 0; q < dim; q++) {
            const double v = std::pow(x[q] - y[q], 2.0);
            if (q == 0) { f = v; continue; }  // int 0 + float: exact
            const double tt = f + v;
            if (std::fabs(f) >= std::fabs(v)) cmp += (f - tt) + v;
            else cmp += (v - tt) + f;
            f = tt;
          }
          if (cmp != 0.0 && std::isfinite(cmp)) f += cmp;
          Dh[(size_t)i * k + j] = f;
          Dh[(size_t)j * k + i] = f;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; t++) pool.emplace_back(work, t);
    work(0);
    for (auto &th : pool) th.join();
    CU(cudaMemcpy(D.p, Dh.data(), sizeof(double) * (size_t)k * k, cudaMemcpyHostToDevice));
  }
  WardState ws;
  ws.K = k;
  ws.D = D.as<double>();
  ws.id = id.as<int64_t>();
  ws.size = sz.as<int64_t>();
  ws.rmin = rmin.as<double>();
  ws.rarg = rarg.as<int32_t>();
  ws.alive = alive.as<uint8_t>();
  ws.flag = flag.as<int32_t>();
  ws.out_a = oa.as<int64_t>();
  ws.out_b = ob.as<int64_t>();
  ws.out_size = os.as<int64_t>();
  ws.out_d = od.as<double>();
  ward_kernel<<<1, WARD_THREADS>>>(ws);
  g_launches += 2;
  CU(cudaGetLastError());
  CU(cudaMemcpy(out_a, oa.p, sizeof(int64_t) * (k - 1), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(out_b, ob.p, sizeof(int64_t) * (k - 1), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(out_d, od.p, sizeof(double) * (k - 1), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(out_size, os.p, sizeof(int64_t) * (k - 1), cudaMemcpyDeviceToHost));
  return CFGSIM_OK;
}

}  // extern "C"
