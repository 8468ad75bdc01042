/*
 * cfgsim — B200-native IsoRank CFG-pair similarity (C ABI).
 *
 * Drop-in boundary for the reference's ISO measure path
 * (/root/reference/pkg/src/sasscfg, pure Python).  The reference has no FFI
 * layer; each entry point below replaces the Python function cited, and the
 * Python package paper_1707_02423_b200 binds them with ctypes
 * (INTEGRATION.md shows the binding a sasscfg maintainer would add).
 *
 * Conventions
 *  - every function returns int status (CFGSIM_OK == 0); no C++ exception
 *    crosses the ABI; cfgsim_last_error() returns a thread-local message.
 *  - plain pointers and sizes only.  Arrays marked [host|device] may be
 *    either; the library detects device pointers (cudaPointerGetAttributes)
 *    and stages host arrays itself.  Calls that touch a host output
 *    synchronise the stream before returning; all-device calls are
 *    stream-ordered and asynchronous.
 *  - results are bitwise deterministic: independent of stream, launch
 *    order, tile, grid size or device count.
 *  - threading: any host thread may call any function.  The library keeps
 *    per-device scratch (work counters, overflow lists, combo tables) shared
 *    by all handles on that device; calls that use it are serialised per
 *    device (a mutex for host threads, plus an event so a call's stream
 *    waits for the previous call's stream work).  A corpus handle is
 *    read-only after creation and may be used by several threads; destroy
 *    it only after every call using it has returned and its stream work
 *    has completed.  While a stream is being captured into a CUDA graph the
 *    cross-stream event ordering is skipped: replay the graph on one stream
 *    (or order it yourself) against other library calls.
 *
 * Packed corpus (CSR of the raw TransitionMatrix.entries, matrix.py:24-42):
 *  graph g has n_nodes[g] rows; its row pointer is
 *  rowptr[rp_off[g] .. rp_off[g] + n_nodes[g]] (local, starts at 0); its
 *  column indices / values are col[nz_off[g] + e], val[nz_off[g] + e].
 *  Values must be finite and >= 0 (matrix.py:35-36).
 */
#ifndef CFGSIM_H
#define CFGSIM_H

#include <stdint.h>

#if defined(__GNUC__)
#define CFGSIM_API __attribute__((visibility("default")))
#else
#define CFGSIM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CFGSIM_OK 0
#define CFGSIM_ERR_ARG 1      /* bad argument (reference: ValueError)          */
#define CFGSIM_ERR_DIM 2      /* unequal sizes (reference: DimMismatch)         */
#define CFGSIM_ERR_CUDA 3     /* CUDA runtime / launch failure                  */
#define CFGSIM_ERR_NOMEM 4    /* device allocation failed                       */
#define CFGSIM_ERR_NODEVICE 5 /* no usable sm_100 device: there is no CPU path  */
#define CFGSIM_ERR_DEGENERATE 6 /* measure undefined (reference: DegenerateInput) */
#define CFGSIM_ERR_ORDER 7    /* Minkowski order p < 1 (reference: BadOrder)    */
/* loader errors (errors.py:10-65) */
#define CFGSIM_ERR_LISTING_SYNTAX 8   /* ListingSyntaxError(line_no, reason)     */
#define CFGSIM_ERR_UNRESOLVED_LABEL 9 /* UnresolvedLabel                         */
#define CFGSIM_ERR_PROFILE_SYNTAX 10  /* ProfileSyntaxError(line_no, reason)     */
#define CFGSIM_ERR_DUPLICATE_KERNEL 11 /* DuplicateKernel                        */
#define CFGSIM_ERR_EMPTY_GRAPH 12     /* EmptyGraph                              */
#define CFGSIM_ERR_CORPUS 13          /* CorpusError (no profile for the kernel) */
#define CFGSIM_ERR_VALUE 14           /* ValueError from KernelProfile checks    */
#define CFGSIM_ERR_INDEX 15           /* IndexError (time_ns / calls without a value) */

/* transition-matrix modes (matrix.py:17-19) */
#define CFGSIM_MODE_ROW_STOCHASTIC 0
#define CFGSIM_MODE_GLOBAL 1
#define CFGSIM_MODE_RAW_COUNTS 2

/* flat measures (similarity.py:20-66) */
#define CFGSIM_EUC 0
#define CFGSIM_MAN 1
#define CFGSIM_MIN 2
#define CFGSIM_JAC 3
#define CFGSIM_COS 4

#define CFGSIM_FP64 0
#define CFGSIM_FP32 1

typedef struct cfgsim_corpus cfgsim_corpus;

/* alpha/tol/max_iter as isorank_align (similarity.py:111-118, defaults
 * 0.85/1e-9/1000, corpus.py:86-88).  precision: CFGSIM_FP64 reproduces the
 * reference (fp64); CFGSIM_FP32 iterates in fp32 and stops on
 * delta < max(tol, tol_fp32) (fp32 cannot reach 1e-9). */
typedef struct {
  double alpha;
  double tol;
  int32_t max_iter;
  int32_t precision;
  double tol_fp32;
} cfgsim_params;

CFGSIM_API const char *cfgsim_last_error(void);
CFGSIM_API int cfgsim_version(void);
/* Number of sm_100 devices visible; 0 if none (callers must then fail). */
CFGSIM_API int cfgsim_device_count(int32_t *n);

/* Pack + upload a corpus to `device` (replaces the list[TransitionMatrix]
 * that pairwise() walks, similarity.py:229).  Graphs are also ordered by
 * node count internally (tier bucketing). */
CFGSIM_API int cfgsim_corpus_create(int32_t device, int32_t n_graphs, const int32_t *n_nodes,
                         const int64_t *rp_off, const int32_t *rowptr, const int64_t *nz_off,
                         const int32_t *col, const double *val, cfgsim_corpus **out);
/* Same from dense row-major matrices (mats[g]: n_nodes[g]^2 doubles, the
 * TransitionMatrix.entries themselves): the CSR is built natively. */
CFGSIM_API int cfgsim_corpus_create_dense(int32_t device, int32_t n_graphs, const int32_t *n_nodes,
                                          const double *const *mats, cfgsim_corpus **out);
CFGSIM_API int cfgsim_corpus_destroy(cfgsim_corpus *c);
CFGSIM_API int cfgsim_corpus_info(const cfgsim_corpus *c, int32_t *n_graphs, int32_t *max_nodes,
                       int64_t *device_bytes);

/* measure_distance(A[ia[p]], B[ib[p]], MeasureId.ISO) for p < n_pairs
 * (similarity.py:176-189: normalize_pair -> isorank_align ->
 * isorank_distance).  Outputs d (distance in [1,2]), W (matched weight,
 * similarity.py:150), iters, converged; any output may be NULL.
 * A and B must live on the same device.  [host|device] arrays. */
CFGSIM_API int cfgsim_isorank_pairs(const cfgsim_corpus *A, const cfgsim_corpus *B, int64_t n_pairs,
                         const int32_t *ia, const int32_t *ib, const cfgsim_params *p,
                         double *d, double *W, int32_t *iters, uint8_t *converged,
                         void *cuda_stream);

/* All-pairs over one corpus (pairwise(..., MeasureId.ISO), similarity.py:211-246).
 * Work is the upper triangle in size-sorted order: n_units =
 * K(K+1)/2 unordered pairs {i <= j}.  ordered == 0: one alignment per unit,
 * d(j,i) := d(i,j) (ISO symmetry).  ordered == 1: both
 * directions computed separately exactly like the reference's double loop.
 * cfgsim_allpairs_units  -> number of units.
 * cfgsim_allpairs_split  -> world+1 cost-balanced unit boundaries (for
 *                           row-free sharding across GPUs).
 * cfgsim_allpairs_range  -> computes units [u0,u1) into unit-linear outputs
 *                           d_lin/iters_lin ((u1-u0) entries, x2 when ordered;
 *                           [device]).
 * cfgsim_allpairs_scatter-> scatters a full unit-linear vector (all units)
 *                           into the K x K row-major matrix in the caller's
 *                           graph order, both triangles [device].
 * cfgsim_allpairs        -> convenience: range(all) + scatter, [host|device]
 *                           K x K outputs (iters_mat may be NULL). */
CFGSIM_API int cfgsim_allpairs_units(const cfgsim_corpus *c, int64_t *n_units);
CFGSIM_API int cfgsim_allpairs_split(const cfgsim_corpus *c, int32_t world, int64_t *bounds);
CFGSIM_API int cfgsim_allpairs_range(const cfgsim_corpus *c, int64_t u0, int64_t u1, int32_t ordered,
                          const cfgsim_params *p, double *d_lin, int32_t *iters_lin,
                          void *cuda_stream);
CFGSIM_API int cfgsim_allpairs_scatter(const cfgsim_corpus *c, int32_t ordered, const double *d_lin,
                            const int32_t *iters_lin, double *d_mat, int32_t *iters_mat,
                            void *cuda_stream);
CFGSIM_API int cfgsim_allpairs(const cfgsim_corpus *c, int32_t ordered, const cfgsim_params *p,
                    double *d_mat, int32_t *iters_mat, void *cuda_stream);

/* One alignment with full outputs: isorank_align(a, b, alpha, tol, max_iter,
 * start) (similarity.py:111-157) after normalize_pair.  A (na x na), B
 * (nb x nb) dense row-major host arrays; x0 = start/sum(start) (N*N) or
 * NULL; X_out (N*N) and match_out (N) may be NULL.  N = max(na, nb). */
CFGSIM_API int cfgsim_isorank_single(int32_t device, int32_t na, const double *A, int32_t nb,
                          const double *B, const cfgsim_params *p, const double *x0,
                          double *X_out, int32_t *match_out, double *d, double *W,
                          int32_t *iters, uint8_t *converged);

/* Query-vs-corpus best match: for each query q, argmin_j d(Q[q], C[j]) over
 * j in [c0, c1) with ties to the lowest j (np.argmin over a pairwise row).
 * best_idx is the corpus index.  [host|device] outputs. */
CFGSIM_API int cfgsim_nearest(const cfgsim_corpus *Q, const cfgsim_corpus *C, int32_t c0, int32_t c1,
                   const cfgsim_params *p, double *best_d, int64_t *best_idx,
                   void *cuda_stream);

/* interpolate_to(m, target) (matrix.py:74-106), bit-exact, on the device.
 * src n x n, dst target x target, dense row-major host arrays. */
CFGSIM_API int cfgsim_interpolate(int32_t device, int32_t n, const double *src, int32_t target,
                       double *dst);

/* Flat measures after normalize_pair: measure_distance(a, b, EUC|MAN|MIN|JAC|COS,
 * p) (similarity.py:29-66,176-200).  cfgsim_flat_single: dense host inputs;
 * returns CFGSIM_ERR_DEGENERATE where jaccard / cosine are undefined and
 * CFGSIM_ERR_ORDER for minkowski with p < 1.  cfgsim_flat_pairs: batched over
 * two corpora, NaN where undefined.  cfgsim_flat_allpairs: pairwise(...) for a
 * flat measure (similarity.py:247-255): symmetric K x K in the caller's graph
 * order, zero diagonal, NaN for undefined pairs.  [host|device] outputs. */
CFGSIM_API int cfgsim_flat_single(int32_t device, int32_t na, const double *A, int32_t nb, const double *B,
                                  int32_t measure, double p, double *out);
CFGSIM_API int cfgsim_flat_pairs(const cfgsim_corpus *A, const cfgsim_corpus *B, int64_t n_pairs, const int32_t *ia,
                                 const int32_t *ib, int32_t measure, double p, double *out, void *cuda_stream);
CFGSIM_API int cfgsim_flat_allpairs(const cfgsim_corpus *c, int32_t measure, double p, double *d_mat,
                                    void *cuda_stream);
/* `compare --measure all` (cli.py:154-164) for the five flat measures in ONE
 * pass: d_mats = 5 consecutive K x K matrices in the order EUC, MAN, MIN, JAC,
 * COS (CFGSIM_EUC..CFGSIM_COS), each exactly cfgsim_flat_allpairs' output for
 * that measure (the six sums are formed from the same interpolated entries;
 * EUC and JAC share sum (x-y)^2).  [host|device] output. */
CFGSIM_API int cfgsim_flat_all_allpairs(const cfgsim_corpus *c, double p, double *d_mats, void *cuda_stream);

/* Page-locked host memory for result arrays (the Python API returns K x K
 * score matrices in reused pinned buffers: the device results land there by
 * DMA, with no page faults on the host scatter). */
CFGSIM_API int cfgsim_host_alloc(int64_t bytes, void **ptr);
CFGSIM_API int cfgsim_host_free(void *ptr);

/* Diagnostics (not on any alignment path): fp64 mma.sync.m8n8k4 and DFMA
 * throughput of the device in TFLOP/s, measured now (bench.py's roofline
 * denominator, at the clocks of the run). */
CFGSIM_API int cfgsim_probe_fp64(int32_t device, double *mma_tflops, double *fma_tflops);

/* export_heatmap_csv (similarity.py:287-293), native and multi-threaded (host
 * code; the K x K text for K = 20k is ~4 GB): ids = concatenated UTF-8
 * kernel ids, id_off[k+1] their byte offsets, scores K x K row-major.  With
 * out == NULL only *len (bytes) is returned; else out needs cap >= *len.
 * Byte-identical to the reference's f"{x:.6f}" / "nan" formatting. */
CFGSIM_API int cfgsim_heatmap_csv(int32_t k, const char *ids, const int64_t *id_off, const double *scores,
                                  char *out, int64_t cap, int64_t *len, int32_t threads);

/* ward_linkage (cluster.py:88-134) on the GPU, exact (same double arithmetic
 * and tie rule, O(k^2) work): features k x dim row-major [host]; k-1 merges
 * out (ids a < b, leaves 0..k-1, merged k..2k-2; distance; merged size). */
CFGSIM_API int cfgsim_ward(int32_t device, int32_t k, int32_t dim, const double *features, int64_t *out_a,
                           int64_t *out_b, double *out_d, int64_t *out_size);

/* Corpus loader, host code, multi-threaded over kernels:
 * listing text (+ optional profile text) per kernel -> transition matrix in
 * canonical order.  Replaces, per kernel, cli.py:55-74 _load_kernel
 * (parse_listing sass.py:162-221, build_cfg cfg.py:186-259, parse_profiles
 * profile.py:74-151, attribute_profile profile.py:178-233) followed by
 * transition_matrix (matrix.py:45-71), with identical entries and ordering.
 * profiles may be NULL, or hold NULL for kernels without a profile.  All
 * kernels are processed; the return value is the first failing kernel's code
 * (input order) and cfgsim_matrices_status() has every kernel's code, line
 * number and the reference's message.  *out is set whenever the return is not
 * CFGSIM_ERR_ARG / CFGSIM_ERR_NOMEM; free it with cfgsim_matrices_destroy. */
typedef struct cfgsim_matrices cfgsim_matrices;
CFGSIM_API int cfgsim_matrices_from_listings(int32_t count, const char *const *kernel_ids,
                                             const char *const *listings, const int64_t *listing_lens,
                                             const char *const *profiles, const int64_t *profile_lens,
                                             int32_t mode, int32_t n_threads, cfgsim_matrices **out);
/* sizes[count] (0 for failed kernels) and the total number of entries */
CFGSIM_API int cfgsim_matrices_sizes(const cfgsim_matrices *m, int32_t *sizes, int64_t *total_entries);
/* concatenated row-major entries (sum n^2) and canonical orderings (sum n) */
CFGSIM_API int cfgsim_matrices_read(const cfgsim_matrices *m, double *entries, int32_t *orderings);
CFGSIM_API int cfgsim_matrices_status(const cfgsim_matrices *m, int32_t index, int32_t *code, int64_t *line_no,
                                      char *msg, int64_t cap);
CFGSIM_API void cfgsim_matrices_destroy(cfgsim_matrices *m);

/* Number of pair-kernel launches issued by this process so far (bench
 * evidence for gpu_launches). */
CFGSIM_API int64_t cfgsim_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CFGSIM_H */
