/*
 * C restatement of the reference IsoRank pair path — TEST INFRASTRUCTURE ONLY.
 *
 * Reference: /root/reference/pkg/src/sasscfg (pure Python + numpy).
 * Follows, operation by operation and in the same floating-point order where
 * numpy's order is defined:
 *   interpolate_to      matrix.py:74-106   (bilinear; expression order of :104)
 *   normalize_pair      matrix.py:109-114
 *   _row_normalized     similarity.py:85-93 (row sums in numpy pairwise order)
 *   isorank_align       similarity.py:111-157
 *   _greedy_matching    similarity.py:96-108
 *   isorank_distance    similarity.py:160-173
 * The one deliberate change: kron(A',B')^T @ x (similarity.py:133,140, a BLAS
 * dgemv over an N^2 x N^2 matrix) is evaluated as A'^T X B' (X = x reshaped
 * row-major), the same linear map with a different summation order.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -pthread); output
 * oracle/build/liboracle.so.  Only tests/, smoke() and bench.py's CPU arms
 * load it.
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* numpy's DOUBLE_pairwise_sum (umath/loops_utils.h.src), PW_BLOCKSIZE 128.
 * np.sum over a contiguous run uses exactly this order. */
static double pw_sum(const double *a, long n, long stride) {
  if (n < 8) {
    double res = 0.;
    for (long i = 0; i < n; i++) res += a[i * stride];
    return res;
  } else if (n <= 128) {
    double r[8];
    long i;
    for (int k = 0; k < 8; k++) r[k] = a[k * stride];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; k++) r[k] += a[(i + k) * stride];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i * stride];
    return res;
  } else {
    long n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum(a, n2, stride) + pw_sum(a + n2 * stride, n - n2, stride);
  }
}

/* matrix.py:74-106 into dst (N x N, row-major). */
static void interpolate(const double *src, int n, int N, double *dst) {
  if (N == n) {
    memcpy(dst, src, sizeof(double) * (size_t)n * n);
    return;
  }
  if (n == 1) {
    for (long e = 0; e < (long)N * N; e++) dst[e] = src[0];
    return;
  }
  int *lo = (int *)malloc(sizeof(int) * N);
  double *fr = (double *)malloc(sizeof(double) * N);
  for (int p = 0; p < N; p++) {
    double pos = (double)((long)p * (n - 1)) / (double)(N - 1); /* :93 */
    int l = (int)floor(pos);
    if (l > n - 2) l = n - 2; /* :94 */
    lo[p] = l;
    fr[p] = pos - (double)l; /* :95 */
  }
  for (int p = 0; p < N; p++) {
    const double frp = fr[p];
    const double *r0 = src + (long)lo[p] * n, *r1 = src + (long)(lo[p] + 1) * n;
    for (int q = 0; q < N; q++) {
      const double fc = fr[q];
      const int c = lo[q];
      /* :104, left to right */
      double top = (1.0 - fc) * r0[c] + fc * r0[c + 1];
      double bot = (1.0 - fc) * r1[c] + fc * r1[c + 1];
      dst[(long)p * N + q] = (1.0 - frp) * top + frp * bot;
    }
  }
  free(lo);
  free(fr);
}

/* similarity.py:85-93 in place. */
static void row_normalize(double *m, int N) {
  for (int i = 0; i < N; i++) {
    double *row = m + (long)i * N;
    double s = pw_sum(row, N, 1);
    if (s == 0.0) {
      for (int k = 0; k < N; k++) row[k] = 1.0 / N;
    } else {
      for (int k = 0; k < N; k++) row[k] = row[k] / s;
    }
  }
}

/* similarity.py:96-108 */
static void greedy(const double *X, int N, int32_t *match, double *work) {
  memcpy(work, X, sizeof(double) * (size_t)N * N);
  for (int r = 0; r < N; r++) {
    long best = 0;
    double bv = work[0];
    for (long e = 1; e < (long)N * N; e++)
      if (work[e] > bv) { bv = work[e]; best = e; } /* argmax: first occurrence */
    int row = (int)(best / N), col = (int)(best % N);
    match[row] = col;
    for (int k = 0; k < N; k++) work[(long)row * N + k] = -1.0;
    for (int k = 0; k < N; k++) work[(long)k * N + col] = -1.0;
  }
}

/* Core: A, B dense with sizes na, nb; normalize_pair then isorank_align. */
int oracle_iso_pair(int na, const double *A, int nb, const double *B, double alpha, double tol,
                    int max_iter, const double *x0, double *X_out, int32_t *match_out, double *d_out,
                    double *W_out, int32_t *iters_out, uint8_t *conv_out) {
  if (na < 1 || nb < 1 || !(alpha > 0.0 && alpha < 1.0) || max_iter < 1) return 1;
  const int N = na > nb ? na : nb;
  const long NN = (long)N * N;
  double *ap = (double *)malloc(sizeof(double) * NN);
  double *bp = (double *)malloc(sizeof(double) * NN);
  double *x = (double *)malloc(sizeof(double) * NN);
  double *y = (double *)malloc(sizeof(double) * NN);
  double *z = (double *)malloc(sizeof(double) * NN);
  int32_t *match = (int32_t *)malloc(sizeof(int32_t) * N);
  if (!ap || !bp || !x || !y || !z || !match) return 2;

  interpolate(A, na, N, ap); /* normalize_pair, matrix.py:109-114 */
  interpolate(B, nb, N, bp);
  row_normalize(ap, N); /* similarity.py:133 */
  row_normalize(bp, N);

  /* nonzero lists of B' rows (for the second product) */
  long *bnz_ptr = (long *)malloc(sizeof(long) * (N + 1));
  long nnzb = 0;
  for (long e = 0; e < NN; e++) nnzb += bp[e] != 0.0;
  int *bnz_col = (int *)malloc(sizeof(int) * (nnzb + 1));
  double *bnz_val = (double *)malloc(sizeof(double) * (nnzb + 1));
  if (!bnz_ptr || !bnz_col || !bnz_val) return 2;
  nnzb = 0;
  for (int j = 0; j < N; j++) {
    bnz_ptr[j] = nnzb;
    for (int l = 0; l < N; l++)
      if (bp[(long)j * N + l] != 0.0) {
        bnz_col[nnzb] = l;
        bnz_val[nnzb++] = bp[(long)j * N + l];
      }
  }
  bnz_ptr[N] = nnzb;

  const double uniform = 1.0 / (double)NN; /* :134 */
  if (x0) {
    memcpy(x, x0, sizeof(double) * NN); /* caller passes start/sum(start) (:135) */
  } else {
    for (long e = 0; e < NN; e++) x[e] = uniform;
  }

  int conv = 0, it = 0;
  for (it = 1; it <= max_iter; it++) { /* :139 */
    /* y = A'^T x : y[k,:] += A'[i,k] * x[i,:] */
    memset(y, 0, sizeof(double) * NN);
    for (int i = 0; i < N; i++)
      for (int k = 0; k < N; k++) {
        const double a = ap[(long)i * N + k];
        if (a == 0.0) continue;
        const double *xi = x + (long)i * N;
        double *yk = y + (long)k * N;
        for (int j = 0; j < N; j++) yk[j] += a * xi[j];
      }
    /* z = y B' : z[k,l] += y[k,j] * B'[j,l] (j ascending; zero entries of B'
     * skipped via its nonzero lists, which leaves every sum unchanged) */
    memset(z, 0, sizeof(double) * NN);
    for (int k = 0; k < N; k++)
      for (int j = 0; j < N; j++) {
        const double yv = y[(long)k * N + j];
        double *zk = z + (long)k * N;
        for (long e = bnz_ptr[j]; e < bnz_ptr[j + 1]; e++) zk[bnz_col[e]] += yv * bnz_val[e];
      }
    /* :140  fresh = alpha*kx + (1-alpha)*uniform */
    const double teleport = (1.0 - alpha) * uniform;
    for (long e = 0; e < NN; e++) z[e] = alpha * z[e] + teleport;
    const double s = pw_sum(z, NN, 1); /* :141 */
    for (long e = 0; e < NN; e++) z[e] = z[e] / s;
    for (long e = 0; e < NN; e++) y[e] = fabs(z[e] - x[e]);
    const double delta = pw_sum(y, NN, 1); /* :142 */
    double *t = x;
    x = z;
    z = t;
    if (delta < tol) { /* :144 */
      conv = 1;
      break;
    }
  }
  if (it > max_iter) it = max_iter;

  greedy(x, N, match, y); /* :149 */
  double w = 0.0;
  for (int i = 0; i < N; i++) w += x[(long)i * N + match[i]]; /* :150 */
  double d;
  if (N == 1) {
    d = 1.0;
  } else {
    double c = (w - 1.0 / N) / (1.0 - 1.0 / N); /* :171 */
    c = c < 1.0 ? c : 1.0;
    c = c > 0.0 ? c : 0.0;
    d = 1.0 + (1.0 - c);
  }
  if (X_out) memcpy(X_out, x, sizeof(double) * NN);
  if (match_out) memcpy(match_out, match, sizeof(int32_t) * N);
  if (d_out) *d_out = d;
  if (W_out) *W_out = w;
  if (iters_out) *iters_out = it;
  if (conv_out) *conv_out = (uint8_t)conv;
  free(bnz_ptr);
  free(bnz_col);
  free(bnz_val);
  free(ap);
  free(bp);
  free(x);
  free(y);
  free(z);
  free(match);
  return 0;
}

/* Densify graph g of a packed CSR corpus (same layout as include/cfgsim.h). */
static double *densify(int g, const int32_t *n_nodes, const int64_t *rp_off, const int32_t *rowptr,
                       const int64_t *nz_off, const int32_t *col, const double *val) {
  const int n = n_nodes[g];
  double *m = (double *)calloc((size_t)n * n, sizeof(double));
  const int32_t *rp = rowptr + rp_off[g];
  const int32_t *cc = col + nz_off[g];
  const double *vv = val + nz_off[g];
  for (int r = 0; r < n; r++)
    for (int e = rp[r]; e < rp[r + 1]; e++) m[(long)r * n + cc[e]] = vv[e];
  return m;
}

/* Batch over index pairs of one packed corpus; pthreads pull pairs from an
 * atomic counter. */
typedef struct {
  const int32_t *n_nodes, *rowptr, *col, *ia, *ib;
  const int64_t *rp_off, *nz_off;
  const double *val;
  int64_t n_pairs;
  double alpha, tol;
  int max_iter;
  double *d, *W;
  int32_t *iters;
  uint8_t *conv;
  atomic_llong next;
  atomic_int rc;
} batch_t;

static void *batch_worker(void *arg) {
  batch_t *B = (batch_t *)arg;
  for (;;) {
    const int64_t p = atomic_fetch_add(&B->next, 1);
    if (p >= B->n_pairs) break;
    double *a = densify(B->ia[p], B->n_nodes, B->rp_off, B->rowptr, B->nz_off, B->col, B->val);
    double *b = densify(B->ib[p], B->n_nodes, B->rp_off, B->rowptr, B->nz_off, B->col, B->val);
    int rc = oracle_iso_pair(B->n_nodes[B->ia[p]], a, B->n_nodes[B->ib[p]], b, B->alpha, B->tol,
                             B->max_iter, NULL, NULL, NULL, B->d ? B->d + p : NULL,
                             B->W ? B->W + p : NULL, B->iters ? B->iters + p : NULL,
                             B->conv ? B->conv + p : NULL);
    if (rc) atomic_store(&B->rc, rc);
    free(a);
    free(b);
  }
  return NULL;
}

int oracle_iso_batch(const int32_t *n_nodes, const int64_t *rp_off, const int32_t *rowptr,
                     const int64_t *nz_off, const int32_t *col, const double *val, int64_t n_pairs,
                     const int32_t *ia, const int32_t *ib, double alpha, double tol, int max_iter,
                     int threads, double *d, double *W, int32_t *iters, uint8_t *conv) {
  batch_t B = {n_nodes, rowptr, col, ia, ib, rp_off, nz_off, val, n_pairs, alpha, tol, max_iter,
               d, W, iters, conv};
  atomic_init(&B.next, 0);
  atomic_init(&B.rc, 0);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  for (int t = 0; t < threads; t++) pthread_create(&tid[t], NULL, batch_worker, &B);
  for (int t = 0; t < threads; t++) pthread_join(tid[t], NULL);
  return atomic_load(&B.rc);
}
