/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement ("oracle") of the FlashFPS
 * reference hot path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library, and only as the
 * checker or the timed CPU baseline.  The product path never calls it.
 *
 * Restates, in plain C with every binary64/binary32 operation separately
 * rounded (compiled with -ffp-contract=off, no -ffast-math):
 *
 *   run_kernel            pkg/src/flashfps/fps_core.py:110-175
 *     dist2 sweep          fps_core.py:74-83   ((dx*dx + dy*dy) + dz*dz), dx = x - px
 *     min update           fps_core.py:93      np.minimum(dist, d2)
 *     first-max argmax     fps_core.py:94, :98-107 (lowest index on ties)
 *     init                 fps_core.py:124-130 (dist=+inf, dist[seed]=-inf,
 *                                               order[0]=seed, sel_d2[0]=+inf)
 *   run_restricted        pkg/src/flashfps/fps_cache.py:189-201 (index_map gather,
 *                                               positions mapped back)
 *   budget fill (slice)   pkg/src/flashfps/fps_prune.py:96-100 (ascending
 *                                               indices not selected, first fill_n)
 *
 * T = double reproduces the reference bit for bit (NumPy elementwise binary64
 * ufuncs are correctly rounded); T = float is the same algorithm in binary32
 * (the throughput path's arithmetic).  Parity pinning: tests/golden/ holds
 * vectors produced by the unmodified reference (make_golden.py) and by an
 * independent NumPy-float32 restatement; tests/test_oracle.py checks this
 * file against both.
 *
 * The batch entry points run one cloud per host thread (pthreads) so the
 * same code doubles as the multi-core CPU baseline.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DEFINE_RUN_KERNEL(T, SUF)                                               \
  /* returns distance_evals = n*(m-1) (fps_core.py:175); -1 on alloc error */   \
  int64_t ffps_oracle_run_kernel_##SUF(const T* xyz, int64_t n, int64_t m,     \
                                       int64_t seed, const int64_t* index_map,  \
                                       int64_t* order, T* sel_d2) {             \
    T* xs = (T*)malloc(sizeof(T) * (size_t)n * 4);                              \
    if (!xs) return -1;                                                         \
    T* ys = xs + n;                                                             \
    T* zs = ys + n;                                                             \
    T* dist = zs + n;                                                           \
    for (int64_t i = 0; i < n; ++i) {                                           \
      int64_t src = index_map ? index_map[i] : i;                               \
      xs[i] = xyz[3 * src + 0];                                                 \
      ys[i] = xyz[3 * src + 1];                                                 \
      zs[i] = xyz[3 * src + 2];                                                 \
      dist[i] = (T)INFINITY;                                                    \
    }                                                                           \
    order[0] = seed;                                                            \
    sel_d2[0] = (T)INFINITY;                                                    \
    dist[seed] = -(T)INFINITY;                                                  \
    T px = xs[seed], py = ys[seed], pz = zs[seed];                              \
    for (int64_t k = 1; k < m; ++k) {                                           \
      /* pass 1: min-update and running max (vectorizable; minps/maxps have    \
       * exactly the `a < b ? a : b` semantics, no NaN can occur) */            \
      T mx = -(T)INFINITY;                                                      \
      for (int64_t i = 0; i < n; ++i) {                                         \
        T dx = xs[i] - px;                                                      \
        T dy = ys[i] - py;                                                      \
        T dz = zs[i] - pz;                                                      \
        T d = (dx * dx + dy * dy) + dz * dz;                                    \
        T o = dist[i];                                                          \
        o = (d < o) ? d : o;                                                    \
        dist[i] = o;                                                            \
        mx = (o > mx) ? o : mx;                                                 \
      }                                                                         \
      /* pass 2: first occurrence of the max == np.argmax + chunk-order fold */ \
      int64_t best = 0;                                                         \
      while (dist[best] != mx) ++best;                                          \
      order[k] = best;                                                          \
      sel_d2[k] = mx;                                                           \
      dist[best] = -(T)INFINITY;                                                \
      px = xs[best];                                                            \
      py = ys[best];                                                            \
      pz = zs[best];                                                            \
    }                                                                           \
    if (index_map)                                                              \
      for (int64_t k = 0; k < m; ++k) order[k] = index_map[order[k]];           \
    free(xs);                                                                   \
    return n * (m - 1);                                                         \
  }

DEFINE_RUN_KERNEL(float, f32)
DEFINE_RUN_KERNEL(double, f64)

/* Budget fill, DETERMINISTIC_SLICE (fps_prune.py:96-100): the first fill_n
 * ascending indices of [0, n) that are not in order[0:k). */
int ffps_oracle_fill_slice(const int64_t* order, int64_t k, int64_t n,
                           int64_t fill_n, int64_t* out) {
  unsigned char* sel = (unsigned char*)calloc((size_t)n, 1);
  if (!sel) return -1;
  for (int64_t i = 0; i < k; ++i) sel[order[i]] = 1;
  int64_t w = 0;
  for (int64_t i = 0; i < n && w < fill_n; ++i)
    if (!sel[i]) out[w++] = i;
  free(sel);
  return w == fill_n ? 0 : -2;
}

/* ---- batch driver: one cloud per host thread ---------------------------- */
typedef struct {
  int dtype; /* 0 = f32, 1 = f64 */
  const void* xyz;
  int64_t cloud_stride; /* points between clouds */
  int64_t n, m;
  const int64_t* seeds;
  const int64_t* index_map;
  int64_t map_stride;
  int64_t* order;
  void* sel_d2;
  int64_t out_stride;
  int64_t batch;
  int64_t next; /* shared work counter */
  pthread_mutex_t mu;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int64_t b = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (b >= j->batch) break;
    const int64_t* map = j->index_map ? j->index_map + b * j->map_stride : 0;
    if (j->dtype == 0)
      ffps_oracle_run_kernel_f32((const float*)j->xyz + 3 * b * j->cloud_stride,
                                 j->n, j->m, j->seeds[b], map,
                                 j->order + b * j->out_stride,
                                 (float*)j->sel_d2 + b * j->out_stride);
    else
      ffps_oracle_run_kernel_f64((const double*)j->xyz + 3 * b * j->cloud_stride,
                                 j->n, j->m, j->seeds[b], map,
                                 j->order + b * j->out_stride,
                                 (double*)j->sel_d2 + b * j->out_stride);
  }
  return 0;
}

int ffps_oracle_run_kernel_batch(int dtype, const void* xyz, int64_t batch,
                                 int64_t cloud_stride, int64_t n, int64_t m,
                                 const int64_t* seeds, const int64_t* index_map,
                                 int64_t map_stride, int64_t* order,
                                 void* sel_d2, int64_t out_stride,
                                 int nthreads) {
  batch_job j;
  memset(&j, 0, sizeof j);
  j.dtype = dtype;
  j.xyz = xyz;
  j.cloud_stride = cloud_stride;
  j.n = n;
  j.m = m;
  j.seeds = seeds;
  j.index_map = index_map;
  j.map_stride = map_stride;
  j.order = order;
  j.sel_d2 = sel_d2;
  j.out_stride = out_stride;
  j.batch = batch;
  pthread_mutex_init(&j.mu, 0);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > batch) nthreads = (int)batch;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], 0, batch_worker, &j);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], 0);
  free(th);
  pthread_mutex_destroy(&j.mu);
  return 0;
}
