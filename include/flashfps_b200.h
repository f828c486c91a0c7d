/*
 * flashfps_b200.h — C ABI of the B200-native FlashFPS hot path.
 *
 * The reference (arxiv/paper_2604_17720, pkg/src/flashfps) has no FFI: its
 * hot path is the Python function
 *
 *     run_kernel(points (n,3) f64, m, seed_pos, threads=1)
 *         -> (order int64[m], selection_dist2 f64[m], distance_evals)
 *                                        pkg/src/flashfps/fps_core.py:110-175
 *
 * called from fps (fps_core.py:193), fps_prune (fps_prune.py:92),
 * verify_prefix_property (fps_cache.py:177) and run_restricted
 * (fps_cache.py:196).  Each entry point below replaces one of those seams
 * for a whole batch of clouds; the Python mirror of the reference API
 * (paper_2604_17720_b200/) binds them through ctypes (GIL released during the
 * call).  INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - All data pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *     on the current device, except where a name ends in _host.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered and do not synchronize the host, except *_host.
 *   - Return value: FFPS_OK (0) or a negative FFPS_E* code; the message of
 *     the last failure on the calling thread is ffps_last_error().
 *   - No global mutable state besides per-device kernel attribute caches;
 *     calls on different streams / host threads are independent.
 *   - Argument validation mirrors the reference's exceptions, which the
 *     Python layer raises BEFORE calling in (fps_core.py:178-182,
 *     fps_prune.py:78-88): a violated precondition here returns FFPS_EINVAL.
 */
#ifndef FLASHFPS_B200_H
#define FLASHFPS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFPS_ABI_VERSION 1

/* FFPS_F32      float coordinates, binary32 arithmetic, float sel_d2;
 * FFPS_F64      double coordinates, binary64 arithmetic, double sel_d2 (the
 *               reference's arithmetic, fps_core.py:74-83,124-126);
 * FFPS_F32_F64  float coordinates, binary64 arithmetic, double sel_d2: the
 *               reference run on fp32 clouds (PointCloud upcasts them exactly,
 *               geometry.py:52-54), with coordinates stored and moved as
 *               float.  Results are bit-identical to FFPS_F64 on the upcast
 *               cloud. */
enum ffps_dtype { FFPS_F32 = 0, FFPS_F64 = 1, FFPS_F32_F64 = 2 };

enum ffps_status {
  FFPS_OK = 0,
  FFPS_EINVAL = -1,       /* precondition violated (budget, seed, sizes)   */
  FFPS_EUNSUPPORTED = -2, /* shape outside every kernel configuration       */
  FFPS_ECUDA = -3         /* CUDA runtime / launch failure                 */
};

/* Farthest-first selection over a batch of clouds (replaces run_kernel,
 * fps_core.py:110-175, and its run_restricted form, fps_cache.py:189-201).
 *
 *   xyz          [batch][cloud_stride][3] AoS, float or double (dtype)
 *   n            points per cloud taking part: the candidate prefix
 *                xyz[b][0:n) (candidate pruning is a prefix slice,
 *                fps_prune.py:54-65,92) — or, when index_map != NULL, the
 *                gathered points xyz[b][index_map[b][i]], i < n
 *   iters        greedy iterations m (or the pruned budget k), 1 <= iters <= n
 *   seed_pos     [batch] int64 start positions (local to the point set)
 *   index_map    NULL or [batch][map_stride] int64 original indices
 *   order        [batch][out_stride] int64: order[b][0:iters) receives the
 *                selected ORIGINAL indices (mapped through index_map)
 *   sel_d2       [batch][out_stride] float/double: selection distances,
 *                sel_d2[b][0] = +inf
 * Ties break to the lowest position; results are bit-identical to the
 * reference's binary64 (F64) or to the same algorithm in binary32 (F32). */
int ffps_run_kernel(int dtype, const void* xyz, int64_t batch,
                    int64_t cloud_stride, int64_t n, int64_t iters,
                    const int64_t* seed_pos, const int64_t* index_map,
                    int64_t map_stride, int64_t* order, void* sel_d2,
                    int64_t out_stride, void* stream);

/* Greedy schedules behind ffps_run_kernel (identical results, bit for bit):
 *   FFPS_ALGO_STREAM  K1: one thread-block cluster per cloud, every point's
 *                     distance updated every iteration, state on chip
 *                     (registers + shared memory), DSMEM argmax exchange —
 *                     the "standard" exhaustive-update FPS schedule;
 *   FFPS_ALGO_BUCKET  K0 + K1b: points binned into spatial buckets, one CTA
 *                     per cloud; each iteration re-evaluates only the buckets
 *                     whose exact lower bound (same rounded ops) is below
 *                     their max distance;
 *   FFPS_ALGO_MULTI   retired (round 2): the register-table multi-winner K1m was
 *                     never faster than K1g; the value selects FFPS_ALGO_GRID;
 *   FFPS_ALGO_GRID    K0 + K1g: up to 16 winners per round, the buckets held in
 *                     shared memory and indexed by groups of 32 (kd order), so
 *                     a selected point only tests the buckets within its reach;
 *                     each cloud's buckets are split over a cluster of 1, 2 or
 *                     4 CTAs: FFPS_ALGO_GRID_CL(c) fixes c, plain
 *                     FFPS_ALGO_GRID takes 4 for n >= 40000 while the batch's
 *                     4-CTA clusters are all resident at once, else 2 for
 *                     n >= 20000 while batch * 2 <= SM count, else 1;
 *   FFPS_ALGO_SMALL   K1s: clouds of up to 8192 points, one CTA per cloud, points in
 *                     registers, one barrier per greedy step (larger clouds fall
 *                     back to STREAM);
 *   FFPS_ALGO_AUTO    binary32: SMALL for n <= 8192, GRID from n >= 10000
 *                     (2 CTAs per cloud from n >= 20000 while the batch fits
 *                     the SMs twice), BUCKET for smaller clouds when the batch
 *                     fills the GPU, else STREAM; binary64: SMALL up to 4608
 *                     points, GRID on 1 CTA below 16384, GRID beyond (the
 *                     environment variable
 *                     FFPS_ALGO=stream|small|bucket|grid overrides
 *                     AUTO). */
enum ffps_algo { FFPS_ALGO_AUTO = 0, FFPS_ALGO_STREAM = 1, FFPS_ALGO_BUCKET = 2,
                 FFPS_ALGO_MULTI = 3, FFPS_ALGO_GRID = 4, FFPS_ALGO_SMALL = 5 };
#define FFPS_ALGO_GRID_CL(c) (FFPS_ALGO_GRID | ((c) << 8))

/* ffps_run_kernel_ex plus per-cloud counters of the multi-winner schedule:
 * when `stats` (device, [batch][FFPS_STATS_WORDS] int64, caller-zeroed) is not
 * NULL the GRID schedule writes, per cloud, the rounds of its greedy loop,
 * the SM cycles the loop took on cluster rank 0, the buckets re-evaluated and
 * the rounds whose candidate ranking took the general path (both summed over
 * the cluster's CTAs);
 * other schedules leave it untouched.  Used to report the latency roofline
 * (cycles per round) next to the kernel time. */
#define FFPS_STATS_WORDS 4
int ffps_run_kernel_stats(int dtype, const void* xyz, int64_t batch,
                          int64_t cloud_stride, int64_t n, int64_t iters,
                          const int64_t* seed_pos, const int64_t* index_map,
                          int64_t map_stride, int64_t* order, void* sel_d2,
                          int64_t out_stride, void* stream, int algo, int64_t* stats);

/* Host -> device copy of the candidate prefix xyz[b][0:n_prefix) of every
 * cloud (the only coordinates a cache-on FlashFPS run reads,
 * fps_prune.py:92) into a dense [batch][n_prefix][3] device buffer: one
 * pitched copy (source pitch = cloud_stride points).  `src_host` should be
 * pinned for the copy to be asynchronous. */
int ffps_h2d_prefix(void* dst, const void* src_host, int64_t batch, int64_t n_prefix,
                    int64_t cloud_stride, int dtype, void* stream);

/* Device -> host copy of the first n_prefix elements (elem_bytes each) of
 * every row of a [batch][src_stride] device array into a [batch][dst_stride]
 * (pinned) host array, one pitched copy, stream-ordered: the greedy part of
 * the selection distances (the fill's are 0 by definition,
 * fps_prune.py:104-105, and are written on the host). */
int ffps_d2h_prefix(void* dst_host, int64_t dst_stride, const void* src, int64_t src_stride,
                    int64_t batch, int64_t n_prefix, int64_t elem_bytes, void* stream);

/* The schedule FFPS_ALGO_AUTO picks for a batch of `batch` clouds of n points
 * (FFPS_ALGO_STREAM, FFPS_ALGO_BUCKET or FFPS_ALGO_GRID_CL(c) with the
 * cluster size chosen for the whole batch); callers that split one batch into
 * concurrent chunks decide once for the whole batch and pass the result. */
int ffps_auto_schedule(int64_t n, int64_t batch);  /* binary32 arithmetic */
/* The same for the arithmetic of `dtype` (binary64 prefers the multi-winner
 * schedule from 4,609 points on, binary32 from 10,000). */
int ffps_auto_schedule_ex(int64_t n, int64_t batch, int dtype);

/* The multi-winner (K1g) configuration for a batch, under FFPS_ALGO_AUTO or a
 * FFPS_ALGO_GRID_CL(c) schedule: out[0]=CTAs per cloud, out[1]=points per
 * lane (buckets of 32 x out[1] points), out[2]=buckets per cloud,
 * out[3]=dynamic shared memory per CTA (bytes). */
int ffps_grid_plan(int dtype, int64_t n, int64_t batch, int algo, int64_t* out);

/* ffps_run_kernel with an explicit schedule (same arguments; algo as above). */
int ffps_run_kernel_ex(int dtype, const void* xyz, int64_t batch,
                       int64_t cloud_stride, int64_t n, int64_t iters,
                       const int64_t* seed_pos, const int64_t* index_map,
                       int64_t map_stride, int64_t* order, void* sel_d2,
                       int64_t out_stride, void* stream, int algo);

/* Budget fill, FillMode.DETERMINISTIC_SLICE (fps_prune.py:96-100,104-105):
 * for every cloud writes order[b][k + w], w < m1 - k, = the w-th smallest
 * index of [0, n) absent from order[b][0:k), and sel_d2[b][k + w] = 0. */
int ffps_fill_slice(int dtype, int64_t* order, void* sel_d2, int64_t batch,
                    int64_t out_stride, int64_t k, int64_t m1, void* stream);

/* Budget fill, FillMode.SEEDED_RANDOM (fps_prune.py:96-103): for every cloud
 * writes order[b][k + w], w < m1 - k, = the w-th entry of
 *     np.random.default_rng(seed).choice(pool, m1 - k, replace=False)
 * with pool the ascending complement of order[b][0:k) in [0, n), and
 * sel_d2[b][k + w] = 0.  The generator state is NumPy's PCG64(seed) state
 * (np.random.PCG64(seed).state: 128-bit state and increment, split in
 * high/low 64-bit halves); every cloud starts from it, as the reference
 * seeds one generator per call.  Draws follow NumPy 2.x's Generator.choice
 * (tail partial Fisher-Yates or Floyd + shuffle, Lemire bounded integers),
 * bit-identical to NumPy (oracle/npchoice.py pins the restatement). */
int ffps_fill_random(int dtype, int64_t* order, void* sel_d2, int64_t batch,
                     int64_t out_stride, int64_t n, int64_t k, int64_t m1,
                     uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                     uint64_t inc_lo, void* stream);

/* The whole FlashFPS pyramid in one call (replaces hierarchical_sample /
 * hierarchical_sample_detailed, fps_cache.py:204-256, with FPS-Prune layer 1,
 * fps_prune.py:68-111): layer 1 = greedy over the candidate prefix xyz[b][0:c)
 * for k iterations (k, c = PruneConfig.kernel_budget / candidate_count,
 * computed by the caller in IEEE double, fps_prune.py:45-51) followed by the
 * budget fill of [k, budgets[0]) (fill_mode 0 = DETERMINISTIC_SLICE, 1 =
 * SEEDED_RANDOM with pcg = NumPy's PCG64(rng_seed) state {state_hi, state_lo,
 * inc_hi, inc_lo}); with cache_enabled the deeper layers are prefixes of
 * layer 1 (fps_cache.py:141-148: order[l], sel_d2[l] for l >= 1 are not
 * written and may be NULL); without it layer l re-runs exact FPS over layer
 * l-1's points in their order, seeded at position 0 (fps_cache.py:189-201),
 * reported in original indices.
 *   budgets   HOST [nlayers], non-increasing, >= 1
 *   seed_pos  DEVICE [batch] layer-1 seed positions (< c)
 *   order     HOST array of nlayers DEVICE pointers, order[l] = [batch][budgets[l]] int64
 *   sel_d2    HOST array of nlayers DEVICE pointers, [batch][budgets[l]] (dtype's result type)
 * Stream-ordered launches, no host synchronisation. */
int ffps_hierarchical_sample(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride,
                             int64_t n, const int64_t* budgets, int nlayers, int64_t k,
                             int64_t c, int fill_mode, const uint64_t* pcg,
                             int cache_enabled, const int64_t* seed_pos, int64_t* const* order,
                             void* const* sel_d2, void* stream);

/* Covering radius of samples (replaces coverage_radius / _min_dist2_to,
 * metrics.py:29-52): out_d2[b] = max over p in xyz[b][0:n) of min over
 * i < m of d2(p, xyz[b][idx[b][i]]), the reference's rounded d2; the caller
 * takes sqrt (metrics.py:52).  Bit-exact (max/min of exactly rounded d2).
 *   idx     [batch][idx_stride] int64 sample indices into the cloud
 *   out_d2  [batch] float/double (dtype) */
int ffps_coverage(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride,
                  int64_t n, const int64_t* idx, int64_t idx_stride, int64_t m,
                  void* out_d2, void* stream);

/* Kernel configuration the library would use (for benches / reports).
 * out[0]=threads/CTA, out[1]=register slots/thread, out[2]=smem slots/thread,
 * out[3]=spill slots/thread, out[4]=CTAs per cluster (per cloud),
 * out[5]=resident CTAs per SM, out[6]=max resident clusters on the device. */
int ffps_plan(int dtype, int64_t n, int64_t batch, int64_t* out);

/* Bucketed-schedule configuration for n points: out[0]=threads/CTA,
 * out[1]=points per bucket, out[2]=buckets, out[3]=buckets owned per thread. */
int ffps_bucket_plan(int dtype, int64_t n, int64_t* out);

/* Hand the library's cached scratch memory (a private stream-ordered pool
 * per device, up to 4 GiB kept mapped between calls) back to the driver;
 * synchronises the current device. */
int ffps_trim_scratch(void);

/* Number of kernel launches the last successful call on this thread issued. */
int64_t ffps_last_launch_count(void);

const char* ffps_last_error(void);
int ffps_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FLASHFPS_B200_H */
