// Internal declarations shared by the kernel translation units and the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace ffps {

// Arguments of the persistent greedy kernel (one thread-block cluster per
// cloud).  See include/flashfps_b200.h, ffps_run_kernel, for the meaning.
struct GreedyParams {
  const void* xyz;
  int64_t cloud_stride;
  const int64_t* index_map;
  int64_t map_stride;
  int64_t n;
  int64_t iters;
  const int64_t* seed_pos;
  int64_t* order;
  void* sel_d2;
  int64_t out_stride;
  void* spill;      // [batch][C][G][2?][NT] vectors, only when spill_slots > 0
  int spill_slots;  // G: per-thread slots streamed from global memory
  float neg_zero;   // -0.0f, opaque to ptxas (see sq2 in fps_greedy.cu)
  long long* trace;     // optional phase trace (FFPS_TRACE_STREAM), else null
  int64_t trace_iters;
};

// K1s: one compiled configuration of the small-cloud kernel (fps_small.cu):
// nt threads per CTA, q points per thread (n <= nt * q), one CTA per cloud.
struct SmallInst {
  int dtype;  // 0 f32, 1 f64
  int nt;
  int q;
  const void* fn;
  size_t smem;  // dynamic shared memory (the shared copy of the points)
};
const SmallInst* small_instances(int* count);

// One compiled configuration of the greedy kernel.
struct KernelInst {
  int dtype;  // 0 f32, 1 f64
  int nt;     // threads per CTA
  int p;      // register-resident slots per thread (xyz + dist in registers)
  int s;      // smem-resident slots per thread (xyz in smem, dist in registers)
  int minb;   // CTAs per SM the register budget is sized for (__launch_bounds__)
  bool spill; // streams slots beyond P + S from a global spill buffer
  const void* fn;
  size_t smem_base;      // dynamic shared memory per CTA: points + mbarriers
  size_t smem_per_rank;  // + exchange records per cluster rank
  size_t smem_bytes(int C) const { return smem_base + (size_t)C * smem_per_rank; }
};

// All compiled configurations (fps_greedy.cu).
const KernelInst* greedy_instances(int* count);

// Spill-buffer bytes per (cloud, CTA) for G spill slots.
inline size_t spill_bytes_per_cta(int dtype, int nt, int g) {
  return static_cast<size_t>(g) * nt * (dtype == 0 ? 16 : 32);
}

// ---- bucketed path (K0 bucket_kd.cu + K1b fps_bucket.cu, K1g fps_grid*.cu) ----
constexpr int kBucketThreads = 512;

struct BucketBuildParams {
  const void* xyz;
  int64_t cloud_stride;
  const int64_t* index_map;
  int64_t map_stride;
  int64_t n;
  void *X, *Y, *Z, *D;  // [batch][nslots] bucket-major SoA
  int32_t* O;           // [batch][nslots] position in the run's point list (-1: padding)
  void* BB;             // [batch][nbuckets][6] bucket boxes
  int64_t nslots;
  int64_t nbuckets;
  int64_t bs;           // points per bucket
  void *TX, *TY, *TZ;   // [batch][nslots] scratch for the second sort level (or null)
  int32_t* TO;
  int d_wide;           // 1: D is double while the coordinates are float (FFPS_F32_F64)
};

struct BucketParams {
  const void *X, *Y, *Z;
  void* D;
  const int32_t* O;
  const void* BB;
  int64_t nslots;
  int64_t nbuckets;
  const void* xyz;  // original input (seed coordinates)
  int64_t cloud_stride;
  const int64_t* index_map;
  int64_t map_stride;
  int64_t iters;
  const int64_t* seed_pos;
  int64_t* order;
  void* sel_d2;
  int64_t out_stride;
  float neg_zero;  // -0.0f, opaque to ptxas (sq2)
  long long* trace;     // optional phase trace (FFPS_TRACE_BUCKET), else null
  int64_t trace_iters;
  long long* stats;     // optional [batch][4] counters (K1g, ffps_run_kernel_stats), else null
};

struct BucketInst {
  int dtype;
  int nt;
  int ppl;  // points per lane per bucket (bucket size 32 * ppl)
  int nbt;  // buckets owned per thread (max buckets = nt * nbt)
  const void* fn;
  size_t smem_per_bucket;
};

const BucketInst* bucket_instances(int* count);

// K1g (fps_grid.cu): multi-winner rounds with a cell index of the buckets
struct GridInst {
  int dtype;       // 0 f32, 1 f64, 2 f32 coordinates + binary64 arithmetic
  int nt;
  int ppl;
  int km;          // winners per round at most
  int cl;          // CTAs per cloud (thread-block cluster size)
  const void* fn;  // fps_grid_kernel(BucketParams)
  size_t esz;      // bytes per stored coordinate
};
const GridInst* grid_instances(int* count);  // all of the three below
const GridInst* grid_instances_f32(int* count);
const GridInst* grid_instances_f64(int* count);
const GridInst* grid_instances_mixed(int* count);
size_t grid_smem(int dtype, int64_t nb);
size_t bucket_kd_smem();
// kernel launches one launch_bucket_build issues (kd: CTA phase + leaf kernel)
int bucket_build_launches(const BucketBuildParams& p);
cudaError_t launch_bucket_kd(int dtype, const BucketBuildParams& p, int64_t batch,
                             cudaStream_t st);
cudaError_t launch_bucket_build(int dtype, const BucketBuildParams& p, int64_t batch,
                                cudaStream_t st);

// ---- K5 coverage radius (coverage.cu) ----
struct CoverageParams {
  const void *pX, *pY, *pZ, *pBB;  // cloud points, K0 buckets
  int64_t p_nslots, p_nbuckets, p_bs;
  const void *sX, *sY, *sZ, *sBB;  // sampled points, K0 buckets
  int64_t s_nslots, s_nbuckets, s_bs;
  void* out;  // [batch] max-min d2 (T), zero-initialised
};
cudaError_t launch_coverage(int dtype, const CoverageParams& p, int64_t batch, int sms,
                            cudaStream_t st);

// FFPS_F32_F64 on kernels without a float-coordinate variant: widen the
// [batch][cloud_stride][3] float rows [0, rows) into dense [batch][rows][3]
// doubles (convert.cu).
cudaError_t launch_upcast(const void* src, int64_t batch, int64_t cloud_stride, int64_t rows,
                          void* dst, int sms, cudaStream_t st);

// Library scratch: stream-ordered allocations from a private per-device pool
// (abi.cu), so the device's default pool and its attributes stay the caller's.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st);
cudaError_t scratch_free(void* p, cudaStream_t st);

// K2: slice fill (fill.cu).
cudaError_t launch_fill_slice(int dtype, int64_t* order, void* sel_d2, int64_t batch,
                              int64_t out_stride, int64_t k, int64_t m1, cudaStream_t st);

// K2r: seeded random fill (fill_random.cu); scratch = batch * words uint32.
int64_t fill_random_scratch_words(int64_t n, int64_t k, int64_t m1);
cudaError_t launch_fill_random(int dtype, int64_t* order, void* sel_d2, int64_t batch,
                               int64_t out_stride, int64_t n, int64_t k, int64_t m1,
                               const uint64_t pcg[4], uint32_t* scratch, cudaStream_t st,
                               bool sequential = false);

}  // namespace ffps
