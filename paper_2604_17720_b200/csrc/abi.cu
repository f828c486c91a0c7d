// C ABI (include/flashfps_b200.h): argument checks, kernel-configuration
// planning and cluster launches.  No torch types cross this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "../../include/flashfps_b200.h"
#include "ffps_internal.h"

namespace {

thread_local std::string g_last_error;
thread_local int64_t g_last_launches = 0;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(FFPS_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

struct DeviceInfo {
  int sms = 0;
  size_t smem_optin = 0;
};

std::mutex g_mu;
std::map<int, DeviceInfo> g_dev;
std::map<std::tuple<int, const void*, int>, int> g_occ;  // (device, fn, C) -> max active clusters
std::map<std::pair<int, const void*>, bool> g_attr_done;

std::map<int, cudaMemPool_t> g_pool;  // library scratch pool per device

// Scratch (spill buffers, K0 buckets, widened clouds) comes from a private
// stream-ordered pool per device, so the caller's default pool keeps its own
// attributes.  The pool keeps up to kKeepBytes mapped across synchronisations
// (a release threshold of 0 would hand the memory back at every sync and the
// next call would re-map it on the host: tens of ms for ~100 MB); beyond that
// it releases, and ffps_trim_scratch() hands everything back.
constexpr uint64_t kKeepBytes = 4ull << 30;

cudaError_t pool_for(int dev, cudaMemPool_t* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_pool.find(dev);
  if (it != g_pool.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  cudaMemPoolProps props;
  memset(&props, 0, sizeof props);
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool;
  cudaError_t e = cudaMemPoolCreate(&pool, &props);
  if (e != cudaSuccess) return e;
  uint64_t keep = kKeepBytes;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  // no hidden cross-stream waits: chunks of one batch on side streams must
  // not be serialised by the pool reusing another stream's freed block
  int no = 0;
  cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  cudaGetLastError();
  g_pool[dev] = pool;
  *out = pool;
  return cudaSuccess;
}

DeviceInfo device_info_nolock(int dev) {
  auto it = g_dev.find(dev);
  if (it != g_dev.end()) return it->second;
  DeviceInfo d;
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  d.sms = v;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  d.smem_optin = (size_t)v;
  g_dev[dev] = d;
  return d;
}

DeviceInfo device_info(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  return device_info_nolock(dev);
}

cudaError_t prepare_fn(int dev, const ffps::KernelInst& k) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, k.fn);
  if (g_attr_done.count(key)) return cudaSuccess;
  const DeviceInfo di = device_info_nolock(dev);
  cudaError_t e = cudaFuncSetAttribute(
      k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)std::min(k.smem_bytes(16), di.smem_optin));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  g_attr_done[key] = true;
  return cudaSuccess;
}

int max_active_clusters(int dev, const ffps::KernelInst& k, int C) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_occ.find(std::make_tuple(dev, k.fn, C));
    if (it != g_occ.end()) return it->second;
  }
  int result = 0;
  if (prepare_fn(dev, k) == cudaSuccess) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(C * 64, 1, 1);
    cfg.blockDim = dim3(k.nt, 1, 1);
    cfg.dynamicSmemBytes = k.smem_bytes(C);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&result, k.fn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      result = 0;
    }
  } else {
    cudaGetLastError();
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_occ[std::make_tuple(dev, k.fn, C)] = result;
  return result;
}

struct Plan {
  const ffps::KernelInst* inst = nullptr;
  int C = 0;
  int G = 0;
  int ctas_per_sm = 0;
  int max_clusters = 0;
};

// Cost model (SM cycles per greedy iteration of the slowest wave):
//   issue work of one CTA  W = NT * Q * c / 128   (c ~ 9.5 instr per register
//                            slot, ~10.3 per smem slot, 4 warp-instr/clk/SM)
//   exposed latency of the reduction + DSMEM push  L(C) = 450 + 25 C
//   t_iter = max(W + L, r * W) with r resident CTAs per SM, times the waves.
// FFPS_FORCE_PLAN="nt,p,s,C" overrides (benchmark sweeps).
bool make_plan(int dev, int dtype, int64_t n, int64_t batch, Plan* out) {
  const DeviceInfo di = device_info(dev);
  int cnt = 0;
  const ffps::KernelInst* insts = ffps::greedy_instances(&cnt);
  const char* force = getenv("FFPS_FORCE_PLAN");
  if (force && *force) {
    int nt = 0, p = -1, s = -1, C = 0;
    if (sscanf(force, "%d,%d,%d,%d", &nt, &p, &s, &C) == 4 && C >= 1 && C <= 16) {
      const int64_t cap = (int64_t)C * nt * (p + s);
      const bool spill = cap < n;
      for (int i = 0; i < cnt; ++i) {
        const auto& k = insts[i];
        if (k.dtype == dtype && k.nt == nt && k.p == p && k.s == s && k.spill == spill) {
          const int64_t need = (n + (int64_t)C * k.nt - 1) / ((int64_t)C * k.nt);
          out->inst = &k;
          out->C = C;
          out->G = spill ? (int)(need - (k.p + k.s)) : 0;
          out->max_clusters = max_active_clusters(dev, k, C);
          out->ctas_per_sm = k.minb;
          return out->max_clusters > 0;
        }
      }
    }
    return false;
  }
  double best = 1e300;
  for (int i = 0; i < cnt; ++i) {
    const auto& k = insts[i];
    if (k.dtype != dtype || k.spill) continue;
    const int Q = k.p + k.s;
    const int64_t per_cta = (int64_t)k.nt * Q;
    const int64_t Cmin = (n + per_cta - 1) / per_cta;
    if (Cmin > 16) continue;
    const int C = (int)Cmin;
    if (k.smem_bytes(C) > di.smem_optin) continue;
    const int mc = max_active_clusters(dev, k, C);
    if (mc <= 0) continue;
    const double waves = std::ceil((double)batch / mc);
    const int64_t resident = std::min<int64_t>(batch, mc) * C;
    const int r = (int)std::min<int64_t>(k.minb, (resident + di.sms - 1) / di.sms);
    // issue cycles per point: ~5.5 (f32 packed) / ~10 (f64) plus an LDS per
    // 4 (f32) / 2 (f64) smem points; 4 warp-instructions per clock per SM
    const double cr = dtype == FFPS_F32 ? 5.5 : 10.0;
    const double cs = cr + (dtype == FFPS_F32 ? 0.75 : 1.5);
    const double c = (k.p * cr + k.s * cs) / std::max(1, Q);
    const double W = k.nt * Q * c / 128.0;
    const double L = 700.0 + 20.0 * C;
    const double t = std::max(W + L, r * W) * waves;
    if (t < best * 0.999) {
      best = t;
      out->inst = &k;
      out->C = C;
      out->G = 0;
      out->ctas_per_sm = r;
      out->max_clusters = mc;
    }
  }
  if (out->inst) return true;
  // Spill: the largest on-chip configuration at 16 CTAs/cloud, the remainder
  // of each thread's range streamed from global memory every iteration.
  const ffps::KernelInst* big = nullptr;
  for (int i = 0; i < cnt; ++i) {
    const auto& k = insts[i];
    if (k.dtype != dtype || !k.spill || k.smem_bytes(16) > di.smem_optin) continue;
    if (!big || (int64_t)k.nt * (k.p + k.s) * 4 / k.minb >
                    (int64_t)big->nt * (big->p + big->s) * 4 / big->minb)
      big = &k;
  }
  if (!big) return false;
  const int C = 16;
  const int64_t per_thread = (n + (int64_t)C * big->nt - 1) / ((int64_t)C * big->nt);
  if (per_thread - (big->p + big->s) > (1 << 20)) return false;
  out->inst = big;
  out->C = C;
  out->G = (int)(per_thread - (big->p + big->s));
  out->max_clusters = max_active_clusters(dev, *big, C);
  out->ctas_per_sm = big->minb;
  return out->max_clusters > 0;
}

}  // namespace

namespace ffps {

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  e = pool_for(dev, &pool);
  if (e != cudaSuccess) return e;
  return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

cudaError_t scratch_free(void* p, cudaStream_t st) { return cudaFreeAsync(p, st); }

}  // namespace ffps

extern "C" {

int ffps_trim_scratch(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  cudaMemPool_t pool;
  e = pool_for(dev, &pool);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemPoolTrimTo(pool, 0);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemPoolTrimTo");
  return FFPS_OK;
}

int ffps_abi_version(void) { return FFPS_ABI_VERSION; }

const char* ffps_last_error(void) { return g_last_error.c_str(); }

int64_t ffps_last_launch_count(void) { return g_last_launches; }

int ffps_plan(int dtype, int64_t n, int64_t batch, int64_t* out) {
  if ((dtype != FFPS_F32 && dtype != FFPS_F64 && dtype != FFPS_F32_F64) || n < 1 || batch < 1 ||
      !out)
    return fail(FFPS_EINVAL, "ffps_plan: bad arguments");
  if (dtype == FFPS_F32_F64) dtype = FFPS_F64;  // K1 runs on the widened cloud
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  Plan p;
  if (!make_plan(dev, dtype, n, batch, &p))
    return fail(FFPS_EUNSUPPORTED, "no kernel configuration for n=%lld", (long long)n);
  out[0] = p.inst->nt;
  out[1] = p.inst->p;
  out[2] = p.inst->s;
  out[3] = p.G;
  out[4] = p.C;
  out[5] = p.ctas_per_sm;
  out[6] = p.max_clusters;
  return FFPS_OK;
}

}  // extern "C"

namespace {

struct BucketPlan {
  const ffps::BucketInst* inst = nullptr;
  int64_t nbuckets = 0;
  size_t smem = 0;
};

// Smallest bucket size whose bucket count fits the owned-bucket registers
// (nt * nbt) and whose per-bucket keys fit shared memory.
bool make_bucket_plan(int dev, int dtype, int64_t n, BucketPlan* out) {
  const DeviceInfo di = device_info(dev);
  int cnt = 0;
  const ffps::BucketInst* insts =
      ffps::bucket_instances(&cnt);
  const size_t static_smem = 1024;
  const char* want_nt = getenv("FFPS_BUCKET_NT");  // sweeps: restrict the CTA size
  const int force_nt = want_nt ? atoi(want_nt) : 0;

  for (int ppl = 1; ppl <= 4; ppl *= 2) {
    const ffps::BucketInst* pick = nullptr;
    const int64_t nb = (n + 32 * ppl - 1) / (32 * ppl);
    for (int i = 0; i < cnt; ++i) {
      const auto& k = insts[i];
      if (k.dtype != dtype || k.ppl != ppl || (int64_t)k.nt * k.nbt < nb) continue;
      if (force_nt && k.nt != force_nt) continue;
      if ((size_t)nb * k.smem_per_bucket + static_smem > di.smem_optin) continue;
      // default CTA size first (FFPS_BUCKET_NT selects others), then fewest boxes/lane
      const int want = force_nt ? force_nt : ffps::kBucketThreads;
      const bool pk = pick && pick->nt == want, kk = k.nt == want;
      if (!pick || (kk && !pk) || (kk == pk && k.nbt < pick->nbt)) pick = &k;
    }
    if (pick) {
      out->inst = pick;
      out->nbuckets = nb;
      out->smem = (size_t)nb * pick->smem_per_bucket;
      return true;
    }
  }
  return false;
}

// bytes of the bucket-box array [batch][nb][6], rounded up to 256 so that the
// arrays carved after it (O, TX..TO) stay 16-B aligned for the TMA staging of K0
size_t box_bytes(int64_t nb, size_t esz, int64_t batch) {
  return ((size_t)nb * 6 * esz * (size_t)batch + 255) / 256 * 256;
}

int run_bucketed(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n,
                 int64_t iters, const int64_t* seed_pos, const int64_t* index_map,
                 int64_t map_stride, int64_t* order, void* sel_d2, int64_t out_stride,
                 cudaStream_t st, int dev) {
  BucketPlan bp;
  if (!make_bucket_plan(dev, dtype, n, &bp))
    return fail(FFPS_EUNSUPPORTED, "no bucketed configuration for n=%lld", (long long)n);
  const ffps::BucketInst& k = *bp.inst;
  const int64_t bs = 32 * k.ppl;
  const int64_t nslots = bp.nbuckets * bs;
  const size_t esz = dtype == FFPS_F32 ? 4 : 8;
  // scratch: X, Y, Z, D (esz) + O (4 B) per slot, boxes 6 * esz per bucket,
  // + TX, TY, TZ, TO for the second sort level of K0
  const size_t per_cloud = (size_t)nslots * (7 * esz + 8) + (size_t)bp.nbuckets * 6 * esz;
  unsigned char* scratch = nullptr;
  cudaError_t e = ffps::scratch_alloc(reinterpret_cast<void**>(&scratch),
                                  per_cloud * (size_t)batch + 512, st);
  if (e != cudaSuccess) return cuda_fail(e, "scratch_alloc(buckets)");
  const size_t arr = (size_t)nslots * esz * (size_t)batch;
  ffps::BucketBuildParams bb;
  bb.d_wide = 0;
  bb.xyz = xyz;
  bb.cloud_stride = cloud_stride;
  bb.index_map = index_map;
  bb.map_stride = map_stride;
  bb.n = n;
  bb.X = scratch;
  bb.Y = scratch + arr;
  bb.Z = scratch + 2 * arr;
  bb.D = scratch + 3 * arr;
  bb.BB = scratch + 4 * arr;
  bb.O = reinterpret_cast<int32_t*>(scratch + 4 * arr +
                                    box_bytes(bp.nbuckets, esz, batch));
  bb.nslots = nslots;
  bb.nbuckets = bp.nbuckets;
  bb.bs = bs;
  {
    unsigned char* t = reinterpret_cast<unsigned char*>(bb.O) + (size_t)nslots * 4 * (size_t)batch;
    bb.TX = t;
    bb.TY = t + arr;
    bb.TZ = t + 2 * arr;
    bb.TO = reinterpret_cast<int32_t*>(t + 3 * arr);
  }
  e = ffps::launch_bucket_build(dtype, bb, batch, st);
  if (e != cudaSuccess) {
    ffps::scratch_free(scratch, st);
    return cuda_fail(e, "bucket_build_kernel launch");
  }
  ffps::BucketParams prm;
  prm.X = bb.X;
  prm.Y = bb.Y;
  prm.Z = bb.Z;
  prm.D = bb.D;
  prm.O = bb.O;
  prm.BB = bb.BB;
  prm.nslots = nslots;
  prm.nbuckets = bp.nbuckets;
  prm.xyz = xyz;
  prm.cloud_stride = cloud_stride;
  prm.index_map = index_map;
  prm.map_stride = map_stride;
  prm.iters = iters;
  prm.seed_pos = seed_pos;
  prm.order = order;
  prm.sel_d2 = sel_d2;
  prm.out_stride = out_stride;
  prm.neg_zero = -0.0f;
  prm.trace = nullptr;
  prm.trace_iters = 0;
  prm.stats = nullptr;
  // FFPS_TRACE_BUCKET=<device pointer>,<iterations>: phase trace of CTA 0
  if (const char* tr = getenv("FFPS_TRACE_BUCKET")) {
    unsigned long long ptr = 0;
    long long it = 0;
    if (sscanf(tr, "%llu,%lld", &ptr, &it) == 2) {
      prm.trace = reinterpret_cast<long long*>(ptr);
      prm.trace_iters = it;
    }
  }
  void* args[] = {&prm};
  e = cudaLaunchKernel(k.fn, dim3((unsigned)batch), dim3(k.nt), args, 0, st);
  if (e != cudaSuccess) {
    ffps::scratch_free(scratch, st);
    return cuda_fail(e, "fps_bucket_kernel launch");
  }
  g_last_launches = 1 + ffps::bucket_build_launches(bb);
  e = ffps::scratch_free(scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "scratch_free(buckets)");
  return FFPS_OK;
}

// K1g: smallest bucket size whose bucket table + cell index fit shared memory
int grid_cluster(int algo, int64_t batch, int sms, int64_t n);

struct GridPick {
  const ffps::GridInst* inst = nullptr;
  int64_t nb = 0;   // buckets per cloud
  size_t smem = 0;  // dynamic shared memory per CTA
};

// Bucket size class (32 x PPL points): the smallest whose per-rank table
// holds at most kGridBucketsPerCta buckets and fits shared memory (else the
// smallest that fits).  Measured over 25K-150K candidates, 16 and 64 clouds,
// 1/2/4 CTAs per cloud, binary64, uniform and LiDAR-like clouds
// (profiles/r02_sweep_ppl_f64.txt, r02_ab_ppl_uniform_lidar.txt,
// tools/gpu_ppl*.sh): tables of ~1,200+ buckets per CTA pay in the group
// statistics and ranking (75K candidates on 2 CTAs: 1,172 buckets of 32 points
// per CTA 13.2 ms, 586 of 64 points 11.5 ms uniform / 13.2 vs 12.2 LiDAR;
// 150K: 586 of 128 points 24.7 ms, 2,344 of 32 points 30.7 ms), while tables of
// fewer than 16 groups take the general ranking path often on uneven clouds
// (50K on 2 CTAs: 782 buckets of 32 points 7.78 ms uniform / 7.96 LiDAR, 391
// of 64 points 7.64 / 8.65).  FFPS_GRID_PPL (A/B) sets the class.
constexpr int64_t kGridBucketsPerCta = 800;

GridPick pick_grid(int dtype, int64_t n, int cl, int km, const DeviceInfo& di) {
  int cnt = 0;
  const ffps::GridInst* insts = ffps::grid_instances(&cnt);
  int ppl0 = 1;  // FFPS_GRID_PPL (A/B): this bucket size class when it fits
  if (const char* v = getenv("FFPS_GRID_PPL")) ppl0 = std::max(1, std::min(8, atoi(v)));
  const bool exact = getenv("FFPS_GRID_PPL") != nullptr;
  GridPick best;
  for (int ppl = ppl0; ppl <= 8; ppl *= 2) {
    GridPick g;
    g.nb = (n + 32 * ppl - 1) / (32 * ppl);
    const int64_t nbl = (g.nb + cl - 1) / cl;  // buckets of cluster rank 0 (the most)
    if (nbl > 4096) continue;                  // <= 128 bucket groups per CTA
    g.smem = ffps::grid_smem(dtype, nbl);
    for (int i = 0; i < cnt; ++i)
      if (insts[i].dtype == dtype && insts[i].ppl == ppl && insts[i].km == km &&
          insts[i].cl == cl) {
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, insts[i].fn) != cudaSuccess) {
          cudaGetLastError();
          continue;
        }
        if (g.smem + fa.sharedSizeBytes <= di.smem_optin) g.inst = &insts[i];  // + static smem
      }
    if (!g.inst) continue;
    if (!best.inst) best = g;          // the smallest class that fits
    if (exact || nbl <= kGridBucketsPerCta) {  // the smallest with a table of the measured size
      best = g;
      break;
    }
  }
  return best;
}

cudaError_t prepare_grid_fn(int dev, const void* fn) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, fn);
  if (g_attr_done.count(key)) return cudaSuccess;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(device_info_nolock(dev).smem_optin - fa.sharedSizeBytes));
  if (e == cudaSuccess) g_attr_done[key] = true;
  return e;
}

// clusters of one K1g instance resident at once (one CTA per SM; a cluster
// must fit in one GPC, so fewer 4-CTA clusters fit than SMs / 4: 33 to 35
// on the B200, measured)
int grid_max_clusters(int dev, const GridPick& g) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_occ.find(std::make_tuple(dev, g.inst->fn, g.inst->cl));
    if (it != g_occ.end()) return it->second;
  }
  int result = 0;
  if (prepare_grid_fn(dev, g.inst->fn) == cudaSuccess) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(g.inst->cl * 64, 1, 1);
    cfg.blockDim = dim3(g.inst->nt, 1, 1);
    cfg.dynamicSmemBytes = g.smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = g.inst->cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&result, g.inst->fn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      result = 0;
    }
  } else {
    cudaGetLastError();
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_occ[std::make_tuple(dev, g.inst->fn, g.inst->cl)] = result;
  return result;
}

// K1g configuration of a batch: CTAs per cloud by grid_cluster; when AUTO
// chose 4 and the batch's clusters would not all be resident at once (a
// second wave doubles the time), halve it
GridPick choose_grid(int dtype, int64_t n, int64_t batch, int algo, int dev, int* cl_out) {
  const DeviceInfo di = device_info(dev);
  const bool forced = (algo >> 8) != 0 || getenv("FFPS_GRID_CL") != nullptr;
  int cl = grid_cluster(algo, batch, di.sms, n);
  GridPick g;
  for (;;) {
    // winners per round at most: 16 (one DSMEM record per lane with 1-2 CTAs
    // per cloud, two per lane with 4); FFPS_GRID_KM=8 forces 8.  (KM = 32 was
    // measured slower at C5: 21 winners per round but 20K cycles per round,
    // DESIGN.md.)
    int km = 16;
    if (const char* v = getenv("FFPS_GRID_KM")) {
      if (atoi(v) == 8) km = 8;
    }
    g = pick_grid(dtype, n, cl, km, di);
    if (!forced && cl > 2 && (!g.inst || grid_max_clusters(dev, g) < batch)) {
      cl /= 2;
      continue;
    }
    break;
  }
  *cl_out = cl;
  return g;
}

int run_grid(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n,
             int64_t iters, const int64_t* seed_pos, const int64_t* index_map, int64_t map_stride,
             int64_t* order, void* sel_d2, int64_t out_stride, cudaStream_t st, int dev,
             int algo, int64_t* stats) {
  int cl = 0;
  const GridPick g = choose_grid(dtype, n, batch, algo, dev, &cl);
  const ffps::GridInst* pick = g.inst;
  const int64_t nb = g.nb;
  const size_t smem = g.smem;
  if (!pick) return fail(FFPS_EUNSUPPORTED, "no grid configuration for n=%lld", (long long)n);
  const int64_t bs = 32 * pick->ppl;
  const int64_t nslots = nb * bs;
  const size_t esz = pick->esz;                     // stored coordinate
  const size_t desz = dtype == FFPS_F32 ? 4 : 8;    // running distance (arithmetic type)
  // X, Y, Z, D, boxes, O + the K0 scratch TX, TY, TZ, TO
  const size_t per_cloud = (size_t)nslots * (6 * esz + desz + 8) + (size_t)nb * 6 * esz;
  unsigned char* scratch = nullptr;
  cudaError_t e = ffps::scratch_alloc(reinterpret_cast<void**>(&scratch),
                                  per_cloud * (size_t)batch + 512, st);
  if (e != cudaSuccess) return cuda_fail(e, "scratch_alloc(grid)");
  const size_t arr = (size_t)nslots * esz * (size_t)batch;
  const size_t darr = (size_t)nslots * desz * (size_t)batch;
  ffps::BucketBuildParams bb;
  bb.d_wide = dtype == FFPS_F32_F64 ? 1 : 0;
  bb.xyz = xyz;
  bb.cloud_stride = cloud_stride;
  bb.index_map = index_map;
  bb.map_stride = map_stride;
  bb.n = n;
  bb.X = scratch;
  bb.Y = scratch + arr;
  bb.Z = scratch + 2 * arr;
  bb.D = scratch + 3 * arr;
  bb.BB = scratch + 3 * arr + darr;
  bb.O = reinterpret_cast<int32_t*>(scratch + 3 * arr + darr + box_bytes(nb, esz, batch));
  bb.nslots = nslots;
  bb.nbuckets = nb;
  bb.bs = bs;
  {
    unsigned char* t = reinterpret_cast<unsigned char*>(bb.O) + (size_t)nslots * 4 * (size_t)batch;
    bb.TX = t;
    bb.TY = t + arr;
    bb.TZ = t + 2 * arr;
    bb.TO = reinterpret_cast<int32_t*>(t + 3 * arr);
  }
  // K0 sorts float coordinates under FFPS_F32_F64 (D written as double)
  e = ffps::launch_bucket_build(dtype == FFPS_F32_F64 ? FFPS_F32 : dtype, bb, batch, st);
  if (e != cudaSuccess) {
    ffps::scratch_free(scratch, st);
    return cuda_fail(e, "bucket_build_kernel launch");
  }
  ffps::BucketParams prm;
  prm.X = bb.X;
  prm.Y = bb.Y;
  prm.Z = bb.Z;
  prm.D = bb.D;
  prm.O = bb.O;
  prm.BB = bb.BB;
  prm.nslots = nslots;
  prm.nbuckets = nb;
  prm.stats = reinterpret_cast<long long*>(stats);
  prm.xyz = xyz;
  prm.cloud_stride = cloud_stride;
  prm.index_map = index_map;
  prm.map_stride = map_stride;
  prm.iters = iters;
  prm.seed_pos = seed_pos;
  prm.order = order;
  prm.sel_d2 = sel_d2;
  prm.out_stride = out_stride;
  prm.neg_zero = -0.0f;
  prm.trace = nullptr;
  prm.trace_iters = 0;
  if (const char* tr = getenv("FFPS_TRACE_GRID")) {
    unsigned long long ptr = 0;
    long long it = 0;
    if (sscanf(tr, "%llu,%lld", &ptr, &it) == 2) {
      prm.trace = reinterpret_cast<long long*>(ptr);
      prm.trace_iters = it;
    }
  }
  e = prepare_grid_fn(dev, pick->fn);
  if (e != cudaSuccess) {
    ffps::scratch_free(scratch, st);
    return cuda_fail(e, "cudaFuncSetAttribute(grid)");
  }
  void* args[] = {&prm};
  {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(batch * pick->cl));
    lc.blockDim = dim3(pick->nt);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)pick->cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    e = cudaLaunchKernelExC(&lc, pick->fn, args);
  }
  if (e != cudaSuccess) {
    ffps::scratch_free(scratch, st);
    return cuda_fail(e, "fps_grid_kernel launch");
  }
  g_last_launches = 1 + ffps::bucket_build_launches(bb);
  e = ffps::scratch_free(scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "scratch_free(grid)");
  return FFPS_OK;
}

// K1s: clouds of up to 8192 points, one CTA per cloud (fps_small.cu); the
// smallest thread count / points-per-thread pair that holds n
int run_small(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n,
              int64_t iters, const int64_t* seed_pos, const int64_t* index_map,
              int64_t map_stride, int64_t* order, void* sel_d2, int64_t out_stride,
              cudaStream_t st) {
  int cnt = 0;
  const ffps::SmallInst* insts = ffps::small_instances(&cnt);
  const ffps::SmallInst* pick = nullptr;
  int fnt = 0, fq = 0;  // FFPS_SMALL_PLAN="nt,q" (sweeps)
  if (const char* v = getenv("FFPS_SMALL_PLAN")) sscanf(v, "%d,%d", &fnt, &fq);
  for (int i = 0; i < cnt; ++i) {
    const auto& k = insts[i];
    if (k.dtype != dtype || (int64_t)k.nt * k.q < n) continue;
    if (fnt) {
      if (k.nt == fnt && k.q == fq) pick = &k;
      continue;
    }
    const int64_t cap = (int64_t)k.nt * k.q, pcap = pick ? (int64_t)pick->nt * pick->q : 0;
    if (!pick || cap < pcap || (cap == pcap && k.nt > pick->nt)) pick = &k;  // fewer slots per thread
  }
  if (!pick) return fail(FFPS_EUNSUPPORTED, "no small-cloud configuration for n=%lld", (long long)n);
  ffps::GreedyParams prm;
  memset(&prm, 0, sizeof prm);
  prm.xyz = xyz;
  prm.cloud_stride = cloud_stride;
  prm.index_map = index_map;
  prm.map_stride = map_stride;
  prm.n = n;
  prm.iters = iters;
  prm.seed_pos = seed_pos;
  prm.order = order;
  prm.sel_d2 = sel_d2;
  prm.out_stride = out_stride;
  prm.neg_zero = -0.0f;
  cudaError_t e = cudaFuncSetAttribute(pick->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pick->smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(small)");
  void* args[] = {&prm};
  e = cudaLaunchKernel(pick->fn, dim3((unsigned)batch), dim3(pick->nt), args, pick->smem, st);
  if (e != cudaSuccess) return cuda_fail(e, "fps_small_kernel launch");
  g_last_launches = 1;
  return FFPS_OK;
}

int run_streaming(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n,
                  int64_t iters, const int64_t* seed_pos, const int64_t* index_map,
                  int64_t map_stride, int64_t* order, void* sel_d2, int64_t out_stride,
                  cudaStream_t st, int dev) {
  Plan plan;
  if (!make_plan(dev, dtype, n, batch, &plan))
    return fail(FFPS_EUNSUPPORTED, "no kernel configuration for n=%lld", (long long)n);
  const ffps::KernelInst& k = *plan.inst;
  cudaError_t e = prepare_fn(dev, k);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");

  ffps::GreedyParams prm;
  prm.xyz = xyz;
  prm.cloud_stride = cloud_stride;
  prm.index_map = index_map;
  prm.map_stride = map_stride;
  prm.n = n;
  prm.iters = iters;
  prm.seed_pos = seed_pos;
  prm.order = order;
  prm.sel_d2 = sel_d2;
  prm.out_stride = out_stride;
  prm.spill = nullptr;
  prm.spill_slots = plan.G;
  prm.neg_zero = -0.0f;
  prm.trace = nullptr;
  prm.trace_iters = 0;
  if (const char* tr = getenv("FFPS_TRACE_STREAM")) {  // <device pointer>,<iterations>
    unsigned long long ptr = 0;
    long long it = 0;
    if (sscanf(tr, "%llu,%lld", &ptr, &it) == 2) {
      prm.trace = reinterpret_cast<long long*>(ptr);
      prm.trace_iters = it;
    }
  }
  if (plan.G > 0) {
    const size_t bytes =
        ffps::spill_bytes_per_cta(dtype, k.nt, plan.G) * (size_t)plan.C * (size_t)batch;
    e = ffps::scratch_alloc(&prm.spill, bytes, st);
    if (e != cudaSuccess) return cuda_fail(e, "scratch_alloc(spill)");
  }

  // Clusters of a batch beyond the device's resident capacity simply queue;
  // each cluster is persistent for its own cloud.  Grid limit: 2^31-1 CTAs.
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3((unsigned)(batch * plan.C), 1, 1);
  cfg.blockDim = dim3(k.nt, 1, 1);
  cfg.dynamicSmemBytes = k.smem_bytes(plan.C);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = plan.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&prm};
  e = cudaLaunchKernelExC(&cfg, k.fn, args);
  if (e != cudaSuccess) {
    if (prm.spill) ffps::scratch_free(prm.spill, st);
    return cuda_fail(e, "fps_greedy_kernel launch");
  }
  g_last_launches = 1;
  if (prm.spill) {
    e = ffps::scratch_free(prm.spill, st);
    if (e != cudaSuccess) return cuda_fail(e, "scratch_free(spill)");
  }
  return FFPS_OK;
}

// FFPS_ALGO_AUTO (measured on B200 over batch 1..64 x n 1K..200K with
// iters = n/4, tools/sweep_auto.py / sweep_cl.py, profiles/r01_sweep_cl.jsonl,
// profiles/r02_sweep_auto_f32.jsonl, r02_sweep_auto_f64.jsonl; the time per
// cloud is flat in the batch until the clusters outnumber the SMs):
// binary32 —
//   SMALL  (one CTA per cloud, points in registers) for clouds of <= 8192 points;
//   GRID   (multi-winner rounds, bucket-group index) from 10,000 points (12K:
//          1 CTA per cloud 2.03-2.17 ms vs 2.25-3.7 for the others);
//   BUCKET for 6K+ clouds when the batch fills the GPU, else STREAM;
// binary64 (FFPS_F64, FFPS_F32_F64) —
//   SMALL  up to 4,608 points (4K: 0.82 ms vs 1.31 on GRID@1);
//   GRID on 1 CTA per cloud below 16K points (6K: 1.49-1.59 ms vs 1.94 on
//          SMALL; 8K: 1.73-1.84 vs 4.7), GRID beyond.
// FFPS_ALGO in the environment ("stream" / "small" / "bucket" / "grid")
// overrides AUTO.
constexpr int64_t kSmallMax = 8192;  // K1s: points per cloud at most

int auto_algo(int64_t n, int64_t batch, int dtype) {
  if (dtype != FFPS_F32) {
    if (n <= 4608) return FFPS_ALGO_SMALL;
    if (n < 16384) return FFPS_ALGO_GRID_CL(1);
    return FFPS_ALGO_GRID;
  }
  if (n <= kSmallMax) return FFPS_ALGO_SMALL;
  if (n >= 10000) return FFPS_ALGO_GRID;
  if ((n >= 6144 && batch >= 48) || (n >= 3072 && batch >= 96)) return FFPS_ALGO_BUCKET;
  return FFPS_ALGO_STREAM;
}

int resolve_algo(int algo, int64_t n, int64_t batch, int dtype) {
  if (algo == FFPS_ALGO_AUTO) {
    const char* force = getenv("FFPS_FORCE_PLAN");  // names a streaming configuration
    if (force && *force) return FFPS_ALGO_STREAM;
    const char* env = getenv("FFPS_ALGO");
    if (env && strcmp(env, "stream") == 0) return FFPS_ALGO_STREAM;
    if (env && strcmp(env, "bucket") == 0) return FFPS_ALGO_BUCKET;
    if (env && strcmp(env, "multi") == 0) return FFPS_ALGO_GRID;  // retired K1m: K1g
    if (env && strcmp(env, "grid") == 0) return FFPS_ALGO_GRID;
    if (env && strcmp(env, "small") == 0) return FFPS_ALGO_SMALL;
    return auto_algo(n, batch, dtype);
  }
  return algo;
}

// CTAs per cloud of the grid schedule: fixed by the algo argument
// (FFPS_ALGO_GRID_CL), else
//   4 for clouds of >= 40K points while batch * 4 <= SMs (crossover 37.5-42K:
//     37.5K 1-2% slower, 42K 1-2% faster, 50K 5-7% faster, 75K 18-19% faster,
//     binary32 and binary64 alike — profiles/r02_ab_cl4_crossover.txt,
//     r02_ab_cl4_top16_merge.txt, tools/sweep_strong.py),
//   2 for clouds of >= 20K points while batch * 2 <= SMs (each CTA keeps
//     >= 10 bucket groups for the KM = 16 candidates),
//   else 1.
// FFPS_GRID_CL in the environment overrides both.
int grid_cluster(int algo, int64_t batch, int sms, int64_t n) {
  int cl = algo >> 8;
  if (cl == 0) {
    if (n >= 40000 && batch * 4 <= sms) cl = 4;
    else if (n >= 20000 && batch * 2 <= sms) cl = 2;
    else cl = 1;
  }
  if (const char* v = getenv("FFPS_GRID_CL")) {
    const int w = atoi(v);
    if (w == 1 || w == 2 || w == 4) cl = w;
  }
  return cl;
}

}  // namespace

extern "C" {

int ffps_bucket_plan(int dtype, int64_t n, int64_t* out) {
  if ((dtype != FFPS_F32 && dtype != FFPS_F64 && dtype != FFPS_F32_F64) || n < 1 || !out)
    return fail(FFPS_EINVAL, "ffps_bucket_plan: bad arguments");
  if (dtype == FFPS_F32_F64) dtype = FFPS_F64;  // K1b runs on the widened cloud
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  BucketPlan bp;
  if (!make_bucket_plan(dev, dtype, n, &bp))
    return fail(FFPS_EUNSUPPORTED, "no bucketed configuration for n=%lld", (long long)n);
  out[0] = bp.inst->nt;
  out[1] = 32 * bp.inst->ppl;
  out[2] = bp.nbuckets;
  out[3] = bp.inst->nbt;
  return FFPS_OK;
}

int ffps_h2d_prefix(void* dst, const void* src_host, int64_t batch, int64_t n_prefix,
                    int64_t cloud_stride, int dtype, void* stream) {
  g_last_launches = 0;
  if ((dtype != FFPS_F32 && dtype != FFPS_F64 && dtype != FFPS_F32_F64) || batch < 0 ||
      n_prefix < 0 || cloud_stride < n_prefix)
    return fail(FFPS_EINVAL, "h2d_prefix: bad arguments");
  if (batch == 0 || n_prefix == 0) return FFPS_OK;
  if (!dst || !src_host) return fail(FFPS_EINVAL, "null pointer");
  const size_t esz = dtype == FFPS_F64 ? 8 : 4;  // coordinates as stored
  cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)n_prefix * 3 * esz, src_host,
                                    (size_t)cloud_stride * 3 * esz, (size_t)n_prefix * 3 * esz,
                                    (size_t)batch, cudaMemcpyHostToDevice,
                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync");
  return FFPS_OK;
}

int ffps_d2h_prefix(void* dst_host, int64_t dst_stride, const void* src, int64_t src_stride,
                    int64_t batch, int64_t n_prefix, int64_t elem_bytes, void* stream) {
  g_last_launches = 0;
  if (batch < 0 || n_prefix < 0 || elem_bytes < 1 || dst_stride < n_prefix ||
      src_stride < n_prefix)
    return fail(FFPS_EINVAL, "d2h_prefix: bad arguments");
  if (batch == 0 || n_prefix == 0) return FFPS_OK;
  if (!dst_host || !src) return fail(FFPS_EINVAL, "null pointer");
  cudaError_t e = cudaMemcpy2DAsync(dst_host, (size_t)(dst_stride * elem_bytes), src,
                                    (size_t)(src_stride * elem_bytes),
                                    (size_t)(n_prefix * elem_bytes), (size_t)batch,
                                    cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync");
  return FFPS_OK;
}

int ffps_auto_schedule_ex(int64_t n, int64_t batch, int dtype) {
  const int a = resolve_algo(FFPS_ALGO_AUTO, n, batch, dtype);
  if ((a & 0xff) != FFPS_ALGO_GRID) return a;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return a;
  }
  int cl = 0;
  choose_grid(dtype, n, batch, a, dev, &cl);
  return FFPS_ALGO_GRID_CL(cl);
}

int ffps_grid_plan(int dtype, int64_t n, int64_t batch, int algo, int64_t* out) {
  if ((dtype != FFPS_F32 && dtype != FFPS_F64 && dtype != FFPS_F32_F64) || n < 1 || batch < 1 ||
      !out)
    return fail(FFPS_EINVAL, "ffps_grid_plan: bad arguments");
  if (algo == FFPS_ALGO_AUTO) algo = FFPS_ALGO_GRID;
  if ((algo & 0xff) != FFPS_ALGO_GRID)
    return fail(FFPS_EINVAL, "ffps_grid_plan: algo must be AUTO or a grid schedule");
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int cl = 0;
  const GridPick g = choose_grid(dtype, n, batch, algo, dev, &cl);
  if (!g.inst) return fail(FFPS_EUNSUPPORTED, "no grid configuration for n=%lld", (long long)n);
  out[0] = cl;
  out[1] = g.inst->ppl;
  out[2] = g.nb;
  out[3] = (int64_t)g.smem;
  return FFPS_OK;
}

int ffps_auto_schedule(int64_t n, int64_t batch) {
  return ffps_auto_schedule_ex(n, batch, FFPS_F32);
}

}  // extern "C"

namespace {

bool valid_dtype(int dtype) {
  return dtype == FFPS_F32 || dtype == FFPS_F64 || dtype == FFPS_F32_F64;
}

int dispatch(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n,
             int64_t iters, const int64_t* seed_pos, const int64_t* index_map,
             int64_t map_stride, int64_t* order, void* sel_d2, int64_t out_stride,
             cudaStream_t st, int dev, int a, bool from_auto, int64_t* stats);

// FFPS_F32_F64 on a schedule without float-coordinate kernels: widen the rows
// the run can read (the prefix [0, n), or the whole cloud for restricted
// runs) into binary64 scratch, then run the binary64 kernels on it
int run_widened(const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n, int64_t iters,
                const int64_t* seed_pos, const int64_t* index_map, int64_t map_stride,
                int64_t* order, void* sel_d2, int64_t out_stride, cudaStream_t st, int dev,
                int a) {
  const int64_t rows = index_map ? cloud_stride : n;
  void* wide = nullptr;
  cudaError_t e = ffps::scratch_alloc(&wide, (size_t)batch * rows * 3 * sizeof(double), st);
  if (e != cudaSuccess) return cuda_fail(e, "scratch_alloc(widen)");
  e = ffps::launch_upcast(xyz, batch, cloud_stride, rows, wide, device_info(dev).sms, st);
  if (e != cudaSuccess) {
    ffps::scratch_free(wide, st);
    return cuda_fail(e, "upcast_kernel launch");
  }
  const int rc = dispatch(FFPS_F64, wide, batch, rows, n, iters, seed_pos, index_map, map_stride,
                          order, sel_d2, out_stride, st, dev, a, false, nullptr);
  e = ffps::scratch_free(wide, st);
  if (rc != FFPS_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "scratch_free(widen)");
  g_last_launches += 1;
  return FFPS_OK;
}

int dispatch(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n,
             int64_t iters, const int64_t* seed_pos, const int64_t* index_map,
             int64_t map_stride, int64_t* order, void* sel_d2, int64_t out_stride,
             cudaStream_t st, int dev, int a, bool from_auto, int64_t* stats) {
  if ((a & 0xff) == FFPS_ALGO_GRID) {
    const int rc = run_grid(dtype, xyz, batch, cloud_stride, n, iters, seed_pos, index_map,
                            map_stride, order, sel_d2, out_stride, st, dev, a, stats);
    if (rc != FFPS_EUNSUPPORTED || !from_auto) return rc;
    // AUTO: the cloud's bucket table does not fit shared memory -> the
    // streaming kernel, which spills the points beyond the cluster to HBM
    a = FFPS_ALGO_STREAM;
  }
  if (dtype == FFPS_F32_F64)
    return run_widened(xyz, batch, cloud_stride, n, iters, seed_pos, index_map, map_stride,
                       order, sel_d2, out_stride, st, dev, a);
  if (a == FFPS_ALGO_BUCKET)
    return run_bucketed(dtype, xyz, batch, cloud_stride, n, iters, seed_pos, index_map,
                        map_stride, order, sel_d2, out_stride, st, dev);
  if (a == FFPS_ALGO_SMALL && n <= kSmallMax)  // larger clouds: the streaming kernel
    return run_small(dtype, xyz, batch, cloud_stride, n, iters, seed_pos, index_map, map_stride,
                     order, sel_d2, out_stride, st);
  return run_streaming(dtype, xyz, batch, cloud_stride, n, iters, seed_pos, index_map,
                       map_stride, order, sel_d2, out_stride, st, dev);
}

int run_kernel_impl(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n,
                    int64_t iters, const int64_t* seed_pos, const int64_t* index_map,
                    int64_t map_stride, int64_t* order, void* sel_d2, int64_t out_stride,
                    void* stream, int algo, int64_t* stats) {
  g_last_launches = 0;
  if (!valid_dtype(dtype))
    return fail(FFPS_EINVAL, "dtype must be FFPS_F32, FFPS_F64 or FFPS_F32_F64");
  if (algo != FFPS_ALGO_AUTO && algo != FFPS_ALGO_STREAM && algo != FFPS_ALGO_BUCKET &&
      algo != FFPS_ALGO_MULTI && algo != FFPS_ALGO_GRID && algo != FFPS_ALGO_GRID_CL(1) &&
      algo != FFPS_ALGO_GRID_CL(2) && algo != FFPS_ALGO_GRID_CL(4) &&
      algo != FFPS_ALGO_SMALL)
    return fail(FFPS_EINVAL, "unknown algorithm %d", algo);
  if (batch < 0) return fail(FFPS_EINVAL, "batch=%lld < 0", (long long)batch);
  if (batch == 0) return FFPS_OK;
  if (!xyz || !seed_pos || !order || !sel_d2)
    return fail(FFPS_EINVAL, "null device pointer");
  if (n < 1 || n > 0x7fffffffLL) return fail(FFPS_EINVAL, "n=%lld out of range", (long long)n);
  if (iters < 1 || iters > n)  // fps_core.py:178-180
    return fail(FFPS_EINVAL, "m=%lld not in [1, %lld]", (long long)iters, (long long)n);
  if (out_stride < iters) return fail(FFPS_EINVAL, "out_stride < iters");
  if (index_map ? map_stride < n : cloud_stride < n)
    return fail(FFPS_EINVAL, "cloud/map stride smaller than n");
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  // FFPS_ALGO_MULTI (K1m, retired in round 2) runs the multi-winner K1g
  const int a = resolve_algo(algo == FFPS_ALGO_MULTI ? FFPS_ALGO_GRID : algo, n, batch, dtype);
  return dispatch(dtype, xyz, batch, cloud_stride, n, iters, seed_pos, index_map, map_stride,
                  order, sel_d2, out_stride, static_cast<cudaStream_t>(stream), dev, a,
                  algo == FFPS_ALGO_AUTO, stats);
}

}  // namespace

extern "C" {

int ffps_run_kernel_ex(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride,
                       int64_t n, int64_t iters, const int64_t* seed_pos,
                       const int64_t* index_map, int64_t map_stride, int64_t* order,
                       void* sel_d2, int64_t out_stride, void* stream, int algo) {
  return run_kernel_impl(dtype, xyz, batch, cloud_stride, n, iters, seed_pos, index_map,
                         map_stride, order, sel_d2, out_stride, stream, algo, nullptr);
}

int ffps_run_kernel_stats(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride,
                          int64_t n, int64_t iters, const int64_t* seed_pos,
                          const int64_t* index_map, int64_t map_stride, int64_t* order,
                          void* sel_d2, int64_t out_stride, void* stream, int algo,
                          int64_t* stats) {
  return run_kernel_impl(dtype, xyz, batch, cloud_stride, n, iters, seed_pos, index_map,
                         map_stride, order, sel_d2, out_stride, stream, algo, stats);
}

int ffps_run_kernel(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n,
                    int64_t iters, const int64_t* seed_pos, const int64_t* index_map,
                    int64_t map_stride, int64_t* order, void* sel_d2, int64_t out_stride,
                    void* stream) {
  return ffps_run_kernel_ex(dtype, xyz, batch, cloud_stride, n, iters, seed_pos, index_map,
                            map_stride, order, sel_d2, out_stride, stream, FFPS_ALGO_AUTO);
}

int ffps_coverage(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride, int64_t n,
                  const int64_t* idx, int64_t idx_stride, int64_t m, void* out_d2,
                  void* stream) {
  g_last_launches = 0;
  if (!valid_dtype(dtype))
    return fail(FFPS_EINVAL, "dtype must be FFPS_F32, FFPS_F64 or FFPS_F32_F64");
  if (batch < 0 || n < 1 || n > 0x7fffffffLL || m < 1 || m > 0x7fffffffLL)
    return fail(FFPS_EINVAL, "coverage: bad sizes");
  if (batch == 0) return FFPS_OK;
  if (!xyz || !idx || !out_d2) return fail(FFPS_EINVAL, "null device pointer");
  if (cloud_stride < n || idx_stride < m) return fail(FFPS_EINVAL, "stride smaller than size");
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  const DeviceInfo di = device_info(dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == FFPS_F32_F64) {  // binary64 on the widened cloud (exact)
    void* wide = nullptr;
    e = ffps::scratch_alloc(&wide, (size_t)batch * n * 3 * sizeof(double), st);
    if (e != cudaSuccess) return cuda_fail(e, "scratch_alloc(widen)");
    e = ffps::launch_upcast(xyz, batch, cloud_stride, n, wide, di.sms, st);
    int rc = e == cudaSuccess ? ffps_coverage(FFPS_F64, wide, batch, n, n, idx, idx_stride, m,
                                              out_d2, stream)
                              : cuda_fail(e, "upcast_kernel launch");
    const int64_t l = g_last_launches + 1;
    e = ffps::scratch_free(wide, st);
    if (rc == FFPS_OK && e != cudaSuccess) rc = cuda_fail(e, "scratch_free(widen)");
    g_last_launches = rc == FFPS_OK ? l : 0;
    return rc;
  }
  const size_t esz = dtype == FFPS_F32 ? 4 : 8;
  // sample buckets: boxes staged in shared memory -> bucket size from the budget
  int64_t bss = 32;
  while ((m + bss - 1) / bss * 6 * (int64_t)esz > (int64_t)di.smem_optin - 4096) bss *= 2;
  const int64_t bsp = 32;
  const int64_t nbp = (n + bsp - 1) / bsp, nbs = (m + bss - 1) / bss;
  const int64_t nsp = nbp * bsp, nss = nbs * bss;
  // per slot: X, Y, Z, D + O, and the K0 scratch TX, TY, TZ + TO
  const size_t per_p = (size_t)nsp * (7 * esz + 8) + (size_t)nbp * 6 * esz;
  const size_t per_s = (size_t)nss * (7 * esz + 8) + (size_t)nbs * 6 * esz;
  unsigned char* scratch = nullptr;
  e = ffps::scratch_alloc(reinterpret_cast<void**>(&scratch), (per_p + per_s) * (size_t)batch + 1024,
                      st);
  if (e != cudaSuccess) return cuda_fail(e, "scratch_alloc(coverage)");
  auto carve = [&](unsigned char* base, int64_t nslots, int64_t nb, int64_t bs,
                   ffps::BucketBuildParams& bb) {
    const size_t arr = (size_t)nslots * esz * (size_t)batch;
    bb.X = base;
    bb.Y = base + arr;
    bb.Z = base + 2 * arr;
    bb.D = base + 3 * arr;
    bb.BB = base + 4 * arr;
    bb.O = reinterpret_cast<int32_t*>(base + 4 * arr + box_bytes(nb, esz, batch));
    bb.nslots = nslots;
    bb.nbuckets = nb;
    bb.bs = bs;
    unsigned char* t = reinterpret_cast<unsigned char*>(bb.O) + (size_t)nslots * 4 * (size_t)batch;
    bb.TX = t;
    bb.TY = t + arr;
    bb.TZ = t + 2 * arr;
    bb.TO = reinterpret_cast<int32_t*>(t + 3 * arr);
  };
  ffps::BucketBuildParams bp{}, bs{};
  bp.xyz = xyz;
  bp.cloud_stride = cloud_stride;
  bp.index_map = nullptr;
  bp.map_stride = 0;
  bp.n = n;
  carve(scratch, nsp, nbp, bsp, bp);
  bs.xyz = xyz;
  bs.cloud_stride = cloud_stride;
  bs.index_map = idx;
  bs.map_stride = idx_stride;
  bs.n = m;
  carve(scratch + per_p * (size_t)batch + 256, nss, nbs, bss, bs);
  int launches = 0;
  e = ffps::launch_bucket_build(dtype, bp, batch, st);
  if (e == cudaSuccess) {
    launches += ffps::bucket_build_launches(bp);
    e = ffps::launch_bucket_build(dtype, bs, batch, st);
  }
  if (e == cudaSuccess) {
    launches += ffps::bucket_build_launches(bs);
    e = cudaMemsetAsync(out_d2, 0, (size_t)batch * esz, st);
  }
  if (e == cudaSuccess) {
    ffps::CoverageParams cp;
    cp.pX = bp.X;
    cp.pY = bp.Y;
    cp.pZ = bp.Z;
    cp.pBB = bp.BB;
    cp.p_nslots = nsp;
    cp.p_nbuckets = nbp;
    cp.p_bs = bsp;
    cp.sX = bs.X;
    cp.sY = bs.Y;
    cp.sZ = bs.Z;
    cp.sBB = bs.BB;
    cp.s_nslots = nss;
    cp.s_nbuckets = nbs;
    cp.s_bs = bss;
    cp.out = out_d2;
    e = ffps::launch_coverage(dtype, cp, batch, di.sms, st);
    if (e == cudaSuccess) ++launches;
  }
  cudaError_t e2 = ffps::scratch_free(scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "coverage launch");
  if (e2 != cudaSuccess) return cuda_fail(e2, "scratch_free(coverage)");
  g_last_launches = launches;
  return FFPS_OK;
}

int ffps_fill_slice(int dtype, int64_t* order, void* sel_d2, int64_t batch, int64_t out_stride,
                    int64_t k, int64_t m1, void* stream) {
  g_last_launches = 0;
  if (!valid_dtype(dtype))
    return fail(FFPS_EINVAL, "dtype must be FFPS_F32, FFPS_F64 or FFPS_F32_F64");
  if (dtype == FFPS_F32_F64) dtype = FFPS_F64;  // sel_d2 is binary64
  if (batch < 0 || k < 1 || m1 < k || out_stride < m1)
    return fail(FFPS_EINVAL, "fill: need 1 <= k <= m1 <= out_stride");
  if (batch == 0 || m1 == k) return FFPS_OK;
  if (!order || !sel_d2) return fail(FFPS_EINVAL, "null device pointer");
  cudaError_t e = ffps::launch_fill_slice(dtype, order, sel_d2, batch, out_stride, k, m1,
                                          static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fill_slice_kernel launch");
  g_last_launches = 1;
  return FFPS_OK;
}

int ffps_fill_random(int dtype, int64_t* order, void* sel_d2, int64_t batch, int64_t out_stride,
                     int64_t n, int64_t k, int64_t m1, uint64_t state_hi, uint64_t state_lo,
                     uint64_t inc_hi, uint64_t inc_lo, void* stream) {
  g_last_launches = 0;
  if (!valid_dtype(dtype))
    return fail(FFPS_EINVAL, "dtype must be FFPS_F32, FFPS_F64 or FFPS_F32_F64");
  if (dtype == FFPS_F32_F64) dtype = FFPS_F64;  // sel_d2 is binary64
  if (batch < 0 || k < 1 || m1 < k || out_stride < m1 || n < m1)
    return fail(FFPS_EINVAL, "fill: need 1 <= k <= m1 <= min(n, out_stride)");
  if (n >= 0x7fffffffLL) return fail(FFPS_EUNSUPPORTED, "fill: n must be < 2^31");
  if (batch == 0 || m1 == k) return FFPS_OK;
  if (!order || !sel_d2) return fail(FFPS_EINVAL, "null device pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t words = ffps::fill_random_scratch_words(n, k, m1);
  uint32_t* scratch = nullptr;
  cudaError_t e = ffps::scratch_alloc(reinterpret_cast<void**>(&scratch),
                                  (size_t)words * 4 * (size_t)batch, st);
  if (e != cudaSuccess) return cuda_fail(e, "scratch_alloc(fill_random)");
  const uint64_t pcg[4] = {state_hi, state_lo, inc_hi, inc_lo};
  // FFPS_FILL_SEQUENTIAL=1 (tests): the single-thread generator that backs up
  // the warp-parallel one when Lemire rejections outrun its value stream
  const char* seq = getenv("FFPS_FILL_SEQUENTIAL");
  e = ffps::launch_fill_random(dtype, order, sel_d2, batch, out_stride, n, k, m1, pcg, scratch,
                               st, seq && strcmp(seq, "1") == 0);
  cudaError_t e2 = ffps::scratch_free(scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "fill_random_kernel launch");
  if (e2 != cudaSuccess) return cuda_fail(e2, "scratch_free(fill_random)");
  g_last_launches = 1;
  return FFPS_OK;
}

int ffps_hierarchical_sample(int dtype, const void* xyz, int64_t batch, int64_t cloud_stride,
                             int64_t n, const int64_t* budgets, int nlayers, int64_t k,
                             int64_t c, int fill_mode, const uint64_t* pcg,
                             int cache_enabled, const int64_t* seed_pos, int64_t* const* order,
                             void* const* sel_d2, void* stream) {
  if (!budgets || nlayers < 1 || !order || !sel_d2)
    return fail(FFPS_EINVAL, "hierarchical_sample: need budgets and per-layer outputs");
  const int64_t m1 = budgets[0];
  for (int l = 0; l < nlayers; ++l) {
    if (budgets[l] < 1 || (l > 0 && budgets[l] > budgets[l - 1]))  // fps_cache.py:42-50
      return fail(FFPS_EINVAL, "budgets must be >= 1 and non-increasing");
    if ((l == 0 || !cache_enabled) && (!order[l] || !sel_d2[l]))
      return fail(FFPS_EINVAL, "layer %d output is NULL", l);
  }
  if (m1 > n || k < 1 || k > m1 || c < k || c > n)  // fps_prune.py:45-51,78-88
    return fail(FFPS_EINVAL, "need 1 <= k <= m1 <= n and k <= c <= n");
  if (fill_mode != 0 && fill_mode != 1) return fail(FFPS_EINVAL, "fill_mode must be 0 or 1");
  if (fill_mode == 1 && m1 > k && !pcg) return fail(FFPS_EINVAL, "random fill needs the PCG64 state");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t launches = 0;
  // layer 1: FPS-Prune = greedy over the candidate prefix, then the fill
  int rc = run_kernel_impl(dtype, xyz, batch, cloud_stride, c, k, seed_pos, nullptr, 0, order[0],
                           sel_d2[0], m1, stream, FFPS_ALGO_AUTO, nullptr);
  if (rc != FFPS_OK) return rc;
  launches += g_last_launches;
  if (m1 > k) {
    rc = fill_mode == 0 ? ffps_fill_slice(dtype, order[0], sel_d2[0], batch, m1, k, m1, stream)
                        : ffps_fill_random(dtype, order[0], sel_d2[0], batch, m1, n, k, m1,
                                           pcg[0], pcg[1], pcg[2], pcg[3], stream);
    if (rc != FFPS_OK) return rc;
    launches += g_last_launches;
  }
  // cache off: every deeper layer re-runs exact FPS over the previous layer's
  // points in its order, seeded at position 0 (fps_cache.py:227-232,189-201);
  // K0 gathers them through the previous layer's indices
  if (!cache_enabled && nlayers > 1) {
    int64_t* zeros = nullptr;
    cudaError_t e = ffps::scratch_alloc(reinterpret_cast<void**>(&zeros),
                                        (size_t)batch * sizeof(int64_t), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(zeros, 0, (size_t)batch * sizeof(int64_t), st);
    if (e != cudaSuccess) return cuda_fail(e, "hierarchical_sample: seed scratch");
    for (int l = 1; l < nlayers && rc == FFPS_OK; ++l) {
      rc = run_kernel_impl(dtype, xyz, batch, cloud_stride, budgets[l - 1], budgets[l], zeros,
                           order[l - 1], budgets[l - 1], order[l], sel_d2[l], budgets[l], stream,
                           FFPS_ALGO_AUTO, nullptr);
      launches += g_last_launches;
    }
    e = ffps::scratch_free(zeros, st);
    if (rc != FFPS_OK) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "scratch_free(seeds)");
  }
  g_last_launches = launches;
  return FFPS_OK;
}

}  // extern "C"
