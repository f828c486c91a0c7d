// K0 — spatial bucketing of the point set of every cloud (input of K1b).
//
// One CTA per cloud.  The points taking part in a greedy run (the candidate
// prefix xyz[b][0:n), fps_prune.py:54-65,92, or the gathered points
// xyz[b][index_map[b][i]], fps_cache.py:195) are counting-sorted by the
// Morton-ordered cell of a 32^3 grid over the cloud's bounding box, then cut
// into buckets of BS consecutive points.  The output is bucket-major SoA in
// global memory (L2-resident at the benchmark sizes):
//     X, Y, Z, D  [nb * BS]   coordinates and running min distance (+inf)
//     O           [nb * BS]   position of the point in the run's point list
//     BB          [nb][6]     bucket bounding box {lo.xyz, hi.xyz}
// Padding slots (>= n) repeat the first point of the last bucket (so they do
// not widen its box) with D = -inf: they can never be selected.
//
// The order of points inside a cell depends on atomic arrival order.  That
// is harmless: K1b breaks ties by the point's position O, never by slot, so
// the sampled indices are independent of the layout.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "ffps_internal.h"

namespace ffps {

constexpr int kBuildThreads = 1024;
constexpr int kGridBits = 5;                          // 32 cells per axis
constexpr int kCells = 1 << (3 * kGridBits);          // 32768 cells
constexpr int kSubBits = 3;                           // 8^3 sub-cells in a crowded cell
constexpr int kSub = 1 << (3 * kSubBits);
constexpr int kCrowd = 64;                            // cells above this are refined

__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 5 bits -> every 3rd bit
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < kGridBits; ++i) r |= ((v >> i) & 1u) << (3 * i);
  return r;
}

template <typename T>
__device__ __forceinline__ int cell_of(T v, T lo, T inv) {
  int c = (int)((v - lo) * inv);
  return c < 0 ? 0 : (c >= (1 << kGridBits) ? (1 << kGridBits) - 1 : c);
}

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_maxv(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}

template <typename T>
__global__ void __launch_bounds__(kBuildThreads, 1) bucket_build_kernel(const BucketBuildParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);  // [kCells]
  __shared__ T red[6][kBuildThreads / 32];
  __shared__ T box[6];
  __shared__ uint32_t part[kBuildThreads];

  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (int)p.n;
  const T* X0 = static_cast<const T*>(p.xyz) + (int64_t)b * p.cloud_stride * 3;
  const int64_t* map = p.index_map ? p.index_map + (int64_t)b * p.map_stride : nullptr;
  const int64_t base = (int64_t)b * p.nslots;
  T* X = static_cast<T*>(p.X) + base;
  T* Y = static_cast<T*>(p.Y) + base;
  T* Z = static_cast<T*>(p.Z) + base;
  // D is T, or double under FFPS_F32_F64 (float coordinates, binary64 keys)
  auto put_d = [&](int64_t i, T v) {
    if (sizeof(T) == 4 && p.d_wide) static_cast<double*>(p.D)[base + i] = (double)v;
    else static_cast<T*>(p.D)[base + i] = v;
  };
  int32_t* O = p.O + base;
  T* BB = static_cast<T*>(p.BB) + (int64_t)b * p.nbuckets * 6;

  auto load = [&](int i, T& x, T& y, T& z) {
    const int64_t s = map ? __ldg(map + i) : i;
    x = X0[3 * s + 0];
    y = X0[3 * s + 1];
    z = X0[3 * s + 2];
  };

  // 1. bounding box of the run's points
  T mn[3], mx[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    mn[c] = (T)INFINITY;
    mx[c] = (T)-INFINITY;
  }
  for (int i = tid; i < n; i += kBuildThreads) {
    T v[3];
    load(i, v[0], v[1], v[2]);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      mn[c] = v[c] < mn[c] ? v[c] : mn[c];
      mx[c] = v[c] > mx[c] ? v[c] : mx[c];
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    mn[c] = warp_min(mn[c]);
    mx[c] = warp_maxv(mx[c]);
    if (lane == 0) {
      red[c][warp] = mn[c];
      red[3 + c][warp] = mx[c];
    }
  }
  for (int i = tid; i < kCells; i += kBuildThreads) hist[i] = 0;
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      T a = lane < kBuildThreads / 32 ? red[c][lane] : (T)INFINITY;
      T z = lane < kBuildThreads / 32 ? red[3 + c][lane] : (T)-INFINITY;
      a = warp_min(a);
      z = warp_maxv(z);
      if (lane == 0) {
        box[c] = a;
        box[3 + c] = z;
      }
    }
  }
  __syncthreads();
  T lo[3], inv[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    lo[c] = box[c];
    const T ext = box[3 + c] - box[c];
    inv[c] = ext > (T)0 ? (T)(1 << kGridBits) / ext : (T)0;
  }
  auto cell = [&](T x, T y, T z) -> uint32_t {
    return spread3((uint32_t)cell_of(x, lo[0], inv[0])) |
           (spread3((uint32_t)cell_of(y, lo[1], inv[1])) << 1) |
           (spread3((uint32_t)cell_of(z, lo[2], inv[2])) << 2);
  };

  // 2. histogram of cells
  for (int i = tid; i < n; i += kBuildThreads) {
    T x, y, z;
    load(i, x, y, z);
    atomicAdd(&hist[cell(x, y, z)], 1u);
  }
  __syncthreads();

  // 3. exclusive scan of the histogram (32 cells per thread)
  constexpr int kPer = kCells / kBuildThreads;
  uint32_t loc[kPer], sum = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    loc[j] = hist[tid * kPer + j];
    sum += loc[j];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) part[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = lane < kBuildThreads / 32 ? part[lane] : 0u;
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += u;
    }
    if (lane < kBuildThreads / 32) part[lane] = ti - t;
  }
  __syncthreads();
  uint32_t run = part[warp] + incl - sum;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    hist[tid * kPer + j] = run;
    run += loc[j];
  }
  __syncthreads();

  // 4. scatter into bucket-major SoA
  const T pinf = (T)INFINITY;
  for (int i = tid; i < n; i += kBuildThreads) {
    T x, y, z;
    load(i, x, y, z);
    const uint32_t s = atomicAdd(&hist[cell(x, y, z)], 1u);
    X[s] = x;
    Y[s] = y;
    Z[s] = z;
    put_d(s, pinf);
    O[s] = i;
  }
  __syncthreads();  // global writes of the block visible to the block

  // 4b. second level: inside every crowded cell (> kCrowd points; skewed
  //     densities such as LiDAR frames) order the points by the Morton code of
  //     an 8^3 grid over the cell's own box.  One warp per cell, per-warp
  //     histogram in shared memory, scatter through the T* scratch arrays.
  if (p.TX != nullptr) {
    uint32_t* sub = hist + kCells + warp * kSub;  // [kSub] per warp
    T* TX = static_cast<T*>(p.TX) + base;
    T* TY = static_cast<T*>(p.TY) + base;
    T* TZ = static_cast<T*>(p.TZ) + base;
    int32_t* TO = p.TO + base;
    for (int c = warp; c < kCells; c += kBuildThreads / 32) {
      const int beg = c == 0 ? 0 : (int)hist[c - 1];
      const int end = (int)hist[c];
      if (end - beg <= kCrowd) continue;
      T a[3] = {pinf, pinf, pinf}, zz[3] = {-pinf, -pinf, -pinf};
      for (int i = beg + lane; i < end; i += 32) {
        const T v[3] = {X[i], Y[i], Z[i]};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          a[d] = v[d] < a[d] ? v[d] : a[d];
          zz[d] = v[d] > zz[d] ? v[d] : zz[d];
        }
      }
      T sinv[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        a[d] = warp_min(a[d]);
        zz[d] = warp_maxv(zz[d]);
        const T ext = zz[d] - a[d];
        sinv[d] = ext > (T)0 ? (T)(1 << kSubBits) / ext : (T)0;
      }
      auto scell = [&](T x, T y, T z) -> uint32_t {
        auto cc = [&](T v, int d) {
          int q = (int)((v - a[d]) * sinv[d]);
          return (uint32_t)(q < 0 ? 0 : (q >= (1 << kSubBits) ? (1 << kSubBits) - 1 : q));
        };
        uint32_t r = 0;
#pragma unroll
        for (int i = 0; i < kSubBits; ++i)
          r |= (((cc(x, 0) >> i) & 1u) << (3 * i)) | (((cc(y, 1) >> i) & 1u) << (3 * i + 1)) |
               (((cc(z, 2) >> i) & 1u) << (3 * i + 2));
        return r;
      };
      for (int i = lane; i < kSub; i += 32) sub[i] = 0;
      __syncwarp();
      for (int i = beg + lane; i < end; i += 32) atomicAdd(&sub[scell(X[i], Y[i], Z[i])], 1u);
      __syncwarp();
      // exclusive scan of the kSub counters (kSub / 32 per lane)
      constexpr int kPerLane = kSub / 32;
      uint32_t loc[kPerLane], sum = 0;
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        loc[j] = sub[lane * kPerLane + j];
        sum += loc[j];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      uint32_t run = (uint32_t)beg + incl - sum;
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        sub[lane * kPerLane + j] = run;
        run += loc[j];
      }
      __syncwarp();
      for (int i = beg + lane; i < end; i += 32) {
        const T x = X[i], y = Y[i], z = Z[i];
        const int32_t o = O[i];
        const uint32_t s = atomicAdd(&sub[scell(x, y, z)], 1u);
        TX[s] = x;
        TY[s] = y;
        TZ[s] = z;
        TO[s] = o;
      }
      __syncwarp();
      for (int i = beg + lane; i < end; i += 32) {
        X[i] = TX[i];
        Y[i] = TY[i];
        Z[i] = TZ[i];
        O[i] = TO[i];
      }
      __syncwarp();
    }
    __syncthreads();
  }

  // 5. padding of the last bucket
  const int first_last = (int)((p.nbuckets - 1) * p.bs);
  for (int s = n + tid; s < (int)p.nslots; s += kBuildThreads) {
    X[s] = X[first_last];
    Y[s] = Y[first_last];
    Z[s] = Z[first_last];
    put_d(s, -pinf);
    O[s] = -1;
  }
  __syncthreads();

  // 6. bucket bounding boxes, one warp per bucket
  for (int q = warp; q < (int)p.nbuckets; q += kBuildThreads / 32) {
    T a[3] = {pinf, pinf, pinf}, z[3] = {-pinf, -pinf, -pinf};
    for (int u = lane; u < (int)p.bs; u += 32) {
      const int s = q * (int)p.bs + u;
      const T v[3] = {X[s], Y[s], Z[s]};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a[c] = v[c] < a[c] ? v[c] : a[c];
        z[c] = v[c] > z[c] ? v[c] : z[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      a[c] = warp_min(a[c]);
      z[c] = warp_maxv(z[c]);
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        BB[(int64_t)q * 6 + c] = a[c];
        BB[(int64_t)q * 6 + 3 + c] = z[c];
      }
    }
  }
}

size_t bucket_build_smem() {
  return (size_t)(kCells + (kBuildThreads / 32) * kSub) * sizeof(uint32_t);
}

int bucket_build_launches(const BucketBuildParams& p) {
  const char* kind = getenv("FFPS_BUCKET_BUILD");
  return (p.TX != nullptr && !(kind && strcmp(kind, "morton") == 0)) ? 2 : 1;
}

cudaError_t launch_bucket_build(int dtype, const BucketBuildParams& p, int64_t batch,
                                cudaStream_t st) {
  // default: kd-tree leaves (bucket_kd.cu; needs the TX..TO scratch);
  // FFPS_BUCKET_BUILD=morton selects the Morton-grid build below
  const char* kind = getenv("FFPS_BUCKET_BUILD");
  if (p.TX != nullptr && !(kind && strcmp(kind, "morton") == 0))
    return launch_bucket_kd(dtype, p, batch, st);
  const void* fn = dtype == 0 ? reinterpret_cast<const void*>(&bucket_build_kernel<float>)
                              : reinterpret_cast<const void*>(&bucket_build_kernel<double>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bucket_build_smem());
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<BucketBuildParams*>(&p)};
  return cudaLaunchKernel(fn, dim3((unsigned)batch), dim3(kBuildThreads), args,
                          bucket_build_smem(), st);
}

}  // namespace ffps
