// K5 — covering radius of a sample (reference metrics.py:29-52):
//     coverage_d2 = max over cloud points p of  min over sampled points s of d2(p, s)
// with d2 the reference's separately rounded ((dx*dx + dy*dy) + dz*dz)
// (fps_core.py:74-83 via metrics.py:39).  Max and min are exact, so the result
// is bit-identical to the reference for every schedule; the host takes the
// square root (metrics.py:52).
//
// Inputs are the K0 buckets of the cloud (points) and of the sample (gathered
// through the index list).  One warp per point bucket, lanes = points:
//   1. the sample-bucket boxes of the cloud are staged in shared memory;
//   2. the warp first evaluates the sample bucket whose box is closest to its
//      own box (tight initial bound), then scans all sample buckets 32 at a
//      time: lane l tests bucket 32c+l with the exact box-box lower bound
//      (RN-monotone, as in K1b) against the warp's current max(best) and only
//      flagged buckets are evaluated (samples broadcast by shuffle);
//   3. warp max -> atomicMax on the non-negative distance bits of the cloud.
// Padding slots of both bucket sets repeat a real point, so they change
// neither a min nor the max.
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"
#include "ffps_internal.h"

namespace ffps {

constexpr int kCovThreads = 256;
constexpr int kCovWarps = kCovThreads / 32;

// exact lower bound of d2(p, s) over p in box a, s in box b ({lo.xyz, hi.xyz}):
// per axis g = max(RN(a.lo - b.hi), RN(b.lo - a.hi), 0) <= |RN(p - s)| (RN is
// monotone and odd), then the reference's rounded square-sum (monotone)
__device__ __forceinline__ float box_box_d2(const float* a, const float* b) {
  const float gx = max3f(__fsub_rn(a[0], b[3]), __fsub_rn(b[0], a[3]), 0.0f);
  const float gy = max3f(__fsub_rn(a[1], b[4]), __fsub_rn(b[1], a[4]), 0.0f);
  const float gz = max3f(__fsub_rn(a[2], b[5]), __fsub_rn(b[2], a[5]), 0.0f);
  return __fadd_rn(__fadd_rn(__fmul_rn(gx, gx), __fmul_rn(gy, gy)), __fmul_rn(gz, gz));
}
__device__ __forceinline__ double box_box_d2(const double* a, const double* b) {
  const double gx = fmax(fmax(__dsub_rn(a[0], b[3]), __dsub_rn(b[0], a[3])), 0.0);
  const double gy = fmax(fmax(__dsub_rn(a[1], b[4]), __dsub_rn(b[1], a[4])), 0.0);
  const double gz = fmax(fmax(__dsub_rn(a[2], b[5]), __dsub_rn(b[2], a[5])), 0.0);
  return __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
}

template <typename T>
__global__ void __launch_bounds__(kCovThreads) coverage_kernel(const CoverageParams prm) {
  using A = Arith<T>;
  extern __shared__ __align__(16) unsigned char smem[];
  T* sbox = reinterpret_cast<T*>(smem);  // [nbs][6]
  const int b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nbp = (int)prm.p_nbuckets, nbs = (int)prm.s_nbuckets;
  const int bsp = (int)prm.p_bs, bss = (int)prm.s_bs;
  const T* __restrict__ PX = static_cast<const T*>(prm.pX) + (int64_t)b * prm.p_nslots;
  const T* __restrict__ PY = static_cast<const T*>(prm.pY) + (int64_t)b * prm.p_nslots;
  const T* __restrict__ PZ = static_cast<const T*>(prm.pZ) + (int64_t)b * prm.p_nslots;
  const T* __restrict__ PB = static_cast<const T*>(prm.pBB) + (int64_t)b * nbp * 6;
  const T* __restrict__ SX = static_cast<const T*>(prm.sX) + (int64_t)b * prm.s_nslots;
  const T* __restrict__ SY = static_cast<const T*>(prm.sY) + (int64_t)b * prm.s_nslots;
  const T* __restrict__ SZ = static_cast<const T*>(prm.sZ) + (int64_t)b * prm.s_nslots;
  const T* __restrict__ SB = static_cast<const T*>(prm.sBB) + (int64_t)b * nbs * 6;
  for (int i = tid; i < nbs * 6; i += kCovThreads) sbox[i] = SB[i];
  __syncthreads();

  T wmax_all = T(0);
  for (int q = blockIdx.x * kCovWarps + warp; q < nbp; q += gridDim.x * kCovWarps) {
    T pbox[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) pbox[c] = PB[(int64_t)q * 6 + c];
    for (int g0 = 0; g0 < bsp; g0 += 32) {
      const int64_t ps = (int64_t)q * bsp + g0 + lane;
      const T px = PX[ps], py = PY[ps], pz = PZ[ps];
      T best = A::pinf();
      auto eval = [&](int j) {  // all lanes: min over the samples of bucket j
        for (int h0 = 0; h0 < bss; h0 += 32) {
          const int64_t ss = (int64_t)j * bss + h0 + lane;
          const T sx = SX[ss], sy = SY[ss], sz = SZ[ss];
#pragma unroll 8
          for (int t = 0; t < 32; ++t) {
            const T qx = __shfl_sync(0xffffffffu, sx, t);
            const T qy = __shfl_sync(0xffffffffu, sy, t);
            const T qz = __shfl_sync(0xffffffffu, sz, t);
            best = A::vmin(best, A::d2(px, py, pz, qx, qy, qz));  // metrics.py:39-41
          }
        }
      };
      // closest sample box first (warp argmin of the box-box bound)
      {
        T lbmin = A::pinf();
        int jmin = 0;
        for (int c0 = 0; c0 < nbs; c0 += 32) {
          const int j = c0 + lane;
          if (j < nbs) {
            const T lb = box_box_d2(pbox, sbox + (size_t)j * 6);
            if (lb < lbmin) {
              lbmin = lb;
              jmin = j;
            }
          }
        }
        const auto key = A::bits(lbmin);
        const auto km = -A::warp_max(-key);  // min over lanes (non-negative bits)
        const int wl = __ffs(__ballot_sync(0xffffffffu, key == km)) - 1;
        eval(__shfl_sync(0xffffffffu, jmin, wl));
      }
      // every sample bucket that can still lower some lane's best
      for (int c0 = 0; c0 < nbs; c0 += 32) {
        const T wb = A::from_bits(A::warp_max(A::bits(best)));
        const int j = c0 + lane;
        const bool f = j < nbs && box_box_d2(pbox, sbox + (size_t)j * 6) < wb;
        unsigned m = __ballot_sync(0xffffffffu, f);
        while (m) {
          const int l = __ffs(m) - 1;
          m &= m - 1u;
          eval(c0 + l);
        }
      }
      wmax_all = A::vmax(wmax_all, best);
    }
  }
  const auto wm = A::warp_max(A::bits(wmax_all));
  if (lane == 0) {
    if (sizeof(T) == 4)
      atomicMax(reinterpret_cast<int*>(prm.out) + b, (int)wm);
    else
      atomicMax(reinterpret_cast<unsigned long long*>(prm.out) + b, (unsigned long long)wm);
  }
}

cudaError_t launch_coverage(int dtype, const CoverageParams& p, int64_t batch, int sms,
                            cudaStream_t st) {
  const size_t esz = dtype == 0 ? 4 : 8;
  const size_t smem = (size_t)p.s_nbuckets * 6 * esz;
  const void* fn = dtype == 0 ? reinterpret_cast<const void*>(&coverage_kernel<float>)
                              : reinterpret_cast<const void*>(&coverage_kernel<double>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  // enough blocks per cloud to cover the SMs a few times over
  int64_t per_cloud = (p.p_nbuckets + kCovWarps - 1) / kCovWarps;
  const int64_t want = ((int64_t)sms * 4 + batch - 1) / batch;
  if (per_cloud > want) per_cloud = want;
  if (per_cloud < 1) per_cloud = 1;
  void* args[] = {const_cast<CoverageParams*>(&p)};
  return cudaLaunchKernel(fn, dim3((unsigned)per_cloud, (unsigned)batch), dim3(kCovThreads),
                          args, smem, st);
}

}  // namespace ffps
