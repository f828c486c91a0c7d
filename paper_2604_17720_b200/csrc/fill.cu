// K2 — budget fill, FillMode.DETERMINISTIC_SLICE (reference
// pkg/src/flashfps/fps_prune.py:96-100, 104-105): after a truncated greedy run
// of k iterations, append the first fill_n = m1 - k ascending indices of the
// cloud that the greedy run did not select; their selection distance is 0.
//
// Because at most k of the indices [0, m1) are selected, the fill always lies
// inside [0, m1): one CTA per cloud builds a selection bitmap of that range in
// shared memory (chunked for very large m1) and emits the zero bits in
// ascending order with a block-wide exclusive scan of per-thread zero counts.
#include <cuda_runtime.h>

#include <cstdint>

#include "ffps_internal.h"

namespace ffps {

constexpr int kFillThreads = 1024;
constexpr int64_t kFillChunkWords = 8192;  // 32 KiB bitmap = 262144 indices per chunk

__global__ void __launch_bounds__(kFillThreads) fill_slice_kernel(int64_t* order_all,
                                                                  void* sel_all, int f64,
                                                                  int64_t out_stride,
                                                                  int64_t k, int64_t m1) {
  __shared__ uint32_t bitmap[kFillChunkWords];
  __shared__ int64_t warp_tot[kFillThreads / 32];
  __shared__ int64_t s_written;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t* order = order_all + (int64_t)blockIdx.x * out_stride;
  const int64_t fill_n = m1 - k;
  if (tid == 0) s_written = 0;

  for (int64_t c0 = 0; c0 < m1; c0 += kFillChunkWords * 32) {
    __syncthreads();
    if (s_written >= fill_n) break;
    const int64_t clen = (m1 - c0) < kFillChunkWords * 32 ? (m1 - c0) : kFillChunkWords * 32;
    const int64_t nwords = (clen + 31) / 32;
    for (int64_t w = tid; w < nwords; w += kFillThreads) bitmap[w] = 0u;
    __syncthreads();
    for (int64_t i = tid; i < k; i += kFillThreads) {
      const int64_t o = order[i] - c0;
      if (o >= 0 && o < clen) atomicOr(&bitmap[o >> 5], 1u << (o & 31));
    }
    __syncthreads();
    // contiguous word range per thread keeps the emission ascending
    const int64_t wpt = (nwords + kFillThreads - 1) / kFillThreads;
    const int64_t w_lo = tid * wpt;
    const int64_t w_hi = (w_lo + wpt) < nwords ? (w_lo + wpt) : nwords;
    int64_t cnt = 0;
    for (int64_t w = w_lo; w < w_hi; ++w) {
      uint32_t free_bits = ~bitmap[w];
      const int64_t valid = clen - w * 32;
      if (valid < 32) free_bits &= (1u << valid) - 1u;
      cnt += __popc(free_bits);
    }
    // block exclusive scan of cnt
    int64_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t t = warp_tot[lane];
      int64_t ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += u;
      }
      warp_tot[lane] = ti - t;  // exclusive per-warp offsets
    }
    __syncthreads();
    const int64_t written = s_written;
    int64_t pos = written + warp_tot[warp] + (incl - cnt);
    for (int64_t w = w_lo; w < w_hi && pos < fill_n; ++w) {
      uint32_t free_bits = ~bitmap[w];
      const int64_t valid = clen - w * 32;
      if (valid < 32) free_bits &= (1u << valid) - 1u;
      while (free_bits && pos < fill_n) {
        const int bit = __ffs(free_bits) - 1;
        free_bits &= free_bits - 1u;
        order[k + pos] = c0 + w * 32 + bit;
        ++pos;
      }
    }
    __syncthreads();
    if (tid == kFillThreads - 1) s_written = written + warp_tot[warp] + incl;
  }
  // fill entries carry selection distance 0 (fps_prune.py:105)
  if (f64) {
    double* sel = static_cast<double*>(sel_all) + (int64_t)blockIdx.x * out_stride;
    for (int64_t i = tid; i < fill_n; i += kFillThreads) sel[k + i] = 0.0;
  } else {
    float* sel = static_cast<float*>(sel_all) + (int64_t)blockIdx.x * out_stride;
    for (int64_t i = tid; i < fill_n; i += kFillThreads) sel[k + i] = 0.0f;
  }
}

cudaError_t launch_fill_slice(int dtype, int64_t* order, void* sel_d2, int64_t batch,
                              int64_t out_stride, int64_t k, int64_t m1, cudaStream_t st) {
  if (m1 - k <= 0 || batch <= 0) return cudaSuccess;
  fill_slice_kernel<<<(unsigned)batch, kFillThreads, 0, st>>>(order, sel_d2, dtype == 1,
                                                              out_stride, k, m1);
  return cudaGetLastError();
}

}  // namespace ffps
