// FFPS_F32_F64 on the schedules without a float-coordinate variant (K1, K1s,
// K1b, K1m, K5): the float cloud is widened to double in a library scratch
// buffer first (exact), then the binary64 kernels run on it.
#include <cuda_runtime.h>

#include <cstdint>

#include "ffps_internal.h"

namespace ffps {

namespace {

// dst[b][i] = (double) src[b * stride3 + i], i < rows * 3; float4 loads where
// the row block is 16-B aligned
__global__ void upcast_kernel(const float* __restrict__ src, int64_t batch, int64_t stride3,
                              int64_t len, double* __restrict__ dst) {
  const int64_t total = batch * len;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / len, j = i - b * len;
    dst[i] = (double)__ldg(src + b * stride3 + j);
  }
}

}  // namespace

cudaError_t launch_upcast(const void* src, int64_t batch, int64_t cloud_stride, int64_t rows,
                          void* dst, int sms, cudaStream_t st) {
  if (batch <= 0 || rows <= 0) return cudaSuccess;
  const int64_t len = rows * 3, total = batch * len;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;  // grid-stride beyond 8 CTAs per SM
  if (blocks > cap) blocks = cap;
  upcast_kernel<<<(unsigned)blocks, 256, 0, st>>>(static_cast<const float*>(src), batch,
                                                  cloud_stride * 3, len,
                                                  static_cast<double*>(dst));
  return cudaGetLastError();
}

}  // namespace ffps
