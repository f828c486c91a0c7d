// Dependent-chain latencies on this GPU (cycles per op): REDUX, SHFL, VOTE+FLO,
// LDS, LDG (L2 hit), atomicAdd smem.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out, int* gbuf, int iters) {
  __shared__ int sm[1024];
  int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i + 1) & 1023;
  __syncthreads();
  int v = lane;
  long long t0, t1;
  // REDUX chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __reduce_max_sync(0xffffffffu, v + lane) - lane;
  t1 = clock64();
  if (threadIdx.x == 0) out[0] = (int)((t1 - t0) / iters);
  // SHFL chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (int)((t1 - t0) / iters);
  // VOTE + FLO chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __ffs(__ballot_sync(0xffffffffu, ((v + lane) & 7) == 0)) + v;
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (int)((t1 - t0) / iters);
  // LDS chain (pointer chase)
  int p = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) p = sm[p];
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (int)((t1 - t0) / iters);
  // LDG chain (L2-resident pointer chase, cache-global so L1 is bypassed)
  int q = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) q = __ldcg(gbuf + q);
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (int)((t1 - t0) / iters);
  // LDG L1 hit chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) q = __ldca(gbuf + (q & 1023));
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (int)((t1 - t0) / iters);
  // REDUX.MIN + SEL + VOTE chain (argmax-style step)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    int m = __reduce_max_sync(0xffffffffu, v);
    unsigned b = __ballot_sync(0xffffffffu, v == m);
    v = __shfl_sync(0xffffffffu, v + lane, __ffs(b) - 1) & 1023;
  }
  t1 = clock64();
  if (threadIdx.x == 0) out[6] = (int)((t1 - t0) / iters);
  // __syncthreads chain (all threads)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { __syncthreads(); v += sm[(v + i) & 1023]; }
  t1 = clock64();
  if (threadIdx.x == 0) out[7] = (int)((t1 - t0) / iters);
  out[8 + threadIdx.x % 8] += v + p + q;  // keep alive
}
int main() {
  int *out, *g;
  cudaMalloc(&out, 64 * sizeof(int));
  cudaMalloc(&g, (1 << 20) * sizeof(int));
  int h[1 << 12];
  for (int i = 0; i < 4096; ++i) h[i] = (i * 97 + 13) % 4096;
  cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
  cudaMemset(out, 0, 64 * sizeof(int));
  for (int nt : {32, 512}) {
    k<<<1, nt>>>(out, g, 2000);
    cudaDeviceSynchronize();
    int r[16];
    cudaMemcpy(r, out, sizeof r, cudaMemcpyDeviceToHost);
    printf("threads=%d REDUX %d SHFL %d VOTE+FFS %d LDS %d LDG(L2) %d LDG(L1) %d argmax-step %d BAR+LDS %d\n",
           nt, r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7]);
  }
  return 0;
}
