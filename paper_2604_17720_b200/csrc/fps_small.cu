// K1s — farthest-point sampling of small clouds (n <= 8192), one CTA per cloud.
//
// Same contract and bit-exact results as K1 / K1b / K1g (restates run_kernel,
// reference pkg/src/flashfps/fps_core.py:110-175).  The streaming cluster
// kernel (K1) splits even a 4K-point cloud over several CTAs and pays a DSMEM
// exchange per greedy step; for clouds that fit one CTA's registers the
// whole step stays on one SM:
//   thread t owns positions [t * Q, t * Q + Q) (registers: xyz, dist);
//   per step: the packed f32x2 distance update (sub2 / sq2 / add2 as in K1,
//   separately rounded, fps_core.py:74-83) with the running min (:93), a
//   thread-local argmax (strict > over ascending slots = lowest position),
//   a warp argmax (REDUX max, then REDUX min of the position), one record per
//   warp in shared memory (double-buffered by step parity), one barrier,
//   and every warp reduces the NW records itself (no broadcast barrier).
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"
#include "ffps_internal.h"

namespace ffps {

namespace {

constexpr uint32_t kNone = 0xffffffffu;

template <typename T>
struct SmallRec {
  typename Arith<T>::bits_t v;
  uint32_t pos;
};

// dist update of one slot pair (f32: packed FADD2 / FFMA2 with -0 addend)
template <typename T>
struct Upd;
template <>
struct Upd<float> {
  __device__ static void pair(float* x, float* y, float* z, float* d, int u, float px, float py,
                              float pz, float nz) {
    const float2 dx = sub2(make_float2(x[u], x[u + 1]), make_float2(px, px));
    const float2 dy = sub2(make_float2(y[u], y[u + 1]), make_float2(py, py));
    const float2 dz = sub2(make_float2(z[u], z[u + 1]), make_float2(pz, pz));
    const float2 z2 = make_float2(nz, nz);
    const float2 s = add2(add2(sq2(dx, z2), sq2(dy, z2)), sq2(dz, z2));
    d[u] = fminf(d[u], s.x);
    d[u + 1] = fminf(d[u + 1], s.y);
  }
};
template <>
struct Upd<double> {
  __device__ static void pair(double* x, double* y, double* z, double* d, int u, double px,
                              double py, double pz, float) {
#pragma unroll
    for (int w = 0; w < 2; ++w)
      d[u + w] = fmin(d[u + w], Arith<double>::d2(x[u + w], y[u + w], z[u + w], px, py, pz));
  }
};

}  // namespace

template <typename T, int NT, int Q>
__global__ void __launch_bounds__(NT, 1) fps_small_kernel(const GreedyParams prm) {
  using A = Arith<T>;
  using bits_t = typename A::bits_t;
  constexpr int NW = NT / 32;
  static_assert(Q % 2 == 0 && NW <= 32, "slot pairs, one record per lane");
  static_assert(NT <= 1024, "one CTA per cloud");
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (int)prm.n;
  const T* X0 = static_cast<const T*>(prm.xyz) + (int64_t)b * prm.cloud_stride * 3;
  const int64_t* map = prm.index_map ? prm.index_map + (int64_t)b * prm.map_stride : nullptr;
  int64_t* order = prm.order + (int64_t)b * prm.out_stride;
  T* sel = static_cast<T*>(prm.sel_d2) + (int64_t)b * prm.out_stride;
  __shared__ SmallRec<T> rec[2][NW];
  // a shared copy of the points: the step's winner is read from it by
  // position, so the argmax carries (value, position) only
  extern __shared__ __align__(16) unsigned char small_smem[];
  T* sx = reinterpret_cast<T*>(small_smem);
  T* sy = sx + NT * Q;
  T* sz = sy + NT * Q;

  // points (fps_core.py:119-122); slots past n hold -inf and never win
  T x[Q], y[Q], z[Q], d[Q];
#pragma unroll
  for (int u = 0; u < Q; ++u) {
    const int pos = tid * Q + u;
    const bool in = pos < n;
    const int64_t s = in ? (map ? map[pos] : pos) : 0;
    x[u] = in ? X0[3 * s + 0] : T(0);
    y[u] = in ? X0[3 * s + 1] : T(0);
    z[u] = in ? X0[3 * s + 2] : T(0);
    d[u] = in ? A::pinf() : A::ninf();
    sx[pos] = x[u];
    sy[pos] = y[u];
    sz[pos] = z[u];
  }
  // seed (fps_core.py:124-130)
  const int seed = (int)prm.seed_pos[b];
  const int64_t s0 = map ? map[seed] : seed;
  T px = X0[3 * s0 + 0], py = X0[3 * s0 + 1], pz = X0[3 * s0 + 2];
#pragma unroll
  for (int u = 0; u < Q; ++u)
    if (tid * Q + u == seed) d[u] = A::ninf();
  if (tid == 0) {
    order[0] = s0;
    sel[0] = A::pinf();
  }
  const float nz = prm.neg_zero;
  const int iters = (int)prm.iters;
  for (int it = 1; it < iters; ++it) {
    const int par = it & 1;
    // update (fps_core.py:86-95) and the thread's argmax
#pragma unroll
    for (int u = 0; u < Q; u += 2) Upd<T>::pair(x, y, z, d, u, px, py, pz, nz);
    bits_t bv = A::bits(d[0]);
#pragma unroll
    for (int u = 1; u < Q; ++u) bv = max(bv, A::bits(d[u]));
    int bu = Q - 1;  // the lowest slot (position) holding the maximum
#pragma unroll
    for (int u = Q - 2; u >= 0; --u) bu = A::bits(d[u]) == bv ? u : bu;
    const uint32_t bi = (uint32_t)(tid * Q + bu);
    // warp argmax: max value, lowest position at that value (:98-107)
    const bits_t wv = A::warp_max(bv);
    const uint32_t wi = __reduce_min_sync(0xffffffffu, bv == wv ? bi : kNone);
    if (bv == wv && bi == wi) rec[par][warp] = SmallRec<T>{wv, wi};
    __syncthreads();
    // every warp: argmax over the NW warp records
    const bits_t rv = lane < NW ? rec[par][lane].v : A::kmin;
    const uint32_t ri = lane < NW ? rec[par][lane].pos : kNone;
    const bits_t gv = A::warp_max(rv);
    const uint32_t gi = __reduce_min_sync(0xffffffffu, rv == gv ? ri : kNone);
    px = sx[gi];
    py = sy[gi];
    pz = sz[gi];
    // the winner leaves the candidate set (:169); its owner marks it
#pragma unroll
    for (int u = 0; u < Q; ++u)
      if ((uint32_t)(tid * Q + u) == gi) d[u] = A::ninf();
    if (tid == 0) {
      order[it] = map ? map[gi] : (int64_t)gi;  // fps_core.py:167-168, :197
      sel[it] = A::from_bits(gv);
    }
  }
}

template <typename T, int NT, int Q>
SmallInst make_sinst() {
  SmallInst k;
  k.smem = (size_t)NT * Q * 3 * sizeof(T);
  k.dtype = sizeof(T) == 4 ? 0 : 1;
  k.nt = NT;
  k.q = Q;
  k.fn = reinterpret_cast<const void*>(&fps_small_kernel<T, NT, Q>);
  return k;
}

const SmallInst* small_instances(int* count) {
  static const SmallInst insts[] = {
      // float: 256 threads up to 8192 points (tools/sweep_small.py: the step
      // time tracks nt * q, 256 threads edge out 512 / 1024 at equal capacity)
      make_sinst<float, 256, 2>(),   make_sinst<float, 256, 4>(),   make_sinst<float, 256, 8>(),
      make_sinst<float, 256, 16>(),  make_sinst<float, 256, 24>(),  make_sinst<float, 256, 32>(),
      make_sinst<double, 256, 2>(),  make_sinst<double, 256, 4>(),  make_sinst<double, 256, 8>(),
      make_sinst<double, 512, 8>(),  make_sinst<double, 512, 12>(), make_sinst<double, 512, 16>(),
  };
  *count = (int)(sizeof(insts) / sizeof(insts[0]));
  return insts;
}

}  // namespace ffps
