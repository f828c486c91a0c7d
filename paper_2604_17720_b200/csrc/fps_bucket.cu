// K1b — bucketed persistent farthest-point sampling (one CTA per cloud).
//
// Same contract as K1 (restates run_kernel, reference
// pkg/src/flashfps/fps_core.py:110-175, bit for bit), different schedule:
// the points of a cloud sit in spatial buckets of BS = 32*PPL points (built
// by K0, bucket_build.cu) in L2-resident bucket-major SoA, and each greedy
// iteration only re-evaluates the buckets the new point can affect.
//
// Exactness.  A bucket is skipped when box_d2(p, bucket box) >= its current
// max distance.  box_d2 uses the reference's own rounded operations, which
// are monotone, so every member's computed d2(x, p) >= box_d2 >= dist(x):
// min(dist, d2) would return dist unchanged (fps_core.py:93).  Ties are broken
// by the point's position in the run's point list (never by slot), i.e. the
// reference's lowest-index rule (np.argmax first occurrence, fps_core.py:94,
// :98-107).  The selected point is set to -inf (fps_core.py:169) the next
// time its bucket is visited: the winner's bucket is always re-evaluated.
//
// State per cloud:
//   registers  thread t owns buckets q = t + j*NT (j < NBT): box lo/hi and a
//              cached copy of the bucket key (max distance bits, position)
//   smem       per bucket: key value, key position, xyz of the key point;
//              the list of buckets flagged this iteration; per-warp argmax
//   global/L2  X, Y, Z, D, O (bucket-major SoA, D = running min distance)
// Per iteration: flag (bound test of owned buckets) | sync | flagged buckets
// re-evaluated, one warp per bucket | sync | owners refresh their keys, warp
// argmax | sync | every warp reduces the NW warp records -> next point.
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"
#include "ffps_internal.h"

namespace ffps {

template <typename T, int NT, int PPL, int NBT>
__global__ void __launch_bounds__(NT, 1) fps_bucket_kernel(const BucketParams prm) {
  using A = Arith<T>;
  using bits_t = typename A::bits_t;
  constexpr int NW = NT / 32;
  constexpr int BS = 32 * PPL;
  constexpr uint32_t kNoIdx = 0xffffffffu;

  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = (int)prm.nbuckets;
  const int64_t off = (int64_t)b * prm.nslots;
  const T* __restrict__ X = static_cast<const T*>(prm.X) + off;
  const T* __restrict__ Y = static_cast<const T*>(prm.Y) + off;
  const T* __restrict__ Z = static_cast<const T*>(prm.Z) + off;
  T* __restrict__ D = static_cast<T*>(prm.D) + off;
  const int32_t* __restrict__ O = prm.O + off;
  const T* __restrict__ BB = static_cast<const T*>(prm.BB) + (int64_t)b * nb * 6;

  extern __shared__ __align__(16) unsigned char smem[];
  bits_t* kv = reinterpret_cast<bits_t*>(smem);                      // [nb]
  T* best = reinterpret_cast<T*>(smem + (size_t)nb * sizeof(bits_t)); // [nb][3]
  uint32_t* ki = reinterpret_cast<uint32_t*>(best + (size_t)nb * 3);  // [nb]
  int32_t* list = reinterpret_cast<int32_t*>(ki + nb);                // [nb]
  __shared__ bits_t wv_s[NW];
  __shared__ uint32_t wi_s[NW];
  __shared__ int32_t wq_s[NW];
  __shared__ int cnt;

  // owned buckets: boxes in registers, keys cached (+inf => visited first)
  T lo[NBT][3], hi[NBT][3];
  bits_t ov[NBT];
  uint32_t oi[NBT];
#pragma unroll
  for (int j = 0; j < NBT; ++j) {
    const int q = tid + j * NT;
    if (q < nb) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        lo[j][c] = BB[(int64_t)q * 6 + c];
        hi[j][c] = BB[(int64_t)q * 6 + 3 + c];
      }
      ov[j] = A::bits(A::pinf());
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) lo[j][c] = hi[j][c] = T(0);
      ov[j] = A::kmin;
    }
    oi[j] = kNoIdx;
  }

  // seed (fps_core.py:124-130): order[0] = seed, sel[0] = +inf
  const int seed = (int)prm.seed_pos[b];
  T px, py, pz;
  {
    const T* X0 = static_cast<const T*>(prm.xyz) + (int64_t)b * prm.cloud_stride * 3;
    const int64_t src = prm.index_map ? prm.index_map[(int64_t)b * prm.map_stride + seed] : seed;
    px = X0[3 * src + 0];
    py = X0[3 * src + 1];
    pz = X0[3 * src + 2];
  }
  int64_t* order = prm.order + (int64_t)b * prm.out_stride;
  T* sel = static_cast<T*>(prm.sel_d2) + (int64_t)b * prm.out_stride;
  if (tid == 0) {
    order[0] = seed;
    sel[0] = A::pinf();
    cnt = 0;
  }
  uint32_t win = (uint32_t)seed;  // position to set to -inf on its next visit
  int prevq = -1;                 // bucket holding it (re-evaluated unconditionally)
  __syncthreads();

  const int iters = (int)prm.iters;
  for (int k = 1; k < iters; ++k) {
    // 1. flag owned buckets the new point can affect ------------------------------
    uint32_t fl = 0;
#pragma unroll
    for (int j = 0; j < NBT; ++j) {
      const int q = tid + j * NT;
      bool f = false;
      if (q < nb)
        f = k == 1 || q == prevq || !(A::box_d2(px, py, pz, lo[j], hi[j]) >= A::from_bits(ov[j]));
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (m) {
        const int leader = __ffs(m) - 1;
        int pos = 0;
        if (lane == leader) pos = atomicAdd(&cnt, __popc(m));
        pos = __shfl_sync(0xffffffffu, pos, leader);
        if (f) list[pos + __popc(m & ((1u << lane) - 1u))] = q;
      }
      fl |= (uint32_t)f << j;
    }
    __syncthreads();  // A: list complete
    const int nflag = cnt;

    // 2. re-evaluate flagged buckets, one warp per bucket ---------------------------
    for (int e = warp; e < nflag; e += NW) {
      const int q = list[e];
      bits_t bv = A::kmin;
      uint32_t bi = kNoIdx;
      T bx = T(0), by = T(0), bz = T(0);
#pragma unroll
      for (int u = 0; u < PPL; ++u) {
        const int64_t s = (int64_t)q * BS + u * 32 + lane;
        const T x = X[s], y = Y[s], z = Z[s], d = D[s];
        const uint32_t o = (uint32_t)O[s];
        T nd = A::vmin(d, A::d2(x, y, z, px, py, pz));  // fps_core.py:93
        if (o == win) nd = A::ninf();                    // fps_core.py:169
        if (A::bits(nd) != A::bits(d)) D[s] = nd;
        const bits_t v = A::bits(nd);
        if (v > bv || (v == bv && o < bi)) {
          bv = v;
          bi = o;
          bx = x;
          by = y;
          bz = z;
        }
      }
      const bits_t wv = A::warp_max(bv);
      const uint32_t wi = __reduce_min_sync(0xffffffffu, bv == wv ? bi : kNoIdx);
      const int wl = __ffs(__ballot_sync(0xffffffffu, bv == wv && bi == wi)) - 1;
      if (lane == wl) {
        kv[q] = wv;
        ki[q] = wi;
        best[3 * q + 0] = bx;
        best[3 * q + 1] = by;
        best[3 * q + 2] = bz;
      }
    }
    __syncthreads();  // B: keys of re-evaluated buckets visible
    if (tid == 0) cnt = 0;

    // 3. owners refresh keys, thread / warp argmax (max value, lowest position) ---
    bits_t tv = A::kmin;
    uint32_t ti = kNoIdx;
    int tq = -1;
#pragma unroll
    for (int j = 0; j < NBT; ++j) {
      const int q = tid + j * NT;
      if ((fl >> j) & 1u) {
        ov[j] = kv[q];
        oi[j] = ki[q];
      }
      if (q < nb && (ov[j] > tv || (ov[j] == tv && oi[j] < ti))) {
        tv = ov[j];
        ti = oi[j];
        tq = q;
      }
    }
    {
      const bits_t wv = A::warp_max(tv);
      const uint32_t wi = __reduce_min_sync(0xffffffffu, tv == wv ? ti : kNoIdx);
      const int wl = __ffs(__ballot_sync(0xffffffffu, tv == wv && ti == wi)) - 1;
      if (lane == wl) {
        wv_s[warp] = wv;
        wi_s[warp] = wi;
        wq_s[warp] = tq;
      }
    }
    __syncthreads();  // C: warp records visible

    // 4. every warp reduces the NW records -> the next point ------------------------
    const bits_t rv = lane < NW ? wv_s[lane] : A::kmin;
    const uint32_t ri = lane < NW ? wi_s[lane] : kNoIdx;
    const int rq = lane < NW ? wq_s[lane] : -1;
    const bits_t gv = A::warp_max(rv);
    const uint32_t gi = __reduce_min_sync(0xffffffffu, rv == gv ? ri : kNoIdx);
    const int gl = __ffs(__ballot_sync(0xffffffffu, rv == gv && ri == gi)) - 1;
    const int gq = __shfl_sync(0xffffffffu, rq, gl);
    px = best[3 * gq + 0];
    py = best[3 * gq + 1];
    pz = best[3 * gq + 2];
    win = gi;
    prevq = gq;
    if (tid == 0) {  // fps_core.py:167-168
      order[k] = gi;
      sel[k] = A::from_bits(gv);
    }
  }

  // positions -> original indices for restricted runs (fps_cache.py:197)
  if (prm.index_map != nullptr) {
    __syncthreads();
    const int64_t* map = prm.index_map + (int64_t)b * prm.map_stride;
    for (int k = tid; k < iters; k += NT) order[k] = __ldg(map + order[k]);
  }
}

template <typename T, int PPL, int NBT>
BucketInst make_binst() {
  BucketInst k;
  k.dtype = sizeof(T) == 4 ? 0 : 1;
  k.nt = kBucketThreads;
  k.ppl = PPL;
  k.nbt = NBT;
  k.fn = reinterpret_cast<const void*>(&fps_bucket_kernel<T, kBucketThreads, PPL, NBT>);
  k.smem_per_bucket = sizeof(typename Arith<T>::bits_t) + 3 * sizeof(T) + 4 + 4;
  return k;
}

const BucketInst* bucket_instances(int* count) {
  static const BucketInst insts[] = {
      make_binst<float, 1, 1>(),  make_binst<float, 1, 2>(),  make_binst<float, 1, 4>(),
      make_binst<float, 1, 8>(),  make_binst<float, 2, 4>(),  make_binst<float, 2, 8>(),
      make_binst<float, 4, 8>(),  make_binst<double, 1, 1>(), make_binst<double, 1, 2>(),
      make_binst<double, 1, 4>(), make_binst<double, 1, 8>(), make_binst<double, 2, 8>(),
      make_binst<double, 4, 8>(),
  };
  *count = (int)(sizeof(insts) / sizeof(insts[0]));
  return insts;
}

}  // namespace ffps
