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
//   registers  lane l of warp w owns buckets q = j*NT + l*NW + w (j < NBT):
//              box as (lo, -hi) pairs, the bucket key (max distance bits,
//              lowest position at that distance) and the xyz of that point
//   smem       per-warp argmax records, double-buffered by iteration parity
//   global/L2  X, Y, Z, D, O (bucket-major SoA, D = running min distance)
// Per iteration: packed bound test of the owned buckets -> ballot -> the warp
// re-evaluates its own flagged buckets (32 lanes = 32 points, one L2 round
// trip) -> owner lane refreshes the key -> warp argmax -> ONE __syncthreads
// -> every warp reduces the NW records to the next point.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "arith.cuh"
#include "ffps_internal.h"

namespace ffps {

template <typename T, int NT, int PPL, int NBT>
__global__ void __launch_bounds__(NT, 1) fps_bucket_kernel(const BucketParams prm) {
  using A = Arith<T>;
  using bits_t = typename A::bits_t;
  using pair_t = typename A::pair_t;
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

  // warp records, double-buffered by iteration parity: one barrier per iteration
  __shared__ bits_t rv_s[2][NW];
  __shared__ uint32_t ri_s[2][NW];
  __shared__ int32_t rq_s[2][NW];
  __shared__ T rx_s[2][NW][3];

  // Owned buckets: q = j*NT + lane*NW + warp, so Morton-consecutive buckets
  // (the ones a new point tends to hit together) belong to different warps.
  // Box as per-axis pairs (lo, -hi); key (max distance bits, lowest position
  // at that distance) and the xyz of that point, all in registers.
  pair_t lnh[NBT][3];
  bits_t ov[NBT];
  uint32_t oi[NBT];
  T ox[NBT], oy[NBT], oz[NBT];
#pragma unroll
  for (int j = 0; j < NBT; ++j) {
    const int q = j * NT + lane * NW + warp;
    if (q < nb) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
        lnh[j][c] = A::mk(BB[(int64_t)q * 6 + c], -BB[(int64_t)q * 6 + 3 + c]);
      ov[j] = A::bits(A::pinf());
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) lnh[j][c] = A::mk(T(0), T(0));
      ov[j] = A::bits(A::ninf());  // never flagged, never wins
    }
    oi[j] = kNoIdx;
    ox[j] = oy[j] = oz[j] = T(0);
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
  }
  uint32_t win = (uint32_t)seed;  // position to set to -inf on its next visit
  int prevq = -1;                 // its bucket (re-evaluated unconditionally)
  const pair_t nz = A::mk((T)prm.neg_zero, (T)prm.neg_zero);

  const int iters = (int)prm.iters;
  // optional phase trace (tools/trace_bucket.py): CTA 0, lane 0 of every warp,
  // per iteration {start, bound test, re-evaluation, argmax, barrier, end, flags}
  long long* trace =
      (prm.trace && b == 0 && lane == 0) ? prm.trace + (int64_t)warp * prm.trace_iters * 8 : nullptr;
  // this warp's record (uniform across its lanes): best key over its buckets.
  // Keys only decrease, so it stays valid unless its own bucket is re-evaluated.
  bits_t rv = A::kmin;
  uint32_t ri = kNoIdx;
  int rq = -1;
  T rx = T(0), ry = T(0), rz = T(0);
  for (int k = 1; k < iters; ++k) {
    const uint32_t par = (uint32_t)k & 1u;
    long long t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    int nflag_w = 0;
    if (trace) t0 = clock64();
    bool stale = k == 1;
    const pair_t ppx = A::mk(-px, px), ppy = A::mk(-py, py), ppz = A::mk(-pz, pz);
    // 1. bound test of the owned buckets ------------------------------------------
    unsigned fm[NBT];
#pragma unroll
    for (int j = 0; j < NBT; ++j) {
      const int q = j * NT + lane * NW + warp;
      const T lb = A::box_d2_pairs(lnh[j], ppx, ppy, ppz, nz);
      const bool f = !(lb >= A::from_bits(ov[j])) || q == prevq || (k == 1 && q < nb);
      fm[j] = __ballot_sync(0xffffffffu, f);
      nflag_w += __popc(fm[j]);
    }
    if (trace) t1 = clock64();
    // 2. the warp re-evaluates its own flagged buckets, lanes = points ------------
#pragma unroll
    for (int j = 0; j < NBT; ++j) {
      unsigned m = fm[j];
      while (m) {
        const int ol = __ffs(m) - 1;  // owner lane
        m &= m - 1;
        const int q = j * NT + ol * NW + warp;
        bits_t bv = A::kmin;
        uint32_t bi = kNoIdx;
        T bx = T(0), by = T(0), bz = T(0);
        T xs[PPL], ys[PPL], zs[PPL], ds[PPL];
        uint32_t os[PPL];
#pragma unroll
        for (int u = 0; u < PPL; ++u) {  // all loads first (one L2 round trip)
          const int64_t s = (int64_t)q * BS + u * 32 + lane;
          xs[u] = X[s];
          ys[u] = Y[s];
          zs[u] = Z[s];
          ds[u] = D[s];
          os[u] = (uint32_t)O[s];
        }
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          T nd = A::vmin(ds[u], A::d2(xs[u], ys[u], zs[u], px, py, pz));  // fps_core.py:93
          if (os[u] == win) nd = A::ninf();                               // fps_core.py:169
          if (A::bits(nd) != A::bits(ds[u])) D[(int64_t)q * BS + u * 32 + lane] = nd;
          const bits_t v = A::bits(nd);
          if (v > bv || (v == bv && os[u] < bi)) {
            bv = v;
            bi = os[u];
            bx = xs[u];
            by = ys[u];
            bz = zs[u];
          }
        }
        const bits_t wv = A::warp_max(bv);
        const uint32_t wi = __reduce_min_sync(0xffffffffu, bv == wv ? bi : kNoIdx);
        const int wl = __ffs(__ballot_sync(0xffffffffu, bv == wv && bi == wi)) - 1;
        bx = __shfl_sync(0xffffffffu, bx, wl);
        by = __shfl_sync(0xffffffffu, by, wl);
        bz = __shfl_sync(0xffffffffu, bz, wl);
        if (lane == ol) {
          ov[j] = wv;
          oi[j] = wi;
          ox[j] = bx;
          oy[j] = by;
          oz[j] = bz;
        }
        stale |= (q == rq);
      }
    }
    if (trace) t2 = clock64();
    // 3. thread / warp argmax over owned keys (max value, lowest position), only
    //    when the warp's record went stale --------------------------------------------
    if (stale) {
      bits_t tv = A::kmin;
      uint32_t ti = kNoIdx;
      int tj = 0;
#pragma unroll
      for (int j = 0; j < NBT; ++j)
        if (ov[j] > tv || (ov[j] == tv && oi[j] < ti)) {
          tv = ov[j];
          ti = oi[j];
          tj = j;
        }
      const bits_t wv = A::warp_max(tv);
      const uint32_t wi = __reduce_min_sync(0xffffffffu, tv == wv ? ti : kNoIdx);
      const int wl = __ffs(__ballot_sync(0xffffffffu, tv == wv && ti == wi)) - 1;
      T cx = ox[0], cy = oy[0], cz = oz[0];
#pragma unroll
      for (int j = 1; j < NBT; ++j)
        if (tj == j) {
          cx = ox[j];
          cy = oy[j];
          cz = oz[j];
        }
      rv = wv;
      ri = wi;
      rq = __shfl_sync(0xffffffffu, tj * NT + lane * NW + warp, wl);
      rx = __shfl_sync(0xffffffffu, cx, wl);
      ry = __shfl_sync(0xffffffffu, cy, wl);
      rz = __shfl_sync(0xffffffffu, cz, wl);
    }
    if (lane == 0) {
      rv_s[par][warp] = rv;
      ri_s[par][warp] = ri;
      rq_s[par][warp] = rq;
      rx_s[par][warp][0] = rx;
      rx_s[par][warp][1] = ry;
      rx_s[par][warp][2] = rz;
    }
    if (trace) t3 = clock64();
    __syncthreads();  // the only barrier of the iteration
    if (trace) t4 = clock64();

    // 4. every warp reduces the NW records -> the next point ------------------------
    const bits_t rv = lane < NW ? rv_s[par][lane] : A::kmin;
    const uint32_t ri = lane < NW ? ri_s[par][lane] : kNoIdx;
    const bits_t gv = A::warp_max(rv);
    const uint32_t gi = __reduce_min_sync(0xffffffffu, rv == gv ? ri : kNoIdx);
    const int gl = __ffs(__ballot_sync(0xffffffffu, rv == gv && ri == gi)) - 1;
    px = rx_s[par][gl][0];
    py = rx_s[par][gl][1];
    pz = rx_s[par][gl][2];
    prevq = rq_s[par][gl];
    win = gi;
    if (tid == 0) {  // fps_core.py:167-168
      order[k] = gi;
      sel[k] = A::from_bits(gv);
    }
    if (trace && k < prm.trace_iters) {
      long long* r = trace + (int64_t)k * 8;
      r[0] = t0; r[1] = t1; r[2] = t2; r[3] = t3; r[4] = t4; r[5] = clock64(); r[6] = nflag_w;
    }
  }

  // positions -> original indices for restricted runs (fps_cache.py:197)
  if (prm.index_map != nullptr) {
    __syncthreads();
    const int64_t* map = prm.index_map + (int64_t)b * prm.map_stride;
    for (int k = tid; k < iters; k += NT) order[k] = __ldg(map + order[k]);
  }
}


template <typename T, int PPL, int NBT, int NT = kBucketThreads>
BucketInst make_binst() {
  BucketInst k;
  k.dtype = sizeof(T) == 4 ? 0 : 1;
  k.nt = NT;
  k.ppl = PPL;
  k.nbt = NBT;
  k.fn = reinterpret_cast<const void*>(&fps_bucket_kernel<T, NT, PPL, NBT>);
  k.smem_per_bucket = 0;  // bucket state lives in registers
  return k;
}

const BucketInst* bucket_instances(int* count) {
  static const BucketInst insts[] = {
      make_binst<float, 1, 1>(),  make_binst<float, 1, 2>(),  make_binst<float, 1, 4>(),
      make_binst<float, 1, 8>(),  make_binst<float, 2, 4>(),  make_binst<float, 2, 8>(),
      make_binst<float, 4, 8>(),
      // 256-thread variants: half the per-warp fixed overhead, twice the boxes per lane
      make_binst<float, 1, 8, 256>(), make_binst<float, 1, 16, 256>(),
      make_binst<float, 2, 16, 256>(),
      make_binst<double, 1, 1>(), make_binst<double, 1, 2>(),
      make_binst<double, 1, 4>(), make_binst<double, 1, 8>(), make_binst<double, 2, 8>(),
      make_binst<double, 4, 8>(),
  };
  *count = (int)(sizeof(insts) / sizeof(insts[0]));
  return insts;
}

}  // namespace ffps
