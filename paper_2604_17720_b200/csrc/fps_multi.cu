// K1m — bucketed farthest-point sampling with multi-winner rounds.
//
// Same contract and bit-exact results as K1 / K1b (restates run_kernel,
// reference pkg/src/flashfps/fps_core.py:110-175), fewer synchronisations:
// every round selects up to KM consecutive greedy winners at once.
//
// Why several winners can be taken from one reduction.  Let c_1, c_2, ... be
// the bucket keys in argmax order (max distance desc, lowest position asc;
// one key per bucket = its best point).  c_1 is the next greedy winner.  The
// candidate c_j is the winner right after c_1..c_{j-1} if
//   (a) its distance is untouched by them: d2(c_j, c_i) >= dist(c_j) for all
//       i < j (the reference's own rounded d2), so min(dist, d2) keeps it;
//   (b) it beats every point left in the chosen buckets: dist(c_j) > v2(B_i),
//       the second-best distance of bucket B_i, for all i < j;
// since every other distance only decreases and every other bucket's key
// ranks below c_j.  The round accepts the longest such prefix c_1..c_J
// (J >= 1) and reports them with their unchanged distances — exactly the
// (order, selection_dist2) entries the reference produces one by one.
// Measured on uniform 50K-point clouds: 7.5 winners per round for KM = 8,
// 13 for KM = 16 (11.7 on LiDAR-like frames).
//
// A round:
//   1. bound test of every owned bucket against the J points of the previous
//      round (box_d2 with the reference's rounded ops, as in K1b) -> ballot;
//   2. the warp re-evaluates its flagged buckets against all J points (one L2
//      round trip per bucket): new key (value, position, xyz) and second
//      best v2 into the owner lane's registers; the points themselves -> -inf;
//   3. per-warp top-KM of the owned keys (KM warp argmax steps) -> smem;
//   | barrier |
//   4. warp 0 merges the NW x KM records to the global top-KM, tests (a) and
//      (b) for all candidate pairs at once, writes the accepted prefix;
//   | barrier |
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"
#include "ffps_internal.h"

namespace ffps {

// lane of the warp argmax of (v desc, i asc)
template <typename A>
__device__ __forceinline__ int argmax_lane(typename A::bits_t v, uint32_t i) {
  const typename A::bits_t wv = A::warp_max(v);
  const uint32_t wi = __reduce_min_sync(0xffffffffu, v == wv ? i : 0xffffffffu);
  return __ffs(__ballot_sync(0xffffffffu, v == wv && i == wi)) - 1;
}

template <typename T, int NT, int PPL, int NBT, int KM>
__global__ void __launch_bounds__(NT, 1) fps_multi_kernel(const BucketParams prm) {
  using A = Arith<T>;
  using bits_t = typename A::bits_t;
  using pair_t = typename A::pair_t;
  constexpr int NW = NT / 32;
  constexpr int BS = 32 * PPL;
  constexpr uint32_t kNoIdx = 0xffffffffu;
  constexpr int NREC = NW * KM;          // records merged by warp 0
  constexpr int RPL = (NREC + 31) / 32;  // records per lane in the merge
  static_assert(KM <= 32, "one candidate per lane in the chain test");

  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = (int)prm.nbuckets;
  const int64_t off = (int64_t)b * prm.nslots;
  const T* __restrict__ X = static_cast<const T*>(prm.X) + off;
  const T* __restrict__ Y = static_cast<const T*>(prm.Y) + off;
  const T* __restrict__ Z = static_cast<const T*>(prm.Z) + off;
  T* __restrict__ D = static_cast<T*>(prm.D) + off;
  const int32_t* __restrict__ O = prm.O + off;
  const T* __restrict__ BB = static_cast<const T*>(prm.BB) + (int64_t)b * nb * 6;

  // per-warp top-KM records and the accepted points of the round
  __shared__ bits_t rv_s[NREC], r2_s[NREC];
  __shared__ uint32_t ri_s[NREC];
  __shared__ int32_t rq_s[NREC];
  __shared__ T rx_s[NREC][3];
  __shared__ T sp_s[KM][3];
  __shared__ uint32_t si_s[KM];
  __shared__ int32_t sq_s[KM];
  __shared__ int nsel_s;

  pair_t lnh[NBT][3];
  bits_t ov[NBT], o2[NBT];
  uint32_t oi[NBT];
  T ox[NBT], oy[NBT], oz[NBT];
#pragma unroll
  for (int j = 0; j < NBT; ++j) {
    const int q = j * NT + lane * NW + warp;
    if (q < nb) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
        lnh[j][c] = A::mk(BB[(int64_t)q * 6 + c], -BB[(int64_t)q * 6 + 3 + c]);
      ov[j] = o2[j] = A::bits(A::pinf());
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) lnh[j][c] = A::mk(T(0), T(0));
      ov[j] = o2[j] = A::kmin;  // never flagged, never a candidate
    }
    oi[j] = kNoIdx;
    ox[j] = oy[j] = oz[j] = T(0);
  }

  // seed (fps_core.py:124-130)
  const int seed = (int)prm.seed_pos[b];
  int64_t* order = prm.order + (int64_t)b * prm.out_stride;
  T* sel = static_cast<T*>(prm.sel_d2) + (int64_t)b * prm.out_stride;
  if (tid == 0) {
    const T* X0 = static_cast<const T*>(prm.xyz) + (int64_t)b * prm.cloud_stride * 3;
    const int64_t src = prm.index_map ? prm.index_map[(int64_t)b * prm.map_stride + seed] : seed;
    sp_s[0][0] = X0[3 * src + 0];
    sp_s[0][1] = X0[3 * src + 1];
    sp_s[0][2] = X0[3 * src + 2];
    si_s[0] = (uint32_t)seed;
    sq_s[0] = -1;
    nsel_s = 1;
    order[0] = seed;
    sel[0] = A::pinf();
  }
  __syncthreads();
  const pair_t nz = A::mk((T)prm.neg_zero, (T)prm.neg_zero);
  const int iters = (int)prm.iters;
  long long* trace =
      (prm.trace && b == 0 && lane == 0) ? prm.trace + (int64_t)warp * prm.trace_iters * 8 : nullptr;

  int k = 1;  // winners reported so far
  for (int round = 0; k < iters; ++round) {
    const int J = nsel_s;
    long long t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    if (trace) t0 = clock64();
    // 1. bound test against the J points of the last round ----------------------
    unsigned fm[NBT];
#pragma unroll
    for (int j = 0; j < NBT; ++j) fm[j] = 0u;
    for (int t = 0; t < J; ++t) {
      const T px = sp_s[t][0], py = sp_s[t][1], pz = sp_s[t][2];
      const int sq = sq_s[t];
      const pair_t ppx = A::mk(-px, px), ppy = A::mk(-py, py), ppz = A::mk(-pz, pz);
#pragma unroll
      for (int j = 0; j < NBT; ++j) {
        const int q = j * NT + lane * NW + warp;
        const T lb = A::box_d2_pairs(lnh[j], ppx, ppy, ppz, nz);
        const bool f = q < nb && (round == 0 || q == sq || !(lb >= A::from_bits(ov[j])));
        fm[j] |= __ballot_sync(0xffffffffu, f);
      }
    }
    if (trace) t1 = clock64();
    // 2. re-evaluate the flagged buckets against all J points ----------------------
#pragma unroll
    for (int j = 0; j < NBT; ++j) {
      unsigned m = fm[j];
      while (m) {
        const int ol = __ffs(m) - 1;
        m &= m - 1u;
        const int q = j * NT + ol * NW + warp;
        T xs[PPL], ys[PPL], zs[PPL], ds[PPL], d0[PPL];
        uint32_t os[PPL];
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          const int64_t s = (int64_t)q * BS + u * 32 + lane;
          xs[u] = X[s];
          ys[u] = Y[s];
          zs[u] = Z[s];
          ds[u] = D[s];
          os[u] = (uint32_t)O[s];
          d0[u] = ds[u];
        }
        for (int t = 0; t < J; ++t) {
          const T px = sp_s[t][0], py = sp_s[t][1], pz = sp_s[t][2];
          const uint32_t pw = si_s[t];
#pragma unroll
          for (int u = 0; u < PPL; ++u) {
            T nd = A::vmin(ds[u], A::d2(xs[u], ys[u], zs[u], px, py, pz));  // :93
            if (os[u] == pw) nd = A::ninf();                                // :169
            ds[u] = nd;
          }
        }
        bits_t b1 = A::kmin, b2 = A::kmin;
        uint32_t i1 = kNoIdx;
        T x1 = T(0), y1 = T(0), z1 = T(0);
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          if (A::bits(ds[u]) != A::bits(d0[u])) D[(int64_t)q * BS + u * 32 + lane] = ds[u];
          const bits_t v = A::bits(ds[u]);
          if (v > b1 || (v == b1 && os[u] < i1)) {
            b2 = b1;
            b1 = v;
            i1 = os[u];
            x1 = xs[u];
            y1 = ys[u];
            z1 = zs[u];
          } else if (v > b2) {
            b2 = v;
          }
        }
        const int wl = argmax_lane<A>(b1, i1);
        const bits_t wv = A::shfl(b1, wl);
        const uint32_t wi = __shfl_sync(0xffffffffu, i1, wl);
        const bits_t w2 = A::warp_max(lane == wl ? b2 : b1);
        x1 = __shfl_sync(0xffffffffu, x1, wl);
        y1 = __shfl_sync(0xffffffffu, y1, wl);
        z1 = __shfl_sync(0xffffffffu, z1, wl);
        if (lane == ol) {
          ov[j] = wv;
          oi[j] = wi;
          o2[j] = w2;
          ox[j] = x1;
          oy[j] = y1;
          oz[j] = z1;
        }
      }
    }
    if (trace) t2 = clock64();
    // 3. per-warp top-KM of the owned keys ------------------------------------------
    {
      unsigned taken = 0;
#pragma unroll 1
      for (int r = 0; r < KM; ++r) {
        bits_t bv = A::kmin;
        uint32_t bi = kNoIdx;
        int bj = 0;
#pragma unroll
        for (int j = 0; j < NBT; ++j)
          if (!((taken >> j) & 1u) && (ov[j] > bv || (ov[j] == bv && oi[j] < bi))) {
            bv = ov[j];
            bi = oi[j];
            bj = j;
          }
        const int wl = argmax_lane<A>(bv, bi);
        if (lane == wl) {
          taken |= 1u << bj;
          const int e = warp * KM + r;
          rv_s[e] = bv;
          ri_s[e] = bi;
          T cx = ox[0], cy = oy[0], cz = oz[0];
          bits_t c2 = o2[0];
#pragma unroll
          for (int j = 1; j < NBT; ++j)
            if (bj == j) {
              cx = ox[j];
              cy = oy[j];
              cz = oz[j];
              c2 = o2[j];
            }
          r2_s[e] = c2;
          rq_s[e] = bj * NT + lane * NW + warp;
          rx_s[e][0] = cx;
          rx_s[e][1] = cy;
          rx_s[e][2] = cz;
        }
      }
    }
    if (trace) t3 = clock64();
    __syncthreads();  // B1: records visible
    // 4. warp 0: global top-KM, chain test, accepted prefix ------------------------
    if (warp == 0) {
      bits_t lv[RPL];
      uint32_t li[RPL];
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int e = lane + 32 * t;
        lv[t] = e < NREC ? rv_s[e] : A::kmin;
        li[t] = e < NREC ? ri_s[e] : kNoIdx;
      }
      unsigned taken = 0;
      int cand = -1;  // lane r holds the record of candidate r
#pragma unroll 1
      for (int r = 0; r < KM; ++r) {
        bits_t bv = A::kmin;
        uint32_t bi = kNoIdx;
        int bt = 0;
#pragma unroll
        for (int t = 0; t < RPL; ++t)
          if (!((taken >> t) & 1u) && (lv[t] > bv || (lv[t] == bv && li[t] < bi))) {
            bv = lv[t];
            bi = li[t];
            bt = t;
          }
        const int wl = argmax_lane<A>(bv, bi);
        if (lane == wl) taken |= 1u << bt;
        const int e = __shfl_sync(0xffffffffu, lane + 32 * bt, wl);
        if (lane == r) cand = e;
      }
      // candidate r on lane r: value, second best of its bucket, coordinates
      const bool live = lane < KM;
      const bits_t cv = live ? rv_s[cand] : A::kmin;
      const bits_t c2 = live ? r2_s[cand] : A::kmin;
      const T cx = live ? rx_s[cand][0] : T(0);
      const T cy = live ? rx_s[cand][1] : T(0);
      const T cz = live ? rx_s[cand][2] : T(0);
      // lane a: does candidate a survive every earlier candidate b < a?
      bool ok = live && cv != A::kmin && A::from_bits(cv) >= T(0);
      for (int bb = 0; bb < KM - 1; ++bb) {
        const T bx = __shfl_sync(0xffffffffu, cx, bb);
        const T by = __shfl_sync(0xffffffffu, cy, bb);
        const T bz = __shfl_sync(0xffffffffu, cz, bb);
        const bits_t b2 = A::shfl(c2, bb);
        if (bb < lane && ok) {
          ok = !(A::d2(cx, cy, cz, bx, by, bz) < A::from_bits(cv)) &&  // (a)
               cv > b2;                                                 // (b)
        }
      }
      const unsigned okm = __ballot_sync(0xffffffffu, ok || lane == 0);
      int acc = __ffs(~okm) - 1;  // longest prefix of accepted candidates
      if (acc < 0 || acc > KM) acc = KM;
      if (acc > iters - k) acc = iters - k;
      if (lane < acc) {
        sp_s[lane][0] = cx;
        sp_s[lane][1] = cy;
        sp_s[lane][2] = cz;
        si_s[lane] = ri_s[cand];
        sq_s[lane] = rq_s[cand];
        order[k + lane] = ri_s[cand];  // fps_core.py:167-168
        sel[k + lane] = A::from_bits(cv);
      }
      if (lane == 0) nsel_s = acc;
    }
    __syncthreads();  // B2: accepted points visible
    if (trace) t4 = clock64();
    if (trace && round < prm.trace_iters) {
      long long* rr = trace + (int64_t)round * 8;
      rr[0] = t0; rr[1] = t1; rr[2] = t2; rr[3] = t3; rr[4] = t4; rr[5] = nsel_s;
      int nf = 0;
#pragma unroll
      for (int j = 0; j < NBT; ++j) nf += __popc(fm[j]);
      rr[6] = nf;
    }
    k += nsel_s;
  }

  // positions -> original indices for restricted runs (fps_cache.py:197)
  if (prm.index_map != nullptr) {
    __syncthreads();
    const int64_t* map = prm.index_map + (int64_t)b * prm.map_stride;
    for (int kk = tid; kk < iters; kk += NT) order[kk] = __ldg(map + order[kk]);
  }
}

template <typename T, int PPL, int NBT, int KM>
BucketInst make_minst() {
  BucketInst k;
  k.dtype = sizeof(T) == 4 ? 0 : 1;
  k.nt = kBucketThreads;
  k.ppl = PPL;
  k.nbt = NBT;
  k.fn = reinterpret_cast<const void*>(&fps_multi_kernel<T, kBucketThreads, PPL, NBT, KM>);
  k.smem_per_bucket = 0;
  return k;
}

const BucketInst* multi_instances(int* count) {
  static const BucketInst insts[] = {
      make_minst<float, 1, 1, 8>(),  make_minst<float, 1, 2, 8>(),  make_minst<float, 1, 4, 8>(),
      make_minst<float, 1, 8, 8>(),  make_minst<float, 2, 4, 8>(),  make_minst<float, 2, 8, 8>(),
      make_minst<float, 4, 8, 8>(),  make_minst<double, 1, 1, 8>(), make_minst<double, 1, 2, 8>(),
      make_minst<double, 1, 4, 8>(), make_minst<double, 1, 8, 8>(), make_minst<double, 2, 8, 8>(),
      make_minst<double, 4, 8, 8>(),
  };
  *count = (int)(sizeof(insts) / sizeof(insts[0]));
  return insts;
}

}  // namespace ffps
