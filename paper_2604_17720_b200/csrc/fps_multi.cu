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
//   2. the warp re-evaluates its flagged buckets against all J points, up to
//      4 buckets per batch so their L2 round trips overlap: new key (value,
//      position, xyz) and second best v2 into the owner lane's registers; the
//      selected points themselves -> -inf;
//   3. warp maxima -> | barrier | -> tau = smallest warp maximum; every owned
//      key >= tau joins a candidate list (each of the NW >= KM warps holds one,
//      so the global top-KM is in it) -> | barrier |
//   4. warp 0 selects the top-KM of the list, tests (a) and (b) for all pairs
//      at once, writes the accepted prefix -> | barrier |
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

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
  constexpr int NREC = 128;              // capacity of the candidate list
  constexpr int RPL = NREC / 32;         // list entries per lane in the merge
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

  // candidate list (keys >= tau), warp maxima, flagged-bucket lists and the
  // accepted points of the round
  __shared__ bits_t wm_s[NW];
  __shared__ int32_t wl_s[NW][32 * NBT];
  __shared__ uint32_t wm2_s[NW][32 * NBT];  // points (of the J) flagging each listed bucket
  __shared__ int ncand_s;
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
    unsigned fm[NBT];  // warp ballot: bucket flagged
    unsigned pm[NBT];  // lane: which of the J points flag its bucket
#pragma unroll
    for (int j = 0; j < NBT; ++j) pm[j] = 0u;
    for (int t = 0; t < J; ++t) {
      const T px = sp_s[t][0], py = sp_s[t][1], pz = sp_s[t][2];
      const int sq = sq_s[t];
      const pair_t ppx = A::mk(-px, px), ppy = A::mk(-py, py), ppz = A::mk(-pz, pz);
#pragma unroll
      for (int j = 0; j < NBT; ++j) {
        const int q = j * NT + lane * NW + warp;
        const T lb = A::box_d2_pairs(lnh[j], ppx, ppy, ppz, nz);
        const bool f = q < nb && (round == 0 || q == sq || !(lb >= A::from_bits(ov[j])));
        pm[j] |= (unsigned)f << t;
      }
    }
#pragma unroll
    for (int j = 0; j < NBT; ++j) fm[j] = __ballot_sync(0xffffffffu, pm[j] != 0u);
    if (trace) t1 = clock64();
    // 2. re-evaluate the flagged buckets against all J points: compacted per-warp
    //    list, up to 4 buckets per batch so their L2 round trips overlap ---------
    int nf = 0;
#pragma unroll
    for (int j = 0; j < NBT; ++j) {
      if ((fm[j] >> lane) & 1u) {
        const int e = nf + __popc(fm[j] & ((1u << lane) - 1u));
        wl_s[warp][e] = j * NT + lane * NW + warp;
        wm2_s[warp][e] = pm[j];
      }
      nf += __popc(fm[j]);
    }
    __syncwarp();
    auto batch = [&](auto chn, int e0) {
      constexpr int CH = decltype(chn)::value;
      int qc[CH];
      T xs[CH][PPL], ys[CH][PPL], zs[CH][PPL], ds[CH][PPL], d0[CH][PPL];
      uint32_t os[CH][PPL];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        qc[c] = wl_s[warp][e0 + c];
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          const int64_t s = (int64_t)qc[c] * BS + u * 32 + lane;
          xs[c][u] = X[s];
          ys[c][u] = Y[s];
          zs[c][u] = Z[s];
          ds[c][u] = D[s];
          os[c][u] = (uint32_t)O[s];
          d0[c][u] = ds[c][u];
        }
      }
      // only the points that flagged a bucket can change it (bound argument)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        unsigned pmask = wm2_s[warp][e0 + c];
        while (pmask) {
          const int t = __ffs(pmask) - 1;
          pmask &= pmask - 1u;
          const T px = sp_s[t][0], py = sp_s[t][1], pz = sp_s[t][2];
          const uint32_t pw = si_s[t];
#pragma unroll
          for (int u = 0; u < PPL; ++u) {
            T nd = A::vmin(ds[c][u], A::d2(xs[c][u], ys[c][u], zs[c][u], px, py, pz));  // :93
            if (os[c][u] == pw) nd = A::ninf();                                          // :169
            ds[c][u] = nd;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int q = qc[c];
        bits_t b1 = A::kmin, b2 = A::kmin;
        uint32_t i1 = kNoIdx;
        T x1 = T(0), y1 = T(0), z1 = T(0);
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          if (A::bits(ds[c][u]) != A::bits(d0[c][u])) D[(int64_t)q * BS + u * 32 + lane] = ds[c][u];
          const bits_t v = A::bits(ds[c][u]);
          if (v > b1 || (v == b1 && os[c][u] < i1)) {
            b2 = b1;
            b1 = v;
            i1 = os[c][u];
            x1 = xs[c][u];
            y1 = ys[c][u];
            z1 = zs[c][u];
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
        const int jq = q / NT, ol = (q % NT) / NW;
        if (lane == ol) {
#pragma unroll
          for (int j = 0; j < NBT; ++j)
            if (j == jq) {
              ov[j] = wv;
              oi[j] = wi;
              o2[j] = w2;
              ox[j] = x1;
              oy[j] = y1;
              oz[j] = z1;
            }
        }
      }
    };
    constexpr int MAXCH = PPL >= 4 ? 1 : 4 / PPL;  // <= 4 points per lane in flight
    for (int e0 = 0; e0 < nf; e0 += MAXCH) {
      const int r = nf - e0;
      if (r >= MAXCH) batch(std::integral_constant<int, MAXCH>{}, e0);
      else if (MAXCH > 2 && r == 3) batch(std::integral_constant<int, (MAXCH > 2 ? 3 : 1)>{}, e0);
      else if (MAXCH > 1 && r == 2) batch(std::integral_constant<int, (MAXCH > 1 ? 2 : 1)>{}, e0);
      else batch(std::integral_constant<int, 1>{}, e0);
    }
    if (trace) t2 = clock64();
    // 3. candidates: every owned key >= tau, tau = the smallest warp maximum (each
    //    of the NW >= KM warps holds a key >= tau, so the global top-KM is among
    //    them) ------------------------------------------------------------------------
    {
      bits_t tv = A::kmin;
#pragma unroll
      for (int j = 0; j < NBT; ++j) tv = ov[j] > tv ? ov[j] : tv;
      const bits_t wv = A::warp_max(tv);
      if (lane == 0) wm_s[warp] = wv;
      if (tid == 0) ncand_s = 0;
    }
    if (trace) t3 = clock64();
    __syncthreads();  // B1: warp maxima visible, list empty
    {
      const bits_t wv = lane < NW ? wm_s[lane] : A::bits(A::pinf());
      const bits_t tau = -A::warp_max(-wv);  // min over the NW warp maxima
#pragma unroll
      for (int j = 0; j < NBT; ++j) {
        const bool c = ov[j] >= tau && ov[j] != A::kmin;
        const unsigned m = __ballot_sync(0xffffffffu, c);
        if (m) {
          int base = 0;
          if (lane == 0) base = atomicAdd(&ncand_s, __popc(m));
          base = __shfl_sync(0xffffffffu, base, 0);
          const int e = base + __popc(m & ((1u << lane) - 1u));
          if (c && e < NREC) {
            rv_s[e] = ov[j];
            ri_s[e] = oi[j];
            r2_s[e] = o2[j];
            rq_s[e] = j * NT + lane * NW + warp;
            rx_s[e][0] = ox[j];
            rx_s[e][1] = oy[j];
            rx_s[e][2] = oz[j];
          }
        }
      }
    }
    __syncthreads();  // B2: candidate list complete
    // 4. warp 0: global top-KM, chain test, accepted prefix ------------------------
    const int ncand = ncand_s;
    if (ncand > NREC) {
      // more than NREC keys at or above tau (massive ties, exhausted buckets):
      // take just the exact argmax this round (one more barrier, CTA-uniform)
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
      T cx = ox[0], cy = oy[0], cz = oz[0];
#pragma unroll
      for (int j = 1; j < NBT; ++j)
        if (tj == j) {
          cx = ox[j];
          cy = oy[j];
          cz = oz[j];
        }
      const int wl = argmax_lane<A>(tv, ti);
      __syncthreads();  // everyone is done reading the list before it is reused
      if (lane == wl) {
        rv_s[warp] = tv;
        ri_s[warp] = ti;
        rq_s[warp] = tj * NT + lane * NW + warp;
        rx_s[warp][0] = cx;
        rx_s[warp][1] = cy;
        rx_s[warp][2] = cz;
      }
      __syncthreads();
      if (warp == 0) {
        const bits_t v = lane < NW ? rv_s[lane] : A::kmin;
        const uint32_t i = lane < NW ? ri_s[lane] : kNoIdx;
        const int gl = argmax_lane<A>(v, i);
        if (lane == 0) {
          sp_s[0][0] = rx_s[gl][0];
          sp_s[0][1] = rx_s[gl][1];
          sp_s[0][2] = rx_s[gl][2];
          si_s[0] = ri_s[gl];
          sq_s[0] = rq_s[gl];
          order[k] = ri_s[gl];  // fps_core.py:167-168
          sel[k] = A::from_bits(rv_s[gl]);
          nsel_s = 1;
        }
      }
    } else if (warp == 0) {
      bits_t lv[RPL];
      uint32_t li[RPL];
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int e = lane + 32 * t;
        lv[t] = e < ncand && e < NREC ? rv_s[e] : A::kmin;
        li[t] = e < ncand && e < NREC ? ri_s[e] : kNoIdx;
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
