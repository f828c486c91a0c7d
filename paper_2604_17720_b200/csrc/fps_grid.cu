// K1g — multi-winner bucketed farthest-point sampling with a cell index.
//
// Same contract and bit-exact results as K1 / K1b / K1m (restates
// run_kernel, reference pkg/src/flashfps/fps_core.py:110-175).
//
// K1m tests every bucket against every point selected in a round, although a
// point can only change buckets within its influence radius.  K1g keeps the
// bucket state in shared memory and indexes the buckets by a uniform grid of
// cells (CSR: cell -> buckets whose box overlaps it), so a selected point p
// only tests the buckets registered in the cells of the cube
// [p - R, p + R]^3 where R^2 is an upper bound of every bucket's key:
//   R^2 = the distance of the first winner of the previous round (keys only
//   decrease, and that winner was the maximum then).
// A bucket outside the cube has box_d2(p, box) >= R^2 >= its key, so the
// exact test of K1b would not flag it either — the flagged set, and therefore
// every result, is unchanged.  Buckets spanning more than kMaxCells cells are
// kept in an "oversize" list tested against every point; while the cube is
// large (early rounds) all buckets are tested.
//
// A round (J points selected by the previous round, J <= KM):
//   A. flag: every selected point tests its candidate buckets exactly
//      (box_d2 with the reference's rounded ops); hits OR the point's bit into
//      the bucket's mask and append new buckets to the round list
//   | barrier |
//   B. re-evaluate the round list (balanced over warps, up to 4 buckets per
//      batch): apply only the points in each bucket's mask -> new key (value,
//      position, xyz) and second-best value into the bucket table
//   | barrier |
//   C. per-warp max over a contiguous slice of the table | barrier | every key
//      >= tau, the KM-th largest warp max, joins the candidate list | barrier |
//   D. every warp: top-KM of the list by rank, chain test (K1m), accepted
//      prefix into its own copy (identical in all warps, no barrier)
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "arith.cuh"
#include "ffps_internal.h"

namespace ffps {

namespace {

constexpr int kMaxCells = 27;  // a bucket registered in at most this many cells
constexpr int kEntryBudget = 12;  // cell entries per bucket on average (shared budget)

template <typename A>
__device__ __forceinline__ int argmax_lane_g(typename A::bits_t v, uint32_t i) {
  const typename A::bits_t wv = A::warp_max(v);
  const uint32_t wi = __reduce_min_sync(0xffffffffu, v == wv ? i : 0xffffffffu);
  return __ffs(__ballot_sync(0xffffffffu, v == wv && i == wi)) - 1;
}

// box_d2 of point p to box {lo.xyz, hi.xyz} with the reference's rounded ops
__device__ __forceinline__ float box_lb(float px, float py, float pz, const float* b) {
  const float gx = max3f(__fsub_rn(b[0], px), __fsub_rn(px, b[3]), 0.0f);
  const float gy = max3f(__fsub_rn(b[1], py), __fsub_rn(py, b[4]), 0.0f);
  const float gz = max3f(__fsub_rn(b[2], pz), __fsub_rn(pz, b[5]), 0.0f);
  return __fadd_rn(__fadd_rn(__fmul_rn(gx, gx), __fmul_rn(gy, gy)), __fmul_rn(gz, gz));
}
__device__ __forceinline__ double box_lb(double px, double py, double pz, const double* b) {
  const double gx = fmax(fmax(__dsub_rn(b[0], px), __dsub_rn(px, b[3])), 0.0);
  const double gy = fmax(fmax(__dsub_rn(b[1], py), __dsub_rn(py, b[4])), 0.0);
  const double gz = fmax(fmax(__dsub_rn(b[2], pz), __dsub_rn(pz, b[5])), 0.0);
  return __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
}

}  // namespace

// dynamic shared memory bytes of fps_grid_kernel for nb buckets
template <typename T>
__host__ __device__ constexpr size_t grid_smem_bytes(int64_t nb, int G) {
  return (size_t)nb * (6 * sizeof(T) + 3 * sizeof(T) + 2 * sizeof(typename Arith<T>::bits_t) +
                       4 /*ki*/ + 4 /*pmask*/ + 4 /*rlist*/ + 2 /*olist*/ +
                       2 * kEntryBudget /*cell entries*/) +
         ((size_t)G * G * G + 1) * 4;
}

template <typename T, int NT, int PPL, int KM>
__global__ void __launch_bounds__(NT, 1) fps_grid_kernel(const BucketParams prm, int G) {
  using A = Arith<T>;
  using bits_t = typename A::bits_t;
  constexpr int NW = NT / 32;
  constexpr int BS = 32 * PPL;
  constexpr uint32_t kNoIdx = 0xffffffffu;
  constexpr int NREC = 128;
  constexpr int RPL = NREC / 32;
  static_assert(KM <= 32, "one candidate per lane in the chain test");
  static_assert(NW >= KM, "KM warp maxima, at least one warp per point");
  constexpr int WPP = NW / KM >= 2 ? 2 : 1;  // warps per selected point in the flag phase

  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = (int)prm.nbuckets;
  const int NC = G * G * G;
  const int64_t off = (int64_t)b * prm.nslots;
  const T* __restrict__ X = static_cast<const T*>(prm.X) + off;
  const T* __restrict__ Y = static_cast<const T*>(prm.Y) + off;
  const T* __restrict__ Z = static_cast<const T*>(prm.Z) + off;
  T* __restrict__ D = static_cast<T*>(prm.D) + off;
  const int32_t* __restrict__ O = prm.O + off;
  const T* __restrict__ BB = static_cast<const T*>(prm.BB) + (int64_t)b * nb * 6;

  // ---- shared memory -----------------------------------------------------------
  extern __shared__ __align__(16) unsigned char smem[];
  T* box = reinterpret_cast<T*>(smem);                   // [nb][6]
  T* kx = box + (size_t)nb * 6;                          // [nb][3] key point xyz
  bits_t* kv = reinterpret_cast<bits_t*>(kx + (size_t)nb * 3);  // [nb] key value
  bits_t* k2 = kv + nb;                                  // [nb] second-best value
  uint32_t* ki = reinterpret_cast<uint32_t*>(k2 + nb);   // [nb] key position
  uint32_t* pmask = ki + nb;                             // [nb] flagging points of the round
  int32_t* rlist = reinterpret_cast<int32_t*>(pmask + nb);  // [nb] round list
  uint32_t* coff = reinterpret_cast<uint32_t*>(rlist + nb);  // [NC + 1] cell -> end offset
  uint16_t* cent = reinterpret_cast<uint16_t*>(coff + NC + 1);  // [nb * kEntryBudget]
  uint16_t* olist = cent + (size_t)nb * kEntryBudget;           // [nb] oversize buckets
  __shared__ bits_t wm_s[NW];
  __shared__ bits_t rv_s[NREC], r2_s[NREC];
  __shared__ uint32_t ri_s[NREC];
  __shared__ int32_t rq_s[NREC];
  __shared__ T rx_s[NREC][3];
  // accepted points of the last round: every warp keeps its own copy (all
  // warps derive the same set from the candidate list, no barrier needed)
  __shared__ T sp_w[NW][KM][3];
  __shared__ uint32_t si_w[NW][KM];
  __shared__ int32_t sq_w[NW][KM];
  __shared__ int16_t top_w[NW][KM];
  __shared__ int ncand_s, rcount_s, ocount_s, ebudget_s;
  __shared__ T glo_s[3], ginv_s[3];
  __shared__ T red_s[2][NW][3];
  __shared__ uint32_t cscr_s[NW][2][32];  // per-warp cell scratch of the flag phase

  // ---- bucket table ------------------------------------------------------------
  T lo[3] = {A::pinf(), A::pinf(), A::pinf()}, hi[3] = {A::ninf(), A::ninf(), A::ninf()};
  for (int q = tid; q < nb; q += NT) {
#pragma unroll
    for (int c = 0; c < 6; ++c) box[q * 6 + c] = BB[(int64_t)q * 6 + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      lo[c] = box[q * 6 + c] < lo[c] ? box[q * 6 + c] : lo[c];
      hi[c] = box[q * 6 + 3 + c] > hi[c] ? box[q * 6 + 3 + c] : hi[c];
    }
    kv[q] = k2[q] = A::bits(A::pinf());
    ki[q] = kNoIdx;
    kx[q * 3 + 0] = kx[q * 3 + 1] = kx[q * 3 + 2] = T(0);
    pmask[q] = 0u;
  }
  for (int c = tid; c <= NC; c += NT) coff[c] = 0u;
  // cloud box -> grid
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    for (int o = 16; o > 0; o >>= 1) {
      const T a = __shfl_xor_sync(0xffffffffu, lo[c], o), z = __shfl_xor_sync(0xffffffffu, hi[c], o);
      lo[c] = a < lo[c] ? a : lo[c];
      hi[c] = z > hi[c] ? z : hi[c];
    }
    if (lane == 0) {
      red_s[0][warp][c] = lo[c];
      red_s[1][warp][c] = hi[c];
    }
  }
  if (tid == 0) {
    ocount_s = 0;
    rcount_s = 0;
    ebudget_s = nb * kEntryBudget;
  }
  __syncthreads();
  if (tid < 3) {
    T a = A::pinf(), z = A::ninf();
    for (int w = 0; w < NW; ++w) {
      a = red_s[0][w][tid] < a ? red_s[0][w][tid] : a;
      z = red_s[1][w][tid] > z ? red_s[1][w][tid] : z;
    }
    glo_s[tid] = a;
    ginv_s[tid] = z > a ? (T)G / (z - a) : T(0);
  }
  __syncthreads();
  const T glo[3] = {glo_s[0], glo_s[1], glo_s[2]}, ginv[3] = {ginv_s[0], ginv_s[1], ginv_s[2]};
  auto cellc = [&](T v, int c) -> int {  // monotone in v
    const int i = (int)((v - glo[c]) * ginv[c]);
    return i < 0 ? 0 : (i >= G ? G - 1 : i);
  };
  // register every bucket in the cells its box overlaps (<= kMaxCells cells,
  // within the shared entry budget), the rest as oversize; pmask marks the
  // registered buckets during the build
  for (int pass = 0; pass < 2; ++pass) {
    for (int q = tid; q < nb; q += NT) {
      int c0[3], c1[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        c0[c] = cellc(box[q * 6 + c], c);
        c1[c] = cellc(box[q * 6 + 3 + c], c);
      }
      const int cnt = (c1[0] - c0[0] + 1) * (c1[1] - c0[1] + 1) * (c1[2] - c0[2] + 1);
      if (pass == 0) {
        const bool reg = cnt <= kMaxCells && atomicSub(&ebudget_s, cnt) >= cnt;
        pmask[q] = reg ? 1u : 0u;
        if (!reg) {
          olist[atomicAdd(&ocount_s, 1)] = (uint16_t)q;
          continue;
        }
      } else if (pmask[q] == 0u) {
        continue;
      }
      for (int x = c0[0]; x <= c1[0]; ++x)
        for (int y = c0[1]; y <= c1[1]; ++y)
          for (int z = c0[2]; z <= c1[2]; ++z) {
            const int cell = (x * G + y) * G + z;
            if (pass == 0) atomicAdd(&coff[cell + 1], 1u);
            else cent[atomicAdd(&coff[cell], 1u)] = (uint16_t)q;
          }
    }
    __syncthreads();
    if (pass == 0) {  // exclusive scan: coff[c] = start of cell c
      if (warp == 0) {
        uint32_t carry = 0;
        for (int c0 = 0; c0 <= NC; c0 += 32) {
          const int c = c0 + lane;
          uint32_t v = c <= NC ? coff[c] : 0u;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
          }
          if (c <= NC) coff[c] = v + carry;
          carry += __shfl_sync(0xffffffffu, v, 31);
        }
      }
      __syncthreads();
    }
  }
  for (int q = tid; q < nb; q += NT) pmask[q] = 0u;
  __syncthreads();
  // after the fill pass coff[c] = end of cell c (= start of c + 1), start(c) = coff[c - 1]

  // ---- seed (fps_core.py:124-130) -----------------------------------------------
  const int seed = (int)prm.seed_pos[b];
  int64_t* order = prm.order + (int64_t)b * prm.out_stride;
  T* sel = static_cast<T*>(prm.sel_d2) + (int64_t)b * prm.out_stride;
  if (lane == 0) {
    const T* X0 = static_cast<const T*>(prm.xyz) + (int64_t)b * prm.cloud_stride * 3;
    const int64_t src = prm.index_map ? prm.index_map[(int64_t)b * prm.map_stride + seed] : seed;
    sp_w[warp][0][0] = X0[3 * src + 0];
    sp_w[warp][0][1] = X0[3 * src + 1];
    sp_w[warp][0][2] = X0[3 * src + 2];
    si_w[warp][0] = (uint32_t)seed;
    sq_w[warp][0] = -1;
  }
  if (tid == 0) {
    order[0] = seed;
    sel[0] = A::pinf();
  }
  int J = 1;                        // points accepted by the last round
  bits_t rmax = A::bits(A::pinf());  // upper bound of every key (R^2 of the cube)
  __syncthreads();
  const int iters = (int)prm.iters;
  const int nover = ocount_s;
  long long* trace =
      (prm.trace && b == 0 && lane == 0) ? prm.trace + (int64_t)warp * prm.trace_iters * 8 : nullptr;

  auto flag = [&](int q, int t) {  // OR point t into bucket q's mask, list it once
    const uint32_t old = atomicOr(&pmask[q], 1u << t);
    if (old == 0u) rlist[atomicAdd(&rcount_s, 1)] = q;
  };
  auto test = [&](int q, int t, T px, T py, T pz) {  // K1b's exact bound test
    if (!(box_lb(px, py, pz, box + (size_t)q * 6) >= A::from_bits(kv[q]))) flag(q, t);
  };
  // warp-converged variant: every lane calls it (valid = has a bucket to test);
  // new buckets are appended with one shared-memory atomic per warp
  auto test_warp = [&](bool valid, int q, int t, T px, T py, T pz) {
    bool isnew = false;
    if (valid && !(box_lb(px, py, pz, box + (size_t)q * 6) >= A::from_bits(kv[q])))
      isnew = atomicOr(&pmask[q], 1u << t) == 0u;
    const unsigned m = __ballot_sync(0xffffffffu, isnew);
    if (m) {
      int base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(&rcount_s, __popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      if (isnew) rlist[base + __popc(m & ((1u << lane) - 1u))] = q;
    }
  };

  int k = 1;
  for (int round = 0; k < iters; ++round) {
    long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    int ntest_w = 0;  // traced: entries tested by this warp
    if (trace) t0 = clock64();
    // A. flag ---------------------------------------------------------------------
    const T r2 = A::from_bits(rmax);
    // half-width of the search cube, padded for the rounding of p +- R
    const T R = round == 0 ? A::pinf() : (T)(sqrt((double)r2) * 1.001) ;
    bool full = round == 0 || !(R * ginv[0] < T(3)) || !(R * ginv[1] < T(3)) ||
                !(R * ginv[2] < T(3));
    if (full) {  // every bucket against every point
      for (int q = tid; q < nb; q += NT) {
        if (round == 0) {
          flag(q, 0);
          continue;
        }
        for (int t = 0; t < J; ++t) test(q, t, sp_w[warp][t][0], sp_w[warp][t][1], sp_w[warp][t][2]);
      }
      if (round > 0 && warp == 0 && lane < J && sq_w[0][lane] >= 0)
        flag(sq_w[0][lane], lane);  // the point -> -inf
    } else {
      // two warps per point (NW >= 2 * KM); the (cell, entry) pairs of the
      // point's cube are spread over the 64 lanes: per chunk of 32 cells the
      // warp publishes each cell's first entry and inclusive entry count in
      // shared scratch, then every lane walks flat entry indices
      for (int t = warp / WPP; t < J; t += NW / WPP) {
        const int half = warp % WPP;
        const T px = sp_w[warp][t][0], py = sp_w[warp][t][1], pz = sp_w[warp][t][2];
        const T pad = (fabs(px) + fabs(py) + fabs(pz) + T(1)) * T(1e-6);
        int c0[3], c1[3];
        const T pc[3] = {px, py, pz};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          c0[c] = cellc(pc[c] - R - pad, c);
          c1[c] = cellc(pc[c] + R + pad, c);
        }
        const int ny = c1[1] - c0[1] + 1, nz = c1[2] - c0[2] + 1;
        const int ncells = (c1[0] - c0[0] + 1) * ny * nz;
        uint32_t* cs = cscr_s[warp][0];  // first entry of each cell of the chunk
        uint32_t* ci = cscr_s[warp][1];  // inclusive entry count
        for (int cb = 0; cb < ncells; cb += 32) {
          const int i = cb + lane;
          uint32_t e0 = 0, cntc = 0;
          if (i < ncells) {
            const int x = c0[0] + i / (ny * nz), y = c0[1] + (i / nz) % ny, z = c0[2] + i % nz;
            const int cell = (x * G + y) * G + z;
            e0 = cell == 0 ? 0u : coff[cell - 1];
            cntc = coff[cell] - e0;
          }
          uint32_t incl = cntc;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
          }
          const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
          ntest_w += (int)total;
          cs[lane] = e0;
          ci[lane] = incl;
          __syncwarp();
          for (uint32_t f0 = 32 * half; f0 < total; f0 += 32 * WPP) {  // uniform trip count
            const uint32_t f = f0 + lane;
            int q = 0;
            if (f < total) {
              int lo_l = 0, hi_l = 31;  // lowest cell whose inclusive count > f
              while (lo_l < hi_l) {
                const int mid = (lo_l + hi_l) >> 1;
                if (ci[mid] > f) hi_l = mid;
                else lo_l = mid + 1;
              }
              const uint32_t before = lo_l == 0 ? 0u : ci[lo_l - 1];
              q = cent[cs[lo_l] + (f - before)];
            }
            test_warp(f < total, q, t, px, py, pz);
          }
          __syncwarp();
        }
        for (int i0 = 32 * half; i0 < nover; i0 += 32 * WPP) {
          const int i = i0 + lane;
          test_warp(i < nover, i < nover ? olist[i] : 0, t, px, py, pz);
        }
        if (lane == 0 && half == 0 && sq_w[warp][t] >= 0) flag(sq_w[warp][t], t);  // -> -inf
      }
    }
    if (trace) t1 = clock64();
    __syncthreads();  // flags and round list complete
    // B. re-evaluate the round list --------------------------------------------------
    const int nr = rcount_s;
    auto batch = [&](auto chn, int e0) {
      constexpr int CH = decltype(chn)::value;
      int qc[CH];
      uint32_t pm[CH];
      T xs[CH][PPL], ys[CH][PPL], zs[CH][PPL], ds[CH][PPL], d0[CH][PPL];
      uint32_t os[CH][PPL];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        qc[c] = rlist[e0 + c * NW];
        pm[c] = pmask[qc[c]];
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
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        unsigned m = pm[c];
        while (m) {  // only the points that flagged the bucket can change it
          const int t = __ffs(m) - 1;
          m &= m - 1u;
          const T px = sp_w[warp][t][0], py = sp_w[warp][t][1], pz = sp_w[warp][t][2];
          const uint32_t pw = si_w[warp][t];
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
        const int wl = argmax_lane_g<A>(b1, i1);
        const bits_t w2 = A::warp_max(lane == wl ? b2 : b1);
        if (lane == wl) {
          kv[q] = b1;
          ki[q] = i1;
          k2[q] = w2;
          kx[q * 3 + 0] = x1;
          kx[q * 3 + 1] = y1;
          kx[q * 3 + 2] = z1;
          pmask[q] = 0u;
        }
      }
    };
    {
      constexpr int CH = PPL <= 1 ? 4 : (PPL == 2 ? 2 : 1);  // <= 4 points per lane in flight
      int e = warp;
      for (; e + (CH - 1) * NW < nr; e += CH * NW) batch(std::integral_constant<int, CH>{}, e);
      for (; e < nr; e += NW) batch(std::integral_constant<int, 1>{}, e);
    }
    if (trace) t2 = clock64();
    __syncthreads();  // keys final for this round
    if (tid == 0) rcount_s = 0;
    // C. candidates: keys >= tau, tau = smallest warp maximum over table slices ------
    const int per = (nb + NW - 1) / NW;
    const int s0 = warp * per, s1 = s0 + per < nb ? s0 + per : nb;
    {
      bits_t mv = A::kmin;
      for (int q = s0 + lane; q < s1; q += 32) mv = kv[q] > mv ? kv[q] : mv;
      mv = A::warp_max(mv);
      if (lane == 0) wm_s[warp] = mv;
      if (tid == 0) ncand_s = 0;
    }
    __syncthreads();
    {
      // tau = the KM-th largest warp maximum: KM warps hold a key >= tau, so
      // the global top-KM is among the keys >= tau (ties at tau included)
      bits_t tau;
      {
        const bits_t mine = lane < NW ? wm_s[lane] : A::kmin;
        int rank = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const bits_t o = wm_s[w];
          rank += (o > mine || (o == mine && w < lane)) ? 1 : 0;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, lane < NW && rank == KM - 1);
        tau = A::shfl(mine, hit ? __ffs(hit) - 1 : 0);
      }
      for (int q0 = s0; q0 < s1; q0 += 32) {
        const int q = q0 + lane;
        const bool c = q < s1 && kv[q] >= tau && kv[q] != A::kmin;
        const unsigned m = __ballot_sync(0xffffffffu, c);
        if (m) {
          int base = 0;
          if (lane == 0) base = atomicAdd(&ncand_s, __popc(m));
          base = __shfl_sync(0xffffffffu, base, 0);
          const int e = base + __popc(m & ((1u << lane) - 1u));
          if (c && e < NREC) {
            rv_s[e] = kv[q];
            ri_s[e] = ki[q];
            r2_s[e] = k2[q];
            rq_s[e] = q;
            rx_s[e][0] = kx[q * 3 + 0];
            rx_s[e][1] = kx[q * 3 + 1];
            rx_s[e][2] = kx[q * 3 + 2];
          }
        }
      }
    }
    if (trace) t3 = clock64();
    __syncthreads();  // candidate list complete
    // D. every warp: top-KM of the list by rank, chain test, accepted prefix --------
    //    (identical in all warps; warp 0 reports them)
    const int ncand = ncand_s;
    int acc = 1;
    if (ncand > NREC) {
      // massive ties: one exact winner from the whole table this round
      bits_t bv = A::kmin;
      uint32_t bi = kNoIdx;
      int bq = 0;
      for (int q = lane; q < nb; q += 32)
        if (kv[q] > bv || (kv[q] == bv && ki[q] < bi)) {
          bv = kv[q];
          bi = ki[q];
          bq = q;
        }
      const int wl = argmax_lane_g<A>(bv, bi);
      const int q = __shfl_sync(0xffffffffu, bq, wl);
      if (lane == 0) {
        sp_w[warp][0][0] = kx[q * 3 + 0];
        sp_w[warp][0][1] = kx[q * 3 + 1];
        sp_w[warp][0][2] = kx[q * 3 + 2];
        si_w[warp][0] = ki[q];
        sq_w[warp][0] = q;
        if (warp == 0) {
          order[k] = ki[q];  // fps_core.py:167-168
          sel[k] = A::from_bits(kv[q]);
        }
      }
      rmax = kv[q];
    } else {
      // rank of every list entry = number of larger keys (value desc, position asc)
      for (int e = lane; e < ncand; e += 32) {
        const bits_t v = rv_s[e];
        const uint32_t i = ri_s[e];
        int rank = 0;
        for (int e2 = 0; e2 < ncand && rank < KM; ++e2) {
          const bits_t v2 = rv_s[e2];
          rank += (v2 > v || (v2 == v && ri_s[e2] < i)) ? 1 : 0;
        }
        if (rank < KM) top_w[warp][rank] = (int16_t)e;
      }
      __syncwarp();
      const int nc = ncand < KM ? ncand : KM;
      const bool live = lane < nc;
      const int cand = live ? top_w[warp][lane] : 0;
      const bits_t cv = live ? rv_s[cand] : A::kmin;
      const bits_t c2 = live ? r2_s[cand] : A::kmin;
      const T cx = live ? rx_s[cand][0] : T(0);
      const T cy = live ? rx_s[cand][1] : T(0);
      const T cz = live ? rx_s[cand][2] : T(0);
      bool ok = live && A::from_bits(cv) >= T(0);
      for (int bb = 0; bb < KM - 1; ++bb) {
        const T bx = __shfl_sync(0xffffffffu, cx, bb);
        const T by = __shfl_sync(0xffffffffu, cy, bb);
        const T bz = __shfl_sync(0xffffffffu, cz, bb);
        const bits_t b2 = A::shfl(c2, bb);
        if (bb < lane && ok)
          ok = !(A::d2(cx, cy, cz, bx, by, bz) < A::from_bits(cv)) && cv > b2;  // (a), (b)
      }
      const unsigned okm = __ballot_sync(0xffffffffu, ok || lane == 0);
      acc = __ffs(~okm) - 1;
      if (acc < 0 || acc > KM) acc = KM;
      if (acc > iters - k) acc = iters - k;
      if (lane < acc) {
        sp_w[warp][lane][0] = cx;
        sp_w[warp][lane][1] = cy;
        sp_w[warp][lane][2] = cz;
        si_w[warp][lane] = ri_s[cand];
        sq_w[warp][lane] = rq_s[cand];
        if (warp == 0) {
          order[k + lane] = ri_s[cand];  // fps_core.py:167-168
          sel[k + lane] = A::from_bits(cv);
        }
      }
      rmax = A::shfl(cv, 0);
    }
    __syncwarp();
    J = acc;
    if (trace && round < prm.trace_iters) {
      long long* rr = trace + (int64_t)round * 8;
      rr[0] = t0; rr[1] = t1; rr[2] = t2; rr[3] = t3; rr[4] = clock64(); rr[5] = acc;
      rr[6] = nr; rr[7] = (long long)full | ((long long)nover << 1) | ((long long)ntest_w << 24);
    }
    k += acc;
  }

  // positions -> original indices for restricted runs (fps_cache.py:197)
  if (prm.index_map != nullptr) {
    __syncthreads();
    const int64_t* map = prm.index_map + (int64_t)b * prm.map_stride;
    for (int kk = tid; kk < iters; kk += NT) order[kk] = __ldg(map + order[kk]);
  }
}

template <typename T, int PPL, int KM>
GridInst make_ginst() {
  GridInst k;
  k.dtype = sizeof(T) == 4 ? 0 : 1;
  k.nt = kBucketThreads;
  k.ppl = PPL;
  k.km = KM;
  k.fn = reinterpret_cast<const void*>(&fps_grid_kernel<T, kBucketThreads, PPL, KM>);
  k.esz = sizeof(T);
  return k;
}

const GridInst* grid_instances(int* count) {
  static const GridInst insts[] = {
      make_ginst<float, 1, 8>(),  make_ginst<float, 2, 8>(),  make_ginst<float, 4, 8>(),
      make_ginst<float, 8, 8>(),  make_ginst<double, 1, 8>(), make_ginst<double, 2, 8>(),
      make_ginst<double, 4, 8>(), make_ginst<double, 8, 8>(),
  };
  *count = (int)(sizeof(insts) / sizeof(insts[0]));
  return insts;
}

size_t grid_smem(int dtype, int64_t nb, int G) {
  return dtype == 0 ? grid_smem_bytes<float>(nb, G) : grid_smem_bytes<double>(nb, G);
}

}  // namespace ffps
