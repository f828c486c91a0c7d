// K1g — multi-winner bucketed farthest-point sampling with a bucket-group index.
//
// Same contract and bit-exact results as K1 / K1s / K1b / K1m (restates
// run_kernel, reference pkg/src/flashfps/fps_core.py:110-175).
//
// A round selects up to KM consecutive greedy winners from one reduction: the
// bucket keys (best point of each bucket) in argmax order c_1, c_2, ...; c_j is
// the winner right after c_1..c_{j-1} if (a) d2(c_j, c_i) >= dist(c_j) and
// (b) dist(c_j) > the second-best distance of c_i's bucket, for every i < j
// (every other distance only decreases, every other key ranks below c_j).
//
// The bucket table lives in shared memory (boxes, key value / position / xyz,
// second best, the round's point mask).  Buckets are grouped by kGS = 32
// consecutive rows (kd order keeps a group compact): each group has a union
// box, its NCG best keys (candidates) and its (NCG+1)-th value.  A cloud's
// buckets are split over a cluster of CL CTAs (bucket q -> rank q % CL).
//
// A round (J points accepted by the previous round, J <= KM):
//   A. flag: warps per point test the group boxes against the group maxima
//      (a group with box_d2 >= its max key holds no bucket the point can flag);
//      | barrier | every hit (point, group) pair tests the group's 32 bucket
//      boxes, one per lane, with the reference's rounded ops; a hit ORs the
//      point's bit into the bucket's mask, the first one lists the bucket.
//      While the search radius (the first winner's distance of the previous
//      round, an upper bound of every key) is large, every bucket is tested.
//   | barrier |
//   B. re-evaluate the listed buckets (balanced over the warps, up to 4 in
//      flight): only the points in each bucket's mask -> new key (value,
//      position, xyz) and second best; the group is marked dirty
//   | barrier |
//   C. dirty groups: NCG best keys and the next value
//   | barrier |
//   R. R1: groups ranked by their maxima, the top-KM groups' candidates copied
//      to a compact list | barrier | R2: ranks of those candidates
//   | barrier |
//   D. warp 0: the rank's top-KM records (the general path when a top group
//      holds more top keys than candidates), pushed to every cluster peer with
//      st.async + mbarrier, bitonic merge of the CL lists, chain test (a)/(b),
//      accepted prefix published
//   | barrier |
#pragma once
// Kernel template; instantiated per arithmetic / storage type in
// fps_grid.cu (float), fps_grid_f64.cu (double) and fps_grid_mixed.cu (float
// coordinates, binary64 arithmetic: FFPS_F32_F64).
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "arith.cuh"
#include "ffps_internal.h"

namespace ffps {

namespace {

constexpr int kGS = 32;  // buckets per group of the two-level index (one per lane)
constexpr int kTraceW = 16;  // trace words per round and warp (FFPS_TRACE_GRID)
constexpr int kMaxGW = 4;    // dirty-group mask words: <= 128 bucket groups per CTA (host)

// flag phase: J points share the NW warps, wpp = NW / J warps per point;
// warp w serves point t[J][w], part s[J][w] (a table instead of divisions)
constexpr int kWppNW = 16, kWppJ = 16;
struct WppTab {
  unsigned char wpp[kWppJ + 1];
  unsigned char t[kWppJ + 1][kWppNW];
  unsigned char s[kWppJ + 1][kWppNW];
};
constexpr WppTab make_wpp_tab() {
  WppTab w{};
  for (int j = 1; j <= kWppJ; ++j) {
    const int wpp = kWppNW / j;
    w.wpp[j] = (unsigned char)wpp;
    for (int x = 0; x < kWppNW; ++x) {
      w.t[j][x] = (unsigned char)(x / wpp);
      w.s[j][x] = (unsigned char)(x % wpp);
    }
  }
  return w;
}
__constant__ WppTab c_wpp = make_wpp_tab();
// rounds re-test every bucket while the search radius is this large a fraction
// of the cloud's extent (little to prune, the whole CTA shares the work)
#ifndef FFPS_GRID_FULLFRAC
#define FFPS_GRID_FULLFRAC 0.375
#endif
constexpr double kFullFrac = FFPS_GRID_FULLFRAC;

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
// binary64 bound of a box stored as double or as float (float corners are
// exact in double: the same bound as on the upcast box)
template <typename S>
__device__ __forceinline__ double box_lb(double px, double py, double pz, const S* b) {
  const double gx = fmax(fmax(__dsub_rn((double)b[0], px), __dsub_rn(px, (double)b[3])), 0.0);
  const double gy = fmax(fmax(__dsub_rn((double)b[1], py), __dsub_rn(py, (double)b[4])), 0.0);
  const double gz = fmax(fmax(__dsub_rn((double)b[2], pz), __dsub_rn(pz, (double)b[5])), 0.0);
  return __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
}

// Lower bound of the binary64 box_lb above, in binary32 with every operation
// rounded down, for float coordinates p and a float box (FFPS_F32_F64).
// Per step RD32(x) <= the exact value and RN64 of anything at least as large
// is >= it (RD32(x) is a double <= x), so box_lb_rd <= box_lb(double).
// Testing box_lb_rd >= RU32(key) therefore skips only buckets the binary64
// test skips (it may flag a few more; re-evaluating them changes nothing).
__device__ __forceinline__ float box_lb_rd(float px, float py, float pz, const float* b) {
  const float gx = fmaxf(fmaxf(__fsub_rd(b[0], px), __fsub_rd(px, b[3])), 0.0f);
  const float gy = fmaxf(fmaxf(__fsub_rd(b[1], py), __fsub_rd(py, b[4])), 0.0f);
  const float gz = fmaxf(fmaxf(__fsub_rd(b[2], pz), __fsub_rd(pz, b[5])), 0.0f);
  return __fadd_rd(__fadd_rd(__fmul_rd(gx, gx), __fmul_rd(gy, gy)), __fmul_rd(gz, gz));
}

}  // namespace

// dynamic shared memory bytes of fps_grid_kernel for nb buckets (per CTA);
// T = arithmetic type (keys), S = coordinate storage type (boxes, key points)
template <typename T, typename S = T>
__host__ __device__ constexpr size_t grid_smem_bytes(int64_t nb) {
  return (size_t)nb * (6 * sizeof(S) + 3 * sizeof(S) + 2 * sizeof(typename Arith<T>::bits_t) +
                       4 /*ki*/ + 4 /*pmask*/ + 4 /*rlist*/) +
         (size_t)((nb + kGS - 1) / kGS) *
             (6 * sizeof(S) + 6 * sizeof(typename Arith<T>::bits_t) + 14 * 4) +  // NCG <= 4
         (size_t)(nb + (nb + kGS - 1) / kGS) * 4 +  // binary32 shadow keys (FFPS_F32_F64)
         16;  // alignment of the coordinate arrays after the keys
}



// DSMEM record of a cluster rank's local top list (CL > 1), 32-bit words:
// float  [v, pos, x, y, z, v2, q, flag]                     (8 words)
// double [v lo, v hi, v2 lo, v2 hi, x, x, y, y, z, z, pos, q | flag << 30] (12:
//        three 16-byte stores; q < 2^30, read only from live records)
template <typename T>
struct GridRec;
template <>
struct GridRec<float> {
  static constexpr int W = 8;

  __device__ static void send(uint32_t dst, uint32_t bar, int32_t v, int32_t v2, uint32_t pos,
                              int q, float x, float y, float z, uint32_t flag) {
    st_async_v4(dst, bar, (uint32_t)v, pos, __float_as_uint(x), __float_as_uint(y));
    st_async_v4(dst + 16, bar, __float_as_uint(z), (uint32_t)v2, (uint32_t)q, flag);
  }
  __device__ static int32_t v(const uint32_t* w) { return (int32_t)w[0]; }
  __device__ static int32_t v2(const uint32_t* w) { return (int32_t)w[5]; }
  __device__ static uint32_t pos(const uint32_t* w) { return w[1]; }
  __device__ static int q(const uint32_t* w) { return (int)w[6]; }
  __device__ static uint32_t flag(const uint32_t* w) { return w[7]; }
  __device__ static float c(const uint32_t* w, int i) { return __uint_as_float(w[2 + i]); }
};
template <>
struct GridRec<double> {
  static constexpr int W = 12;

  __device__ static void send(uint32_t dst, uint32_t bar, int64_t v, int64_t v2, uint32_t pos,
                              int q, double x, double y, double z, uint32_t flag) {
    st_async_v2_b64(dst, bar, (uint64_t)v, (uint64_t)v2);
    st_async_v2_b64(dst + 16, bar, (uint64_t)__double_as_longlong(x),
                    (uint64_t)__double_as_longlong(y));
    const uint32_t qf = ((uint32_t)q & 0x3fffffffu) | (flag << 30);
    st_async_v2_b64(dst + 32, bar, (uint64_t)__double_as_longlong(z),
                    (uint64_t)pos | ((uint64_t)qf << 32));
  }
  __device__ static int64_t u64(const uint32_t* w, int i) {
    return (int64_t)(((uint64_t)w[2 * i + 1] << 32) | w[2 * i]);
  }
  __device__ static int64_t v(const uint32_t* w) { return u64(w, 0); }
  __device__ static int64_t v2(const uint32_t* w) { return u64(w, 1); }
  __device__ static uint32_t pos(const uint32_t* w) { return w[10]; }
  __device__ static int q(const uint32_t* w) { return (int)(w[11] & 0x3fffffffu); }
  __device__ static uint32_t flag(const uint32_t* w) { return w[11] >> 30; }
  __device__ static double c(const uint32_t* w, int i) { return __longlong_as_double(u64(w, 2 + i)); }
};

// CL = CTAs per cloud (thread-block cluster): bucket q belongs to rank q % CL
// and is row q / CL of that rank's table.  Each rank flags, re-evaluates and
// ranks its own buckets; the ranks' top-KM lists are exchanged through DSMEM
// (st.async + mbarrier, double-buffered by round parity) and merged
// identically by every warp of every rank.
//
// S is the coordinate storage type: T, or float under binary64 arithmetic
// (FFPS_F32_F64) — float coordinates convert exactly to double, so every
// rounded operation, bound and result equals the all-double kernel's.
template <typename T, typename S, int NT, int PPL, int KM, int CL>
__global__ void __launch_bounds__(NT, 1) fps_grid_kernel(const BucketParams prm) {
  using A = Arith<T>;
  using bits_t = typename A::bits_t;
  constexpr int NW = NT / 32;
  constexpr int BS = 32 * PPL;
  constexpr uint32_t kNoIdx = 0xffffffffu;
  static_assert(KM <= 32, "one candidate per lane in the chain test");

  static_assert(CL == 1 || CL == 2 || CL == 4, "cluster of 1, 2 or 4 CTAs");
  static_assert(NW == kWppNW, "flag-phase table sized for 16 warps");
  static_assert(CL * KM <= 32 || (CL == 2 && KM == 32) || (CL == 4 && KM == 16),
                "one exchanged record per lane, two lists of 32, or four lists of 16");
  using R = GridRec<T>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = CL > 1 ? (int)cluster_ctarank() : 0;
  const int b = (int)blockIdx.x / CL;  // cloud
  const int nb = ((int)prm.nbuckets - rank + CL - 1) / CL;  // buckets of this rank
  const int ng = (nb + kGS - 1) / kGS;  // bucket groups (kGS consecutive table rows)
  const int64_t off = (int64_t)b * prm.nslots;
  const S* __restrict__ X = static_cast<const S*>(prm.X) + off;
  const S* __restrict__ Y = static_cast<const S*>(prm.Y) + off;
  const S* __restrict__ Z = static_cast<const S*>(prm.Z) + off;
  T* __restrict__ D = static_cast<T*>(prm.D) + off;
  const int32_t* __restrict__ O = prm.O + off;
  const S* __restrict__ BB = static_cast<const S*>(prm.BB) + (int64_t)b * prm.nbuckets * 6;

  // ---- shared memory -----------------------------------------------------------
  extern __shared__ __align__(16) unsigned char smem[];
  // candidates per group (A/B: FFPS_GRID_NCG16 for KM = 16, at most 4: the
  // per-group shared-memory layout of grid_smem_bytes holds 4)
#ifndef FFPS_GRID_NCG16
#define FFPS_GRID_NCG16 4
#endif
  constexpr int NCG = KM == 16 ? FFPS_GRID_NCG16 : (KM < 16 ? KM / 4 : 4);
  static_assert(NCG >= 1 && NCG <= 4, "grid_smem_bytes sizes 4 candidates per group");
  // keys first (8-byte words under binary64), then the coordinate arrays
  bits_t* kv = reinterpret_cast<bits_t*>(smem);          // [nb] key value
  bits_t* k2 = kv + nb;                                  // [nb] second-best value
  // per group (phase C): max key, the (NCG+1)-th value; candidates NCG*g + k =
  // the group's k-th best key (value, position, table row)
  bits_t* gmax = k2 + nb;                                // [ng] group max key
  bits_t* gnext = gmax + ng;                             // [ng]
  bits_t* cand_v = gnext + ng;                           // [NCG ng]
  S* box = reinterpret_cast<S*>(cand_v + NCG * ng);      // [nb][6]
  // groups: union box and max key of kGS consecutive rows (kd / Morton order
  // keeps them spatially compact); max keys refreshed every round (phase C)
  S* gbox = box + (size_t)nb * 6;                        // [ng][6]
  S* kx = gbox + (size_t)ng * 6;                         // [nb][3] key point xyz
  uint32_t* ki = reinterpret_cast<uint32_t*>(kx + (size_t)nb * 3);  // [nb] key position
  uint32_t* pmask = ki + nb;                             // [nb] flagging points of the round
  int32_t* rlist = reinterpret_cast<int32_t*>(pmask + nb);  // [nb] round list
  uint32_t* cand_p = reinterpret_cast<uint32_t*>(rlist + nb);  // [NCG ng]
  int32_t* cand_q = reinterpret_cast<int32_t*>(cand_p + NCG * ng);  // [NCG ng]
  // FFPS_F32_F64: the flag phase tests in binary32, rounded down, against the
  // keys rounded up (box_lb_rd): shadow keys of the buckets and group maxima
  constexpr bool SHADOW = sizeof(T) == 8 && sizeof(S) == 4;
  float* kv32 = reinterpret_cast<float*>(cand_q + NCG * ng);  // [nb]
  float* gmax32 = kv32 + nb;                                 // [ng]
  // phase D: per-warp candidate list (<= 32)
  __shared__ bits_t cv_w[1][64];
  __shared__ uint32_t ci_w[1][64];
  __shared__ int16_t cq_w[1][64];
  __shared__ int16_t top_s[KM];  // rows of the ranked top-KM candidates
  __shared__ bits_t topv_s[KM];
  __shared__ int topg_s[KM];     // the KM groups with the best maxima (phase R1)
  __shared__ int16_t grank_s[128];  // group -> its rank among them, -1 (general path)
  __shared__ int ngv_s;          // non-empty groups (phase R1)
  __shared__ int rr_s[KM * NCG];  // phase R2 ranks (0x7fffffff: empty)
  // phase R1 -> R2: the candidates of the top-KM groups, group rank major
  // (empty entries: value kmin), so R2 reads them without indirection
  __shared__ bits_t compv_s[KM * NCG];
  __shared__ uint32_t compp_s[KM * NCG];
  __shared__ int compq_s[KM * NCG];
  __shared__ unsigned dmask_s[kMaxGW];  // groups with a re-evaluated bucket this round
  // accepted points of the last round: every warp keeps its own copy (all
  // warps derive the same set from the candidate list, no barrier needed)
  __shared__ T sp_w[1][KM][3];
  __shared__ float sp32_w[SHADOW ? KM : 1][3];  // the same points as float (exact, SHADOW)
  __shared__ uint32_t si_w[1][KM];
  __shared__ int32_t sq_w[1][KM];
  __shared__ int16_t top_w[1][KM];
  __shared__ int acc_s;
  __shared__ bits_t rmax_s;
  // chain test: the ranked candidates' coordinates and bucket bounds,
  // broadcast from shared memory (cheaper than 4-8 shuffles per pair)
  struct __align__(16) ChainRec {
    T x, y, z;
    bits_t b2;
  };
  __shared__ ChainRec ch_s[KM];
  __shared__ int rcount_s, npair_s, ndirty_s;
  __shared__ int pair_s[KM * 128];  // flag phase: (point << 16 | group) pairs
  __shared__ T ext_s;
  __shared__ T red_s[2][NW][3];
  // CL > 1: incoming top lists [parity][rank * KM + e], one mbarrier per parity
  __shared__ __align__(16) uint32_t xrec_s[CL > 1 ? 2 : 1][CL > 1 ? CL * KM * R::W : 1];
  __shared__ __align__(8) uint64_t xbar_s[2];

  // ---- bucket table ------------------------------------------------------------
  T lo[3] = {A::pinf(), A::pinf(), A::pinf()}, hi[3] = {A::ninf(), A::ninf(), A::ninf()};
  for (int q = tid; q < nb; q += NT) {
#pragma unroll
    for (int c = 0; c < 6; ++c) box[q * 6 + c] = BB[((int64_t)q * CL + rank) * 6 + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T bl = (T)box[q * 6 + c], bh = (T)box[q * 6 + 3 + c];
      lo[c] = bl < lo[c] ? bl : lo[c];
      hi[c] = bh > hi[c] ? bh : hi[c];
    }
    kv[q] = k2[q] = A::bits(A::pinf());
    if constexpr (SHADOW) kv32[q] = __int_as_float(0x7f800000);
    ki[q] = kNoIdx;
    kx[q * 3 + 0] = kx[q * 3 + 1] = kx[q * 3 + 2] = S(0);
    pmask[q] = 0u;
  }
  // cloud extent (rounds with a search radius close to it test every bucket)
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
    rcount_s = 0;
    npair_s = 0;
    ndirty_s = 0;
    ngv_s = 0;
  }
  if (tid < kMaxGW) dmask_s[tid] = 0u;
  __syncthreads();
  if (tid == 0) {
    T e = T(0);
    for (int c = 0; c < 3; ++c) {
      T a = A::pinf(), z = A::ninf();
      for (int w = 0; w < NW; ++w) {
        a = red_s[0][w][c] < a ? red_s[0][w][c] : a;
        z = red_s[1][w][c] > z ? red_s[1][w][c] : z;
      }
      e = z - a > e ? z - a : e;
    }
    ext_s = e;
  }
  // group boxes
  for (int g = tid; g < ng; g += NT) {
    S a[3] = {(S)A::pinf(), (S)A::pinf(), (S)A::pinf()},
      z[3] = {(S)A::ninf(), (S)A::ninf(), (S)A::ninf()};
    const int q1 = (g + 1) * kGS < nb ? (g + 1) * kGS : nb;
    for (int q = g * kGS; q < q1; ++q)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a[c] = box[q * 6 + c] < a[c] ? box[q * 6 + c] : a[c];
        z[c] = box[q * 6 + 3 + c] > z[c] ? box[q * 6 + 3 + c] : z[c];
      }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      gbox[g * 6 + c] = a[c];
      gbox[g * 6 + 3 + c] = z[c];
    }
    gmax[g] = A::bits(A::pinf());
    if constexpr (SHADOW) gmax32[g] = __int_as_float(0x7f800000);
  }
  __syncthreads();
  const T full_r2 = (T)(kFullFrac * kFullFrac * (double)ext_s * (double)ext_s);

  // ---- seed (fps_core.py:124-130) -----------------------------------------------
  const int seed = (int)prm.seed_pos[b];
  int64_t* order = prm.order + (int64_t)b * prm.out_stride;
  T* sel = static_cast<T*>(prm.sel_d2) + (int64_t)b * prm.out_stride;
  if (tid == 0) {
    const S* X0 = static_cast<const S*>(prm.xyz) + (int64_t)b * prm.cloud_stride * 3;
    const int64_t src = prm.index_map ? prm.index_map[(int64_t)b * prm.map_stride + seed] : seed;
    sp_w[0][0][0] = (T)X0[3 * src + 0];
    sp_w[0][0][1] = (T)X0[3 * src + 1];
    sp_w[0][0][2] = (T)X0[3 * src + 2];
    if constexpr (SHADOW)
      for (int c = 0; c < 3; ++c) sp32_w[0][c] = (float)X0[3 * src + c];
    si_w[0][0] = (uint32_t)seed;
    sq_w[0][0] = -1;
  }
  if (tid == 0 && rank == 0) {
    order[0] = seed;
    sel[0] = A::pinf();
  }

  if constexpr (CL > 1) {
    if (tid == 0) {
      mbar_init(smem_u32(&xbar_s[0]), 1);
      mbar_init(smem_u32(&xbar_s[1]), 1);
      fence_mbar_init_cluster();
    }
    cluster_sync_all();  // peers' mbarriers initialised before any push
  }
  int J = 1;                        // points accepted by the last round
  bits_t rmax = A::bits(A::pinf());  // upper bound of every key (R^2 of the cube)
  __syncthreads();
  const int iters = (int)prm.iters;
  long long* trace =
      (prm.trace && b == 0 && rank == 0 && lane == 0) ? prm.trace + (int64_t)warp * prm.trace_iters * kTraceW : nullptr;

  auto flag = [&](int q, int t) {  // OR point t into bucket q's mask, list it once
    const uint32_t old = atomicOr(&pmask[q], 1u << t);
    if (old == 0u) {
      const int e = atomicAdd(&rcount_s, 1);
      FFPS_CHECK(e < nb);
      rlist[e] = q;
    }
  };
  // does point t reach bucket q's key?  (K1b's exact bound test; SHADOW: its
  // binary32 lower bound against the key rounded up, a superset of hits)
  auto reaches = [&](int q, int t) -> bool {
    if constexpr (SHADOW)
      return !(box_lb_rd(sp32_w[t][0], sp32_w[t][1], sp32_w[t][2], box + (size_t)q * 6) >=
               kv32[q]);
    else
      return !(box_lb(sp_w[0][t][0], sp_w[0][t][1], sp_w[0][t][2], box + (size_t)q * 6) >=
               A::from_bits(kv[q]));
  };
  auto test = [&](int q, int t) {
    if (reaches(q, t)) flag(q, t);
  };
  // warp-converged variant for two (point, bucket) tests per lane (two pairs of
  // the flag phase in flight): every lane calls it; new buckets are appended
  // with one shared-memory atomic per warp.  (An L2 -> L1 prefetch of the new
  // buckets' points here was measured 3% slower and dropped.)
  auto test_warp2 = [&](bool v0, int q0, int t0, bool v1, int q1, int t1) {
    const bool h0 = v0 && reaches(q0, t0);
    const bool h1 = v1 && reaches(q1, t1);
    const bool n0 = h0 && atomicOr(&pmask[q0], 1u << t0) == 0u;
    const bool n1 = h1 && atomicOr(&pmask[q1], 1u << t1) == 0u;
    const unsigned m0 = __ballot_sync(0xffffffffu, n0), m1 = __ballot_sync(0xffffffffu, n1);
    if (m0 | m1) {
      const int c0 = __popc(m0);
      int base = 0;
      if (lane == 0) base = atomicAdd(&rcount_s, c0 + __popc(m1));
      base = __shfl_sync(0xffffffffu, base, 0);
      const unsigned below = (1u << lane) - 1u;
      FFPS_CHECK(base + c0 + __popc(m1) <= nb);
      if (n0) rlist[base + __popc(m0 & below)] = q0;
      if (n1) rlist[base + c0 + __popc(m1 & below)] = q1;
    }
  };

  // bound of bucket q's next key once its key point c is selected: every
  // other point x keeps min(dist(x), d2(x, c)) <= min(second best, the
  // largest rounded d2 from c to the bucket's box) — per axis
  // max(|RN(lo - c)|, |RN(hi - c)|) bounds |RN(x - c)| (RN is monotone), and
  // the rounded squares and sums are monotone; condition (b) of the chain test
  // uses this instead of the second best alone
  auto tail_bound = [&](int q) -> bits_t {
    const S* bq = box + (size_t)q * 6;
    T g[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const T v = (T)kx[q * 3 + c];
      T lo, hi;
      if constexpr (sizeof(T) == 4) {
        lo = fabsf(__fsub_rn(bq[c], v));
        hi = fabsf(__fsub_rn(bq[3 + c], v));
      } else {
        lo = fabs(__dsub_rn((double)bq[c], v));
        hi = fabs(__dsub_rn((double)bq[3 + c], v));
      }
      g[c] = lo > hi ? lo : hi;
    }
    T fc;
    if constexpr (sizeof(T) == 4)
      fc = __fadd_rn(__fadd_rn(__fmul_rn(g[0], g[0]), __fmul_rn(g[1], g[1])), __fmul_rn(g[2], g[2]));
    else
      fc = __dadd_rn(__dadd_rn(__dmul_rn(g[0], g[0]), __dmul_rn(g[1], g[1])), __dmul_rn(g[2], g[2]));
    const bits_t fb = A::bits(fc);
    return k2[q] < fb ? k2[q] : fb;
  };

  int k = 1;
  // counters (prm.stats): rounds, loop cycles on rank 0, re-evaluated buckets
  const long long loop_t0 = clock64();
  long long nflag = 0;
  int ngeneral = 0;  // rounds whose ranking took the general path (warp 0)
  int round = 0;
  for (; k < iters; ++round) {
    long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    long long td[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // warp 0: sub-steps of phases R, D
    int ntest_w = 0;  // traced: hit groups of this warp
    int ncand_w = 0;  // traced: candidates of this warp
    if (trace) t0 = clock64();
    if constexpr (CL > 1)
      if (tid == 0)
        mbar_arrive_expect_tx(smem_u32(&xbar_s[round & 1]), CL * KM * R::W * 4);
    // A. flag ---------------------------------------------------------------------
    const T r2 = A::from_bits(rmax);
    // search radius: every key is <= R^2 (padded for the rounding of sqrt)
    const bool full = round == 0 || !(r2 < full_r2);
    if (full) {  // every bucket against every point
      for (int q = tid; q < nb; q += NT) {
        if (round == 0) {
          flag(q, 0);
          continue;
        }
        for (int t = 0; t < J; ++t) test(q, t);
      }
      if (round > 0 && warp == 0 && lane < J && sq_w[0][lane] >= 0 &&
          sq_w[0][lane] % CL == rank)
        flag(sq_w[0][lane] / CL, lane);  // the point -> -inf
    } else {
      // A1. wpp warps per selected point test the group boxes against the group
      //     max keys (a group with box_d2 >= its max key holds no bucket the
      //     point can flag); hits become (point, group) pairs
      // (J > 16: one warp per point, warp w takes points w, w + 16)
      const int wpp = J <= kWppJ ? c_wpp.wpp[J] : 1;  // warps per point (NW = 16)
#pragma unroll 1
      for (int tw = warp; tw < (J <= kWppJ ? J * wpp : J); tw += NW) {
        const int t = J <= kWppJ ? c_wpp.t[J][tw] : tw, sub = J <= kWppJ ? c_wpp.s[J][tw] : 0;
        for (int g0 = sub * 32; g0 < ng; g0 += wpp * 32) {
          const int g = g0 + lane;
          bool hit;
          if constexpr (SHADOW)
            hit = g < ng && !(box_lb_rd(sp32_w[t][0], sp32_w[t][1], sp32_w[t][2],
                                        gbox + (size_t)g * 6) >= gmax32[g]);
          else
            hit = g < ng && !(box_lb(sp_w[0][t][0], sp_w[0][t][1], sp_w[0][t][2],
                                     gbox + (size_t)g * 6) >= A::from_bits(gmax[g]));
          const unsigned m = __ballot_sync(0xffffffffu, hit);
          ntest_w += __popc(m);
          if (m) {
            int base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(&npair_s, __popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            FFPS_CHECK(base + __popc(m) <= KM * 128);
            if (hit) pair_s[base + __popc(m & ((1u << lane) - 1u))] = (t << 16) | g;
          }
        }
        if (lane == 0 && sub == 0 && sq_w[0][t] >= 0 && sq_w[0][t] % CL == rank)
          flag(sq_w[0][t] / CL, t);  // the point -> -inf
      }
      __syncthreads();  // pair list complete
      // A2. all warps: the kGS buckets of every pair (one per lane)
      const int np = npair_s;
#ifdef FFPS_GRID_ONEPAIR
      for (int e = warp; e < np; e += NW) {
        const bool two = false;
#else
      for (int e = warp; e < np; e += 2 * NW) {
        const bool two = e + NW < np;
#endif
        const int pr0 = pair_s[e], pr1 = two ? pair_s[e + NW] : pr0;
        const int q0 = (pr0 & 0xffff) * kGS + lane, q1 = (pr1 & 0xffff) * kGS + lane;
        test_warp2(q0 < nb, q0 < nb ? q0 : 0, pr0 >> 16, two && q1 < nb, q1 < nb ? q1 : 0,
                   pr1 >> 16);
      }
    }
    if (trace) t1 = clock64();
    __syncthreads();  // flags and round list complete
    // B. re-evaluate the round list --------------------------------------------------
    const int nr = rcount_s;
    nflag += nr;
    auto batch = [&](auto chn, int e0) {  // CH buckets e0, e0 + NW, ... in flight
      constexpr int CH = decltype(chn)::value;
      int qc[CH];
      uint32_t pm[CH];
      S xs[CH][PPL], ys[CH][PPL], zs[CH][PPL];
      T ds[CH][PPL], d0[CH][PPL];
      uint32_t os[CH][PPL];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        FFPS_CHECK(e0 + c * NW < nr);
        qc[c] = rlist[e0 + c * NW];
        pm[c] = pmask[qc[c]];
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          const int64_t s = ((int64_t)qc[c] * CL + rank) * BS + u * 32 + lane;
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
          const T px = sp_w[0][t][0], py = sp_w[0][t][1], pz = sp_w[0][t][2];
          const uint32_t pw = si_w[0][t];
#pragma unroll
          for (int u = 0; u < PPL; ++u) {
            T nd = A::vmin(ds[c][u], A::d2((T)xs[c][u], (T)ys[c][u], (T)zs[c][u], px, py, pz));  // :93
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
        S x1 = S(0), y1 = S(0), z1 = S(0);
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          if (A::bits(ds[c][u]) != A::bits(d0[c][u]))
            D[((int64_t)q * CL + rank) * BS + u * 32 + lane] = ds[c][u];
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
          if constexpr (SHADOW) kv32[q] = __double2float_ru(A::from_bits(b1));
          ki[q] = i1;
          k2[q] = w2;
          kx[q * 3 + 0] = x1;
          kx[q * 3 + 1] = y1;
          kx[q * 3 + 2] = z1;
          pmask[q] = 0u;
          atomicOr(&dmask_s[(q / kGS) >> 5], 1u << ((q / kGS) & 31));
        }
      }
    };
    {
      // all of a warp's buckets of the round in one batch when they fit
#ifndef FFPS_GRID_CH1
#define FFPS_GRID_CH1 4
#endif
#ifndef FFPS_GRID_CH2
#define FFPS_GRID_CH2 2
#endif
      constexpr int CH = PPL <= 1 ? FFPS_GRID_CH1 : (PPL == 2 ? FFPS_GRID_CH2 : 1);  // buckets in flight
      for (int e = warp; e < nr; e += CH * NW) {
        const int nv = (nr - e + NW - 1) / NW;
        if (nv >= CH) batch(std::integral_constant<int, CH>{}, e);
        else if (CH >= 3 && nv == 3) batch(std::integral_constant<int, (CH >= 3 ? 3 : 1)>{}, e);
        else if (CH >= 2 && nv == 2) batch(std::integral_constant<int, (CH >= 2 ? 2 : 1)>{}, e);
        else batch(std::integral_constant<int, 1>{}, e);
      }
    }
    if (trace) t2 = clock64();
    __syncthreads();  // keys final for this round
    if (tid == 0) {
      rcount_s = 0;
      npair_s = 0;
      ngv_s = 0;
    }
    // C. group statistics (each warp refreshes a slice of whole groups, one
    //    bucket per lane): top-2 keys by (value desc, position asc) + third value
    //    (only the groups with a re-evaluated bucket changed: the dirty list)
    if (tid < KM * NCG) compv_s[tid] = A::kmin;  // R1 fills the ranks it finds
    if (tid < KM) topg_s[tid] = -1;              // ranks of empty groups stay -1
    if (tid < ng) grank_s[tid] = -1;             // R1 sets the top groups' ranks
    for (int wd = 0, base = 0; wd < ((ng + 31) >> 5); ++wd) {
      const unsigned mword = dmask_s[wd];
      const int cw = __popc(mword);
      // lane l holds bit l of the word and its rank among the set bits
      const bool bit = (mword >> lane) & 1u;
      const int brank = __popc(mword & ((1u << lane) - 1u));
      for (int j = ((warp - base) % NW + NW) % NW; j < cw; j += NW) {
        const int g = wd * 32 + __ffs(__ballot_sync(0xffffffffu, bit && brank == j)) - 1;
        const int q = g * kGS + lane;
        const bool in = q < nb;
        bits_t v = in ? kv[q] : A::kmin;
        const uint32_t p = in ? ki[q] : kNoIdx;
        unsigned taken = 0u;
#pragma unroll
        for (int k = 0; k < NCG; ++k) {  // k-th best by (value desc, position asc)
          const bits_t mk = A::warp_max(v);
          const uint32_t pk = __reduce_min_sync(0xffffffffu, v == mk ? p : kNoIdx);
          const unsigned wk = __ballot_sync(0xffffffffu, v == mk && p == pk) & ~taken;
          taken |= wk;
          if (wk & (1u << lane)) v = A::kmin;
          if (lane == 0) {
            if (k == 0) {
              gmax[g] = mk;
              if constexpr (SHADOW) gmax32[g] = __double2float_ru(A::from_bits(mk));
            }
            cand_v[NCG * g + k] = mk;
            cand_p[NCG * g + k] = pk;
            cand_q[NCG * g + k] = wk ? g * kGS + __ffs(wk) - 1 : 0;
          }
        }
        const bits_t mn = A::warp_max(v);
        if (lane == 0) gnext[g] = mn;
      }
      base += cw;
    }
    if (trace) t3 = clock64();
    __syncthreads();  // group statistics final
    if (tid < kMaxGW) dmask_s[tid] = 0u;
    if (trace) td[0] = clock64();
    // R1. all threads: rank of every group by its max key (value desc, position
    //     asc), 16 threads per group; the KM best groups -> topg_s.  Every
    //     top-KM key lies in those groups (a key elsewhere has KM group maxima
    //     above it), and its rank among their candidates is its true rank.
    {
      const int gb = tid >> 4, part = tid & 15;
      for (int g0 = 0; g0 < ng; g0 += NT / 16) {  // uniform trip count
        const int g = g0 + gb;
        const bits_t v = g < ng ? cand_v[NCG * g] : A::kmin;
        const uint32_t p = g < ng ? cand_p[NCG * g] : kNoIdx;
        int cnt = 0;
        if (v != A::kmin)
          for (int e = part; e < ng; e += 16) {
            const bits_t ve = cand_v[NCG * e];
            cnt += (ve > v || (ve == v && cand_p[NCG * e] < p)) ? 1 : 0;
          }
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (part == 0 && v != A::kmin) {
          if (cnt < KM) {
            FFPS_CHECK(g < ng && cnt >= 0);
            topg_s[cnt] = g;
            grank_s[g] = (int16_t)cnt;
#pragma unroll
            for (int k = 0; k < NCG; ++k) {
              compv_s[cnt * NCG + k] = cand_v[NCG * g + k];
              compp_s[cnt * NCG + k] = cand_p[NCG * g + k];
              compq_s[cnt * NCG + k] = cand_q[NCG * g + k];
            }
          }
        }
      }
    }
    __syncthreads();  // group ranks final
    // R2. all threads: ranks among the candidates of the top groups (<= KM * NCG
    //     <= 64, compacted by R1), 8 threads per candidate
    const int ngt = __popc(__ballot_sync(0xffffffffu, lane < KM && topg_s[lane] >= 0));
    const int nrc = ngt * NCG;
    {
      constexpr int NC = KM * NCG;
      constexpr int TPC = NT / NC >= 8 ? 8 : NT / NC;  // threads per candidate
      static_assert(TPC >= 1 && NC % TPC == 0, "R2 layout");
      const int c = tid / TPC, part = tid % TPC;
      if (c < NC) {  // whole warps (NC is a multiple of 4)
        const bits_t v = compv_s[c];
        const uint32_t p = compp_s[c];
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < NC / TPC; ++i) {  // empty entries (kmin) never rank above
          const bits_t ve = compv_s[part + TPC * i];
          const uint32_t pe = compp_s[part + TPC * i];
          cnt += (ve > v || (ve == v && pe < p)) ? 1 : 0;
        }
#pragma unroll
        for (int o = 1; o < TPC; o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (part == 0) rr_s[c] = v != A::kmin ? cnt : 0x7fffffff;
        if (part == 0 && v != A::kmin && cnt < KM) {
          FFPS_CHECK(compq_s[c] >= 0 && compq_s[c] < nb);
          top_s[cnt] = (int16_t)compq_s[c];
          topv_s[cnt] = v;
        }
      }
    }
    if (trace) td[1] = clock64();
    __syncthreads();  // candidate ranks final
    if (trace) td[2] = clock64();
    // D. warp 0 alone: this rank's top-KM keys (table rows, rank order).
    //    tau2 = the KM-th candidate: a group whose third key reaches it may
    //    hold a top-KM key that is not a candidate -> the general path: every
    //    key >= tau2 of the groups with max >= tau2 (KM keys are >= tau2),
    //    more than 32 of them (massive ties) -> the exact maximum alone, marked
    //    truncated.
    if (warp == 0) {
    int nl = 0;
    bool trunc = false;
    {
      const unsigned below = (1u << lane) - 1u;
      // the ranked top-KM rows, tau2 = the KM-th candidate's value; a top group
      // whose (NCG+1)-th key reaches tau2 may hold a top-KM key that is not a
      // candidate -> the general path
      int nvalid = 0;
#pragma unroll
      for (int c0 = 0; c0 < KM * NCG; c0 += 32)
        nvalid += __popc(__ballot_sync(0xffffffffu, c0 + lane < nrc && rr_s[c0 + lane] != 0x7fffffff));
      const bits_t tau2 = nvalid >= KM ? topv_s[KM - 1] : A::kmin;
      const bits_t tn = lane < ngt ? gnext[topg_s[lane]] : A::kmin;
      const bool general = __any_sync(0xffffffffu, tn != A::kmin && tn >= tau2);
      int nct = nvalid;
      if (!general) {
        nl = nvalid < KM ? nvalid : KM;
        if (lane < nl) top_w[0][lane] = top_s[lane];
      } else {
        // every key >= tau2: (a) the candidates of the top groups whose
        // (NCG+1)-th key is below tau2 (all their keys >= tau2 are candidates),
        // (b) all keys >= tau2 of the top groups that overflow and of any other
        // group whose max reaches tau2 (exact ties with the KM-th candidate)
        nct = 0;
        const unsigned ovf = __ballot_sync(0xffffffffu, lane < ngt && tn != A::kmin && tn >= tau2);
#pragma unroll
        for (int c0 = 0; c0 < KM * NCG; c0 += 32) {
          const int c = c0 + lane;
          const bits_t v = c < nrc ? compv_s[c] : A::kmin;
          const bool take = c < nrc && !((ovf >> (c / NCG)) & 1u) && v != A::kmin && v >= tau2;
          const unsigned cm = __ballot_sync(0xffffffffu, take);
          const int slot = nct + __popc(cm & below);
          if (take && slot < 64) {
            cv_w[0][slot] = v;
            ci_w[0][slot] = compp_s[c];
            cq_w[0][slot] = (int16_t)compq_s[c];
          }
          nct += __popc(cm);
        }
#pragma unroll 1
        for (int j = 0; j < (ng + 31) / 32; ++j) {
          const int gj = j * 32 + lane;
          const bits_t gvj = gj < ng ? gmax[gj] : A::kmin;
          const int grk = gj < ng ? grank_s[gj] : -1;  // rank among the top groups, -1: none
          const bool scan = grk < 0 || ((ovf >> grk) & 1u);
          unsigned hm = __ballot_sync(0xffffffffu, gvj >= tau2 && gvj != A::kmin && scan);
          while (hm) {
            const int q = (j * 32 + __ffs(hm) - 1) * kGS + lane;
            hm &= hm - 1u;
            const bits_t v = q < nb ? kv[q] : A::kmin;
            const bool c = v >= tau2 && v != A::kmin;
            const unsigned cm = __ballot_sync(0xffffffffu, c);
            const int slot = nct + __popc(cm & below);
            if (c && slot < 64) {
              cv_w[0][slot] = v;
              ci_w[0][slot] = ki[q];
              cq_w[0][slot] = (int16_t)q;
            }
            nct += __popc(cm);
          }
        }
        __syncwarp();
        if (nct > 64) {
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
          const int qmax = __shfl_sync(0xffffffffu, bq, wl);
          if (lane == 0) top_w[0][0] = (int16_t)qmax;
          nl = 1;
          trunc = true;
        } else if (nct <= 32) {  // one entry per lane: ranks by shuffles
          const bool live = lane < nct;
          const bits_t v = live ? cv_w[0][lane] : A::kmin;
          const uint32_t i = live ? ci_w[0][lane] : kNoIdx;
          int r3 = 0;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const bits_t ve = A::shfl(v, e);
            const uint32_t ie = __shfl_sync(0xffffffffu, i, e);
            r3 += (e < nct && (ve > v || (ve == v && ie < i))) ? 1 : 0;
          }
          if (live && r3 < KM) top_w[0][r3] = cq_w[0][lane];
          nl = nct < KM ? nct : KM;
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {  // entries lane and lane + 32
            const int x = lane + 32 * h;
            const bool live = x < nct;
            const bits_t v = live ? cv_w[0][x] : A::kmin;
            const uint32_t i = live ? ci_w[0][x] : kNoIdx;
            int r3 = 0;
            for (int e = 0; e < nct; ++e) {
              const bits_t ve = cv_w[0][e];
              r3 += (ve > v || (ve == v && ci_w[0][e] < i)) ? 1 : 0;
            }
            if (live && r3 < KM) top_w[0][r3] = cq_w[0][x];
          }
          nl = nct < KM ? nct : KM;
        }
      }
      ncand_w = nct | (general ? 1 << 16 : 0);
      ngeneral += general ? 1 : 0;
      if (trace) td[3] = clock64();
    }
    __syncwarp();
    // candidates in global rank order: lane < nc holds the lane-th
    int nc;
    bits_t cv = A::kmin, c2 = A::kmin;
    T cx = T(0), cy = T(0), cz = T(0);
    uint32_t cpos = kNoIdx;
    int cq = -1;
    if constexpr (CL == 1) {
      nc = nl;
      if (lane < nc) {
        const int q = top_w[0][lane];
        cv = kv[q]; c2 = tail_bound(q); cpos = ki[q]; cq = q;
        cx = (T)kx[q * 3 + 0]; cy = (T)kx[q * 3 + 1]; cz = (T)kx[q * 3 + 2];
      }
    } else {
      const int par = round & 1;
      const uint32_t buf = smem_u32(&xrec_s[par][0]);
#pragma unroll
      for (int r = lane; r < CL * KM; r += 32) {  // push the local list to every rank
        const int peer = r / KM, e = r % KM;
        {
          const uint32_t dst = mapa(buf + (uint32_t)((rank * KM + e) * R::W * 4), (uint32_t)peer);
          const uint32_t bar = mapa(smem_u32(&xbar_s[par]), (uint32_t)peer);
          if (e < nl) {
            const int q = top_w[0][e];
            R::send(dst, bar, kv[q], tail_bound(q), ki[q], q * CL + rank, (T)kx[q * 3 + 0],
                    (T)kx[q * 3 + 1], (T)kx[q * 3 + 2], trunc ? 1u : 0u);
          } else {
            R::send(dst, bar, A::kmin, A::kmin, kNoIdx, -1, T(0), T(0), T(0), 0u);
          }
        }
      }
      if (trace) td[4] = clock64();
      mbar_wait(smem_u32(&xbar_s[par]), (uint32_t)((round >> 1) & 1));
      if (trace) td[5] = clock64();
      // merge the CL sorted lists (value desc, position asc) with bitonic merge
      // stages: lane l takes element e of list c = l / KM, odd lists reversed,
      // so every pair of lists is a bitonic sequence (CL = 4: the upper half
      // is reversed again before the final 2 * KM-wide merge)
      const uint32_t* rec = &xrec_s[par][0];
      int idx = -1;
      bits_t mv = A::kmin;
      uint32_t mp = kNoIdx;
      if constexpr (CL == 4 && KM == 16) {
        // four lists of 16 in two slots (lists 0-1 | 2-3, lane l: element
        // l % 16 of list l / 16 of its pair, odd lists reversed, so each slot
        // is a bitonic 32).  Only the best KM = 16 of the 64 are used: one
        // half-cleaner per slot (one shuffle: lanes 0-15 keep the better 16
        // of slot a, lanes 16-31 those of slot b), four stages sorting lanes
        // 0-15 descending and 16-31 ascending, a half-cleaner across them and
        // four stages sorting the best 16 into lanes 0-15 (10 stages, not the
        // 16 of a full 64-merge)
        auto ld = [&](int list, int e, bits_t& v, uint32_t& p, int& ix) {
          ix = list * KM + ((list & 1) ? KM - 1 - e : e);
          v = R::v(rec + ix * R::W);
          p = R::pos(rec + ix * R::W);
        };
        const bool hi = (lane & 16) != 0;
        {
          bits_t va, vb;
          uint32_t pa, pb;
          int ia, ib;
          ld(lane / KM, lane % KM, va, pa, ia);
          ld(2 + lane / KM, lane % KM, vb, pb, ib);
          // lane l < 16 needs a[l ^ 16]; lane l >= 16 needs b[l ^ 16]
          const bits_t ov = A::shfl(hi ? va : vb, lane ^ 16);
          const uint32_t op = __shfl_sync(0xffffffffu, hi ? pa : pb, lane ^ 16);
          const int oi = __shfl_sync(0xffffffffu, hi ? ia : ib, lane ^ 16);
          mv = hi ? vb : va;
          mp = hi ? pb : pa;
          idx = hi ? ib : ia;
          if (ov > mv || (ov == mv && op < mp)) {
            mv = ov;
            mp = op;
            idx = oi;
          }
        }
        auto st_dir = [&](int j, bool up) {  // up: the better one to the higher lane
          const bits_t ov = __shfl_xor_sync(0xffffffffu, mv, j);
          const uint32_t op = __shfl_xor_sync(0xffffffffu, mp, j);
          const int oi = __shfl_xor_sync(0xffffffffu, idx, j);
          const bool other_better = ov > mv || (ov == mv && op < mp);
          const bool mine_better = mv > ov || (mv == ov && mp < op);
          if (((lane & j) == 0) != up ? other_better : mine_better) {
            mv = ov;
            mp = op;
            idx = oi;
          }
        };
#pragma unroll
        for (int j = 8; j > 0; j >>= 1) st_dir(j, hi);
        st_dir(16, false);
#pragma unroll
        for (int j = 8; j > 0; j >>= 1) st_dir(j, false);
      } else {
      if constexpr (CL == 2 && KM == 32) {
        // two lists of 32: lane l compares element l of list 0 with element
        // 31 - l of list 1 (half-cleaner); the better 32 form a bitonic sequence
        const int ia = lane, ib = KM + KM - 1 - lane;
        const bits_t va = R::v(rec + ia * R::W), vb = R::v(rec + ib * R::W);
        const uint32_t pa = R::pos(rec + ia * R::W), pb = R::pos(rec + ib * R::W);
        const bool a_better = va > vb || (va == vb && pa < pb);
        idx = a_better ? ia : ib;
        mv = a_better ? va : vb;
        mp = a_better ? pa : pb;
      } else if (lane < CL * KM) {
        const int c = lane / KM, e = lane % KM;
        idx = c * KM + ((c & 1) ? KM - 1 - e : e);
        mv = R::v(rec + idx * R::W);
        mp = R::pos(rec + idx * R::W);
      }
      auto stage = [&](int j) {
        const bits_t ov = __shfl_xor_sync(0xffffffffu, mv, j);
        const uint32_t op = __shfl_xor_sync(0xffffffffu, mp, j);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, j);
        const bool other_better = ov > mv || (ov == mv && op < mp);
        const bool mine_better = mv > ov || (mv == ov && mp < op);
        if ((lane & j) == 0 ? other_better : mine_better) {
          mv = ov;
          mp = op;
          idx = oi;
        }
      };
#pragma unroll
      for (int j = (KM < 32 ? KM : 16); j > 0; j >>= 1) stage(j);
      if constexpr (CL == 4) {
        // lanes 16..31 hold the second sorted 16-list: reverse it, merge 32
        const int src = lane < 2 * KM ? lane : 3 * 2 * KM - 1 - lane;
        mv = A::shfl(mv, src);
        mp = __shfl_sync(0xffffffffu, mp, src);
        idx = __shfl_sync(0xffffffffu, idx, src);
#pragma unroll
        for (int j = 2 * KM; j > 0; j >>= 1) stage(j);
      }
      }
      // lane r now holds the r-th record; a truncated list is exact only up to
      // its one record (its head)
      const bool valid = mv != A::kmin;
      const bool thead = valid && (idx % KM) == 0 && R::flag(rec + idx * R::W) != 0u;
      const unsigned th = __ballot_sync(0xffffffffu, thead);
      const int limit = th ? __ffs(th) : 32;
      const int nvalid = __popc(__ballot_sync(0xffffffffu, valid));
      nc = nvalid < KM ? nvalid : KM;
      nc = nc < limit ? nc : limit;
      if (lane < nc) {
        const uint32_t* r = rec + idx * R::W;
        cv = mv; c2 = R::v2(r); cpos = mp; cq = R::q(r);
        cx = R::c(r, 0); cy = R::c(r, 1); cz = R::c(r, 2);
      }
    }
    if (trace) td[6] = clock64();
    int acc;
    {
      // chain test (K1m): candidate j joins iff it is not closer than its own
      // key to any earlier accepted candidate and beats their buckets' second best
      const bool live = lane < nc;
      bool ok = live && A::from_bits(cv) >= T(0);
#ifdef FFPS_GRID_CHAIN_SHFL
#pragma unroll
      for (int bb = 0; bb < KM - 1; ++bb) {
        const T bx = __shfl_sync(0xffffffffu, cx, bb);
        const T by = __shfl_sync(0xffffffffu, cy, bb);
        const T bz = __shfl_sync(0xffffffffu, cz, bb);
        const bits_t b2 = A::shfl(c2, bb);
        const bool ca = !(A::d2(cx, cy, cz, bx, by, bz) < A::from_bits(cv));
        ok = ok & ((bb >= lane) | (ca & (cv > b2)));
      }
#else
      if (lane < KM) ch_s[lane] = ChainRec{cx, cy, cz, c2};
      __syncwarp();
#pragma unroll
      for (int bb = 0; bb < KM - 1; ++bb) {
        const ChainRec cb = ch_s[bb];
        // (a), (b); evaluated for every lane without branches (bitwise ops)
        const bool ca = !(A::d2(cx, cy, cz, cb.x, cb.y, cb.z) < A::from_bits(cv));
        ok = ok & ((bb >= lane) | (ca & (cv > cb.b2)));
      }
#endif
      const unsigned okm = __ballot_sync(0xffffffffu, ok || lane == 0);
      acc = __ffs(~okm) - 1;
      if (acc < 0 || acc > nc) acc = nc;
      if (acc < 1) acc = 1;
      if (acc > iters - k) acc = iters - k;
      if (lane < acc) {
        sp_w[0][lane][0] = cx;
        sp_w[0][lane][1] = cy;
        sp_w[0][lane][2] = cz;
        if constexpr (SHADOW) {
          sp32_w[lane][0] = (float)cx;  // float coordinates: exact
          sp32_w[lane][1] = (float)cy;
          sp32_w[lane][2] = (float)cz;
        }
        si_w[0][lane] = cpos;
        sq_w[0][lane] = cq;
        if (rank == 0) {
          order[k + lane] = cpos;  // fps_core.py:167-168
          sel[k + lane] = A::from_bits(cv);
        }
      }
      const bits_t r0 = A::shfl(cv, 0);
      if (trace) td[7] = clock64();
      if (lane == 0) {
        acc_s = acc;
        rmax_s = r0;
      }

    }
    }  // warp 0
    __syncthreads();  // accepted points of the round visible to every warp
    const int acc = acc_s;
    rmax = rmax_s;
    J = acc;
    if (trace && round < prm.trace_iters) {
      long long* rr = trace + (int64_t)round * kTraceW;
      rr[0] = t0; rr[1] = t1; rr[2] = t2; rr[3] = t3; rr[4] = clock64(); rr[5] = acc;
      rr[6] = nr | ((long long)ncand_w << 32); rr[7] = (long long)full | ((long long)ng << 1) | ((long long)ntest_w << 24);
      for (int i = 0; i < 8; ++i) rr[8 + i] = td[i];
    }
    k += acc;
  }

  if (prm.stats != nullptr && tid == 0) {
    unsigned long long* st = reinterpret_cast<unsigned long long*>(prm.stats) + (int64_t)b * 4;
    if (rank == 0) {
      st[0] = (unsigned long long)round;
      st[1] = (unsigned long long)(clock64() - loop_t0);
    }
    atomicAdd(st + 2, (unsigned long long)nflag);
    atomicAdd(st + 3, (unsigned long long)ngeneral);
  }
  if constexpr (CL > 1) cluster_sync_all();  // no rank leaves while peers may push into it
  // positions -> original indices for restricted runs (fps_cache.py:197)
  if (prm.index_map != nullptr && rank == 0) {
    __syncthreads();
    const int64_t* map = prm.index_map + (int64_t)b * prm.map_stride;
    for (int kk = tid; kk < iters; kk += NT) order[kk] = __ldg(map + order[kk]);
  }
}

// dtype code of an instance: 0 float, 1 double, 2 float coordinates with
// binary64 arithmetic (FFPS_F32_F64)
template <typename T, typename S, int PPL, int KM, int CL>
GridInst make_ginst() {
  GridInst k;
  k.dtype = sizeof(T) == 4 ? 0 : (sizeof(S) == 4 ? 2 : 1);
  k.nt = kBucketThreads;
  k.ppl = PPL;
  k.km = KM;
  k.cl = CL;
  k.fn = reinterpret_cast<const void*>(&fps_grid_kernel<T, S, kBucketThreads, PPL, KM, CL>);
  k.esz = sizeof(S);
  return k;
}

#define FFPS_GRID_PPL(T, S, KM, CL)                                                       \
  make_ginst<T, S, 1, KM, CL>(), make_ginst<T, S, 2, KM, CL>(), make_ginst<T, S, 4, KM, CL>(), \
      make_ginst<T, S, 8, KM, CL>()

}  // namespace ffps
