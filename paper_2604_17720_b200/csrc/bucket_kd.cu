// K0-kd — kd-tree bucketing of the point set of every cloud (default K0).
//
// Same output contract as the Morton K0 (bucket_build.cu): bucket-major SoA
// X, Y, Z, D, O [nb * BS] and boxes BB [nb][6]; padding slots (>= n) repeat
// the first point of the last bucket with D = -inf, O = -1.
//
// Buckets are the leaves of a kd-tree: a segment of m > BS points is split on
// the longest axis of its box so that the left child holds nl =
// ((m / BS + 1) / 2) * BS points (a whole number of buckets: every segment
// starts on a bucket boundary and only the rightmost leaf — the last bucket —
// can be partial).  The split value is located with a 1024-bin histogram of
// the segment along that axis; the boundary bin is divided by arrival order.
// A leaf's box is then as compact as 32 * PPL points allow, whatever the
// density: on LiDAR frames (1/r^2 density, scan rings) the Morton buckets of
// a fixed grid span up to ~7 m while kd leaves stay near the local spacing,
// and the greedy kernels flag ~4x (uniform ~2x) fewer buckets per selected
// point (SIMULATED and measured, K0).
//
// One CTA (1024 threads) per cloud; points ping-pong between the output
// arrays (X, Y, Z, O) and the scratch arrays (TX, TY, TZ, TO):
//   CTA phase  level-synchronous while there are < 32 segments: histogram
//              pass, per-segment scan (one warp each), partition pass with
//              warp-aggregated shared-memory counters; children boxes are
//              accumulated during the partition (no separate box pass);
//   warp phase each warp splits its segment(s) depth-first down to the
//              leaves with an explicit stack, counters in registers.
// Leaves that end in the scratch arrays are copied back.  Like the Morton
// build, the slot order inside a bucket depends on arrival order; the greedy
// kernels break ties by position O, never by slot, so results are unchanged.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ffps_internal.h"
#include "ptx.cuh"

namespace ffps {

namespace {

constexpr int kThreads = 1024;
constexpr int kNW = kThreads / 32;
constexpr int kBins1 = 256;    // CTA phase: bins per segment histogram
constexpr int kBinsL = 256;    // leaf kernel: bins per warp histogram
constexpr int kMaxSeg = 128;   // CTA phase stops at this many segments
constexpr int kStack = 24;
constexpr int kU = 4;          // CTA phase: points per thread in flight     // per-warp DFS stack (depth <= log2(n / BS) + 1)

// order-preserving integer image of a float / double (for shared atomics)
template <typename T>
struct Ord;
template <>
struct Ord<float> {
  using I = int;
  __device__ static I enc(float f) {
    const int b = __float_as_int(f);
    return b >= 0 ? b : b ^ 0x7fffffff;
  }
  __device__ static float dec(I i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }
  static constexpr I kMax = 0x7fffffff;
  static constexpr I kMin = (int)0x80000000;
};
template <>
struct Ord<double> {
  using I = long long;
  __device__ static I enc(double f) {
    const long long b = __double_as_longlong(f);
    return b >= 0 ? b : b ^ 0x7fffffffffffffffLL;
  }
  __device__ static double dec(I i) {
    return __longlong_as_double(i >= 0 ? i : i ^ 0x7fffffffffffffffLL);
  }
  static constexpr I kMax = 0x7fffffffffffffffLL;
  static constexpr I kMin = (long long)0x8000000000000000ULL;
};

template <typename T>
__device__ __forceinline__ T wmin(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T wmax(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}
// box reductions: one REDUX on the order-preserving integer image for float
// (five shuffles otherwise; -0 orders below +0, which the bounds tolerate:
// they compare equal in every use)
template <typename T>
__device__ __forceinline__ T bmin(T v) {
  if constexpr (sizeof(T) == 4)
    return Ord<T>::dec(__reduce_min_sync(0xffffffffu, Ord<T>::enc(v)));
  else
    return wmin(v);
}
template <typename T>
__device__ __forceinline__ T bmax(T v) {
  if constexpr (sizeof(T) == 4)
    return Ord<T>::dec(__reduce_max_sync(0xffffffffu, Ord<T>::enc(v)));
  else
    return wmax(v);
}

template <int NB, typename T>
__device__ __forceinline__ int bin_of(T v, T lo, T inv) {
  const int c = (int)((v - lo) * inv);
  return c < 0 ? 0 : (c >= NB ? NB - 1 : c);
}

// split of a segment: nl points (a multiple of bs) to the left child
__device__ __forceinline__ int left_size(int m, int bs) { return ((m / bs + 1) / 2) * bs; }

// histogram layout (NB bins, BPL = NB / 32 per lane): bin b lives at word
// haddr(b) = (b % BPL) * 32 + b / BPL, so the BPL bins a lane owns in
// find_split ([BPL * lane, BPL * lane + BPL)) are read by the warp without
// bank conflicts (word j * 32 + lane)
template <int NB>
__device__ __forceinline__ int haddr(int b) {
  constexpr int BPL = NB / 32;
  return (b % BPL) * 32 + b / BPL;
}

// warp: locate the boundary bin of rank nl in an NB-bin histogram h; returns
// bin, count before it and the bin's own count (uniform across the warp)
template <int NB>
__device__ __forceinline__ void find_split(const uint32_t* h, int nl, int lane, int& bstar,
                                           int& before, int& mid) {
  constexpr int BPL = NB / 32;
  static_assert(BPL >= 1 && BPL <= 32, "32 to 1024 bins");
  uint32_t loc = 0;
#pragma unroll 8
  for (int j = 0; j < BPL; ++j) loc += h[j * 32 + lane];
  uint32_t incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  const unsigned hit = __ballot_sync(0xffffffffu, incl >= (uint32_t)nl);
  const int L = __ffs(hit) - 1;  // nl <= m - 1 < total, so some lane hits
  // lane j < BPL takes bin BPL * L + j: scan those counts across the warp
  const uint32_t run0 = __shfl_sync(0xffffffffu, incl - loc, L);
  const uint32_t v = lane < BPL ? h[lane * 32 + L] : 0u;
  uint32_t iv = v;
#pragma unroll
  for (int o = 1; o < BPL; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, iv, o);
    if (lane >= o) iv += u;
  }
  const int J = __ffs(__ballot_sync(0xffffffffu, lane < BPL && run0 + iv >= (uint32_t)nl)) - 1;
  bstar = BPL * L + J;
  before = (int)(run0 + __shfl_sync(0xffffffffu, iv - v, J));
  mid = (int)__shfl_sync(0xffffffffu, v, J);
}

// shared memory of one warp of the leaf kernel: histogram, DFS stack
// (start, size, parity, box) and, when staged, two SoA buffers of cap points
__host__ __device__ constexpr size_t kd_leaves_warp_bytes(int cap, int esz) {
  return ((size_t)kBinsL * 4 + (size_t)kStack * 3 * 4 + (kStack & 1) * 4 + (size_t)kStack * 6 * esz +
          16 /* staging mbarrier */ + (size_t)2 * cap * (3 * esz + 4) + 15) / 16 * 16;
}

template <typename T>
struct Bufs {
  T *x, *y, *z;
  int32_t* o;
};

}  // namespace

// CL = CTAs per cloud (thread-block cluster of 1 or 2): the points of every
// pass are dealt over CL * kThreads threads; histograms and children boxes are
// partial per CTA and summed through DSMEM; rank 1 places its points after
// rank 0's in every category (rank 0's counts come from its partial
// histogram), so the partition needs no remote atomics; both ranks keep
// identical segment state.
template <typename T, int CL>
__global__ void __launch_bounds__(kThreads, 1) bucket_kd_kernel(const BucketBuildParams p,
                                                                int32_t* seg_hdr, int32_t* seg_sm,
                                                                T* seg_box) {
  using O = Ord<T>;
  using I = typename O::I;
  extern __shared__ __align__(16) uint32_t hist[];  // [kMaxSeg][kBins] / [kNW][kBins], stack boxes
  __shared__ int s_start[kMaxSeg], s_m[kMaxSeg], s_nl[kMaxSeg], s_ax[kMaxSeg];
  __shared__ int s_b[kMaxSeg], s_lt[kMaxSeg], s_take[kMaxSeg], s_mid[kMaxSeg];
  __shared__ int s_cl[kMaxSeg], s_cm[kMaxSeg], s_cr[kMaxSeg];
  __shared__ T s_lo[kMaxSeg], s_inv[kMaxSeg];
  __shared__ I s_box[kMaxSeg][6];       // boxes of the current segments
  __shared__ I s_cbox[2 * kMaxSeg][6];  // boxes of their children
  __shared__ int s_S;
  __shared__ int n_start[kMaxSeg], n_m[kMaxSeg], n_from[kMaxSeg], s_nidx[kMaxSeg];

  static_assert(CL == 1 || CL == 2, "1 or 2 CTAs per cloud");
  constexpr int GT = CL * kThreads;  // threads per cloud
  const int rank = CL > 1 ? (int)cluster_ctarank() : 0;
  const int b = (int)blockIdx.x / CL, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gtid = rank * kThreads + tid;
  const uint32_t peer = (uint32_t)(rank ^ 1);
  auto ld_peer = [&](const I* local) -> I {  // the peer rank's copy of a shared word
    const uint32_t a = mapa(smem_u32(local), peer);
    if constexpr (sizeof(I) == 4) return (I)ld_cluster_u32(a);
    else return (I)ld_cluster_u64(a);
  };
  auto sync_all = [&]() {
    if constexpr (CL > 1) cluster_sync_all();
    else __syncthreads();
  };
  const int n = (int)p.n;
  const int bs = (int)p.bs;
  const T* X0 = static_cast<const T*>(p.xyz) + (int64_t)b * p.cloud_stride * 3;
  const int64_t* map = p.index_map ? p.index_map + (int64_t)b * p.map_stride : nullptr;
  const int64_t base = (int64_t)b * p.nslots;
  const Bufs<T> out{static_cast<T*>(p.X) + base, static_cast<T*>(p.Y) + base,
                   static_cast<T*>(p.Z) + base, p.O + base};
  const Bufs<T> tmp{static_cast<T*>(p.TX) + base, static_cast<T*>(p.TY) + base,
                    static_cast<T*>(p.TZ) + base, p.TO + base};
  auto buf = [&](int pr) { return pr ? tmp : out; };
  T* D = static_cast<T*>(p.D) + base;
  T* BB = static_cast<T*>(p.BB) + (int64_t)b * p.nbuckets * 6;
  const T pinf = (T)INFINITY;

  // 0. gather the run's points into buf[0] (position order) + cloud box
  if (tid < 6) s_box[0][tid] = tid < 3 ? O::kMax : O::kMin;
  __syncthreads();
  {
    T a[3] = {pinf, pinf, pinf}, z[3] = {-pinf, -pinf, -pinf};
    for (int i0 = 0; i0 < n; i0 += GT * kU) {  // kU points per thread in flight
      T v[kU][3];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * GT + gtid;
        const int64_t s = i < n ? (map ? __ldg(map + i) : i) : 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) v[u][c] = i < n ? X0[3 * s + c] : T(0);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * GT + gtid;
        if (i < n) {
          out.x[i] = v[u][0];
          out.y[i] = v[u][1];
          out.z[i] = v[u][2];
          out.o[i] = i;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const bool in = i0 + u * GT + gtid < n;
        a[c] = in && v[u][c] < a[c] ? v[u][c] : a[c];
        z[c] = in && v[u][c] > z[c] ? v[u][c] : z[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      a[c] = bmin(a[c]);
      z[c] = bmax(z[c]);
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        atomicMin(&s_box[0][c], O::enc(a[c]));
        atomicMax(&s_box[0][3 + c], O::enc(z[c]));
      }
    }
  }
  if constexpr (CL > 1) {  // cloud box = both partial boxes
    sync_all();
    I pv = 0;
    if (tid < 6) pv = ld_peer(&s_box[0][tid]);
    sync_all();
    if (tid < 6) s_box[0][tid] = tid < 3 ? (pv < s_box[0][tid] ? pv : s_box[0][tid])
                                         : (pv > s_box[0][tid] ? pv : s_box[0][tid]);
  }
  if (tid == 0) {
    s_S = 1;
    s_start[0] = 0;
    s_m[0] = n;
  }
  __syncthreads();

  // 1. CTA phase: level-synchronous splits while there are few segments
  int par = 0;
  for (;;) {
    const int S = s_S;
    bool any = false;
    for (int s = 0; s < S; ++s) any |= s_m[s] > bs;
    if (!any || 2 * S > kMaxSeg) break;
    const Bufs<T> src = buf(par), dst = buf(par ^ 1);
    // per-segment split parameters; clear histograms and counters
    if (tid < S) {
      const int s = tid;
      T ext[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) ext[c] = O::dec(s_box[s][3 + c]) - O::dec(s_box[s][c]);
      const int ax = ext[0] >= ext[1] ? (ext[0] >= ext[2] ? 0 : 2) : (ext[1] >= ext[2] ? 1 : 2);
      s_ax[s] = ax;
      s_lo[s] = O::dec(s_box[s][ax]);
      s_inv[s] = ext[ax] > (T)0 ? (T)kBins1 / ext[ax] : (T)0;
      s_nl[s] = s_m[s] > bs ? left_size(s_m[s], bs) : s_m[s];
      s_cl[s] = s_cm[s] = s_cr[s] = 0;
    }
    if (tid < 2 * S * 6) {
      const int c = tid % 6;
      s_cbox[tid / 6][c] = c < 3 ? O::kMax : O::kMin;
    }
    for (int i = tid; i < S * kBins1; i += kThreads) hist[i] = 0u;
    __syncthreads();
    // Warp groups: G segments at a time, one per group of kNW / G warps per
    // rank (G = the largest power of two <= min(S, 8)); group wg takes
    // segments wg, wg + G, ...  Deep levels have many small segments, which
    // the whole CTA would walk one by one with most lanes idle.  Both passes
    // use the same point -> thread mapping (gtid_g), so each rank's partial
    // histogram counts exactly the points that rank places.
    const int G = S >= 8 ? 8 : (S >= 4 ? 4 : (S >= 2 ? 2 : 1));
    const int wg = warp % G;
    const int GTg = GT / G;
    const int gtid_g = ((rank * kNW + warp) / G) * 32 + lane;
    // histogram pass (segment-major within each warp group)
    for (int s = wg; s < S; s += G) {
      if (s_m[s] <= bs) continue;
      const int st = s_start[s], m = s_m[s], ax = s_ax[s];
      const T lo = s_lo[s], inv = s_inv[s];
      const T* v = ax == 0 ? src.x : (ax == 1 ? src.y : src.z);
      uint32_t* h = hist + s * kBins1;
      for (int i0 = 0; i0 < m; i0 += GTg * kU) {  // kU loads in flight, then the atomics
        T w[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int i = i0 + u * GTg + gtid_g;
          w[u] = i < m ? v[st + i] : T(0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (i0 + u * GTg + gtid_g < m) atomicAdd(&h[haddr<kBins1>(bin_of<kBins1>(w[u], lo, inv))], 1u);
      }
    }
    // CL > 1: each rank keeps its partial histogram (first half of `hist`,
    // S <= kMaxSeg / 2 inside the loop) and builds the total in the second
    // half; the peer only ever reads the partials, which stay untouched until
    // the next level
    constexpr int kHalf = kMaxSeg / 2 * kBins1;
    if constexpr (CL > 1) {
      sync_all();
      for (int i = tid; i < S * kBins1; i += kThreads)
        hist[kHalf + i] = hist[i] + ld_cluster_u32(mapa(smem_u32(&hist[i]), peer));
    }
    __syncthreads();
    for (int sw = warp; sw < S; sw += kNW) {
      if (s_m[sw] <= bs) continue;
      int bstar, before, mid;
      const uint32_t* ht = hist + (CL > 1 ? kHalf : 0) + sw * kBins1;
      find_split<kBins1>(ht, s_nl[sw], lane, bstar, before, mid);
      if (lane == 0) {
        s_b[sw] = bstar;
        s_lt[sw] = before;
        s_mid[sw] = mid;
        s_take[sw] = s_nl[sw] - before;
      }
      if constexpr (CL > 1) {
        // rank 0's points of each category (its partial histogram: its own
        // half, or total - own for rank 1) -> rank 1's counters start there,
        // so both ranks place their points with local atomics only
        constexpr int BPL = kBins1 / 32;
        const uint32_t* hp = hist + sw * kBins1;
        uint32_t below = 0, at = 0, all = 0;
#pragma unroll
        for (int j = 0; j < BPL; ++j) {
          const int bin = BPL * lane + j, w = j * 32 + lane;
          const uint32_t a0 = rank == 0 ? hp[w] : ht[w] - hp[w];
          all += a0;
          below += bin < bstar ? a0 : 0u;
          at += bin == bstar ? a0 : 0u;
        }
        below = __reduce_add_sync(0xffffffffu, below);
        at = __reduce_add_sync(0xffffffffu, at);
        all = __reduce_add_sync(0xffffffffu, all);
        if (lane == 0 && rank == 1) {
          s_cl[sw] = (int)below;
          s_cm[sw] = (int)at;
          s_cr[sw] = (int)(all - below - at);
        }
      }
    }
    __syncthreads();
    // partition pass + children boxes (the same warp groups)
    for (int s = wg; s < S; s += G) {
      const int st = s_start[s], m = s_m[s];
      const bool split = m > bs;
      const int ax = s_ax[s], bstar = split ? s_b[s] : 0;
      const T lo = s_lo[s], inv = s_inv[s];
      const int nl = s_nl[s], lt = split ? s_lt[s] : 0, take = split ? s_take[s] : 0;
      const int midc = split ? s_mid[s] : 0;
      T a[2][3], z[2][3];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          a[k][c] = pinf;
          z[k][c] = -pinf;
        }
      for (int j0 = 0; j0 < m; j0 += GTg * kU) {  // warp-uniform trip count
       T vv[kU][3];
       int32_t oo[kU];
#pragma unroll
       for (int u = 0; u < kU; ++u) {  // kU points per thread in flight
         const int i = j0 + u * GTg + gtid_g;
         const bool live = i < m;
         vv[u][0] = live ? src.x[st + i] : T(0);
         vv[u][1] = live ? src.y[st + i] : T(0);
         vv[u][2] = live ? src.z[st + i] : T(0);
         oo[u] = live ? src.o[st + i] : 0;
       }
#pragma unroll
       for (int u = 0; u < kU; ++u) {
        const int i = j0 + u * GTg + gtid_g;
        const bool live = i < m;
        const T v[3] = {vv[u][0], vv[u][1], vv[u][2]};
        const int32_t o = oo[u];
        int cat = 3;  // 0 left, 1 boundary bin, 2 right
        if (live) {
          if (split) {
            const int bn = bin_of<kBins1>(ax == 0 ? v[0] : (ax == 1 ? v[1] : v[2]), lo, inv);
            cat = bn < bstar ? 0 : (bn == bstar ? 1 : 2);
          } else {
            cat = 0;
          }
        }
        int pos = 0;
        if (split) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const unsigned mk = __ballot_sync(0xffffffffu, cat == k);
            if (!mk) continue;
            const int ldr = __ffs(mk) - 1;
            int basek = 0;
            if (lane == ldr)  // rank 1's counters start after rank 0's points
              basek = atomicAdd(k == 0 ? &s_cl[s] : (k == 1 ? &s_cm[s] : &s_cr[s]), __popc(mk));
            basek = __shfl_sync(0xffffffffu, basek, ldr);
            if (cat == k) {
              const int t = basek + __popc(mk & ((1u << lane) - 1u));
              if (k == 0) pos = t;
              else if (k == 1) pos = t < take ? lt + t : nl + (t - take);
              else pos = nl + (midc - take) + t;
            }
          }
        } else {
          pos = i;
        }
        if (live) {
          dst.x[st + pos] = v[0];
          dst.y[st + pos] = v[1];
          dst.z[st + pos] = v[2];
          dst.o[st + pos] = o;
          const bool left = pos < nl;  // registers only (no dynamic index)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const T al = v[c] < a[0][c] ? v[c] : a[0][c], ar = v[c] < a[1][c] ? v[c] : a[1][c];
            const T zl = v[c] > z[0][c] ? v[c] : z[0][c], zr = v[c] > z[1][c] ? v[c] : z[1][c];
            a[0][c] = left ? al : a[0][c];
            z[0][c] = left ? zl : z[0][c];
            a[1][c] = left ? a[1][c] : ar;
            z[1][c] = left ? z[1][c] : zr;
          }
        }
       }
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (!__any_sync(0xffffffffu, a[k][0] <= z[k][0])) continue;  // no point of child k
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const T mn = bmin(a[k][c]), mx = bmax(z[k][c]);
          if (lane == 0) {
            atomicMin(&s_cbox[2 * s + k][c], O::enc(mn));
            atomicMax(&s_cbox[2 * s + k][3 + c], O::enc(mx));
          }
        }
      }
    }
    if constexpr (CL > 1) {  // children boxes = both partial boxes
      sync_all();  // also: every rank's partition atomics done
      I pv = 0;
      const bool mine = tid < 2 * S * 6;
      if (mine) pv = ld_peer(&s_cbox[tid / 6][tid % 6]);
      sync_all();
      if (mine) {
        I& o = s_cbox[tid / 6][tid % 6];
        o = tid % 6 < 3 ? (pv < o ? pv : o) : (pv > o ? pv : o);
      }
    }
    __syncthreads();
    // next level's segment list (children in order; unsplit segments carried):
    // warp 0 scans the children counts (S <= kMaxSeg / 2 = 64: two per lane),
    // then one thread per segment writes its children, one per child copies
    if (warp == 0) {
      const int c0 = lane < S ? (s_m[lane] > bs ? 2 : 1) : 0;
      const int c1 = lane + 32 < S ? (s_m[lane + 32] > bs ? 2 : 1) : 0;
      int p0 = c0, p1 = c1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a0 = __shfl_up_sync(0xffffffffu, p0, o), a1 = __shfl_up_sync(0xffffffffu, p1, o);
        if (lane >= o) {
          p0 += a0;
          p1 += a1;
        }
      }
      const int t0 = __shfl_sync(0xffffffffu, p0, 31);
      if (lane < S) s_nidx[lane] = p0 - c0;
      if (lane + 32 < S) s_nidx[lane + 32] = t0 + p1 - c1;
      if (lane == 31) s_S = t0 + p1;
    }
    __syncthreads();
    if (tid < S) {
      const int s = tid, o = s_nidx[s];
      if (s_m[s] > bs) {
        n_start[o] = s_start[s];
        n_m[o] = s_nl[s];
        n_from[o] = 2 * s;
        n_start[o + 1] = s_start[s] + s_nl[s];
        n_m[o + 1] = s_m[s] - s_nl[s];
        n_from[o + 1] = 2 * s + 1;
      } else {
        n_start[o] = s_start[s];
        n_m[o] = s_m[s];
        n_from[o] = 2 * s;
      }
    }
    __syncthreads();
    if (tid < s_S) {
      s_start[tid] = n_start[tid];
      s_m[tid] = n_m[tid];
#pragma unroll
      for (int c = 0; c < 6; ++c) s_box[tid][c] = s_cbox[n_from[tid]][c];
    }
    par ^= 1;
    __syncthreads();
  }

  // 2. hand the segments to the leaf kernel: count, parity of the buffer that
  //    holds them, (start, size) and box of each
  if (rank != 0) return;
  if (tid == 0) {
    seg_hdr[2 * b + 0] = s_S;
    seg_hdr[2 * b + 1] = par;
  }
  if (tid < s_S) {
    seg_sm[((int64_t)b * kMaxSeg + tid) * 2 + 0] = s_start[tid];
    seg_sm[((int64_t)b * kMaxSeg + tid) * 2 + 1] = s_m[tid];
#pragma unroll
    for (int c = 0; c < 6; ++c) seg_box[((int64_t)b * kMaxSeg + tid) * 6 + c] = O::dec(s_box[tid][c]);
  }
}

// K0-kd, second kernel: one warp per segment of the CTA phase, depth-first
// splits down to the leaves (= buckets).  When the host's bound `cap` on the
// segment size fits shared memory, the warp stages its segment there and
// ping-pongs between two shared-memory buffers (every pass is then an LDS/STS
// loop instead of an L2 round trip per 32 points); otherwise (cap == 0) it
// works on the global arrays as the CTA phase does.  Each finished leaf is
// written to the output arrays with its running distances (+inf), its box,
// and — for the last bucket — the padding slots (first point of the bucket,
// D = -inf, O = -1).
template <typename T>
__global__ void __launch_bounds__(512) bucket_kd_leaves_kernel(const BucketBuildParams p,
                                                               const int32_t* seg_hdr,
                                                               const int32_t* seg_sm,
                                                               const T* seg_box, int cap,
                                                               int wpc) {
  extern __shared__ __align__(16) unsigned char kd_smem[];
  const int b = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = blockIdx.x * wpc + warp;
  const int S = seg_hdr[2 * b + 0], par0 = seg_hdr[2 * b + 1];
  if (warp >= wpc || s0 >= S) return;  // warps are independent (no block barriers)
  const int n = (int)p.n;
  const int bs = (int)p.bs;
  const int64_t base = (int64_t)b * p.nslots;
  const Bufs<T> out{static_cast<T*>(p.X) + base, static_cast<T*>(p.Y) + base,
                   static_cast<T*>(p.Z) + base, p.O + base};
  const Bufs<T> tmp{static_cast<T*>(p.TX) + base, static_cast<T*>(p.TY) + base,
                    static_cast<T*>(p.TZ) + base, p.TO + base};
  // D is T, or double under FFPS_F32_F64 (float coordinates, binary64 keys)
  auto put_d = [&](int64_t i, T v) {
    if (sizeof(T) == 4 && p.d_wide) static_cast<double*>(p.D)[base + i] = (double)v;
    else static_cast<T*>(p.D)[base + i] = v;
  };
  T* BB = static_cast<T*>(p.BB) + (int64_t)b * p.nbuckets * 6;
  const T pinf = (T)INFINITY;

  // per-warp shared memory: histogram, DFS stack, then (staged) buffers A, B
  unsigned char* wb = kd_smem + (size_t)warp * kd_leaves_warp_bytes(cap, (int)sizeof(T));
  uint32_t* h = reinterpret_cast<uint32_t*>(wb);
  int* w_start = reinterpret_cast<int*>(h + kBinsL);
  int* w_m = w_start + kStack;
  int* w_par = w_m + kStack;
  T* w_box = reinterpret_cast<T*>(w_par + kStack + (kStack & 1));  // [kStack][6], 8-B aligned

  const int st0 = seg_sm[((int64_t)b * kMaxSeg + s0) * 2 + 0];
  const int m0 = seg_sm[((int64_t)b * kMaxSeg + s0) * 2 + 1];
  FFPS_CHECK(cap == 0 || m0 <= cap);  // the staged segment fits its buffers
  Bufs<T> P0, P1;
  if (cap > 0) {
    // stage the segment with four TMA bulk copies (x, y, z, o; 16-B aligned:
    // segments start on bucket boundaries, sizes rounded up inside the
    // nslots-long arrays); P0 / P1 point at the buffers minus st0, so global
    // positions index them directly
    uint64_t* sbar = reinterpret_cast<uint64_t*>(w_box + kStack * 6);
    T* A = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(sbar) + 16);
    const Bufs<T> src = par0 ? tmp : out;
    Bufs<T> bufA{A, A + cap, A + 2 * cap, reinterpret_cast<int32_t*>(A + 3 * cap)};
    Bufs<T> bufB{A + 3 * cap + cap * 4 / (int)sizeof(T), nullptr, nullptr, nullptr};
    bufB.y = bufB.x + cap;
    bufB.z = bufB.x + 2 * cap;
    bufB.o = reinterpret_cast<int32_t*>(bufB.x + 3 * cap);
    {
      const uint32_t bar = smem_u32(sbar);
      const uint32_t bt = (uint32_t)(((size_t)m0 * sizeof(T) + 15) / 16 * 16);
      const uint32_t bo = (uint32_t)(((size_t)m0 * 4 + 15) / 16 * 16);
      const bool aligned = ((reinterpret_cast<uintptr_t>(src.x + st0) |
                             reinterpret_cast<uintptr_t>(src.y + st0) |
                             reinterpret_cast<uintptr_t>(src.z + st0) |
                             reinterpret_cast<uintptr_t>(src.o + st0)) & 15) == 0;
      if (!aligned) {  // carved arrays are 16-B aligned (abi.cu box_bytes); belt and braces
        for (int i = lane; i < m0; i += 32) {
          bufA.x[i] = src.x[st0 + i];
          bufA.y[i] = src.y[st0 + i];
          bufA.z[i] = src.z[st0 + i];
          bufA.o[i] = src.o[st0 + i];
        }
        __syncwarp();
      } else if (lane == 0) {
        mbar_init(bar, 1);
        fence_mbar_init_cta();
        mbar_arrive_expect_tx(bar, 3 * bt + bo);
        bulk_g2s(smem_u32(bufA.x), src.x + st0, bt, bar);
        bulk_g2s(smem_u32(bufA.y), src.y + st0, bt, bar);
        bulk_g2s(smem_u32(bufA.z), src.z + st0, bt, bar);
        bulk_g2s(smem_u32(bufA.o), src.o + st0, bo, bar);
      }
      __syncwarp();
      if (aligned) mbar_wait(bar, 0);
    }
    P0 = Bufs<T>{bufA.x - st0, bufA.y - st0, bufA.z - st0, bufA.o - st0};
    P1 = Bufs<T>{bufB.x - st0, bufB.y - st0, bufB.z - st0, bufB.o - st0};
  } else {
    P0 = par0 ? tmp : out;
    P1 = par0 ? out : tmp;
  }
  if (lane == 0) {
    w_start[0] = st0;
    w_m[0] = m0;
    w_par[0] = 0;
#pragma unroll
    for (int c = 0; c < 6; ++c) w_box[c] = seg_box[((int64_t)b * kMaxSeg + s0) * 6 + c];
  }
  int top = 1;
  __syncwarp();
  while (top > 0) {
    --top;
    const int st = w_start[top], m = w_m[top], pr = w_par[top];
    T bx[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) bx[c] = w_box[top * 6 + c];
    __syncwarp();
    const Bufs<T> src = pr ? P1 : P0, dst = pr ? P0 : P1;
    if (m <= bs) {
      // leaf = bucket q: into the output arrays (unless it already is there),
      // D = +inf; its box is the exact min/max the split (or the CTA phase)
      // computed for it; the last bucket also gets its padding slots
      const bool copy = src.x + st != out.x + st;
      T f0 = T(0), f1 = T(0), f2 = T(0);
      for (int i = lane; i < m; i += 32) {
        const T v0 = src.x[st + i], v1 = src.y[st + i], v2 = src.z[st + i];
        if (copy) {
          out.x[st + i] = v0;
          out.y[st + i] = v1;
          out.z[st + i] = v2;
          out.o[st + i] = src.o[st + i];
        }
        put_d(st + i, pinf);
        if (i == 0) {
          f0 = v0;
          f1 = v1;
          f2 = v2;
        }
      }
      const int q = st / bs;
      const T bl = lane == 0 ? bx[0] : lane == 1 ? bx[1] : lane == 2 ? bx[2]
                 : lane == 3 ? bx[3] : lane == 4 ? bx[4] : bx[5];  // no dynamic index
      if (lane < 6) BB[(int64_t)q * 6 + lane] = bl;
      if (st + m == n && (int64_t)n < p.nslots) {
        f0 = __shfl_sync(0xffffffffu, f0, 0);
        f1 = __shfl_sync(0xffffffffu, f1, 0);
        f2 = __shfl_sync(0xffffffffu, f2, 0);
        for (int s = n + lane; s < (int)p.nslots; s += 32) {
          out.x[s] = f0;
          out.y[s] = f1;
          out.z[s] = f2;
          put_d(s, -pinf);
          out.o[s] = -1;
        }
      }
      continue;
    }
    const T e0 = bx[3] - bx[0], e1 = bx[4] - bx[1], e2 = bx[5] - bx[2];
    const int ax = e0 >= e1 ? (e0 >= e2 ? 0 : 2) : (e1 >= e2 ? 1 : 2);
    const T ext = ax == 0 ? e0 : (ax == 1 ? e1 : e2);
    const T lo = ax == 0 ? bx[0] : (ax == 1 ? bx[1] : bx[2]);
    const T inv = ext > (T)0 ? (T)kBinsL / ext : (T)0;
    const int nl = left_size(m, bs);
    const T* v = ax == 0 ? src.x : (ax == 1 ? src.y : src.z);
#pragma unroll 8
    for (int j = 0; j < kBinsL / 32; ++j) h[j * 32 + lane] = 0u;
    __syncwarp();
    for (int i = lane; i < m; i += 32) atomicAdd(&h[haddr<kBinsL>(bin_of<kBinsL>(v[st + i], lo, inv))], 1u);
    __syncwarp();
    int bstar, lt, midc;
    find_split<kBinsL>(h, nl, lane, bstar, lt, midc);
    const int take = nl - lt;
    int cl = 0, cm = 0, cr = 0;
    T a[2][3], z[2][3];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a[k][c] = pinf;
        z[k][c] = -pinf;
      }
    for (int i0 = 0; i0 < m; i0 += 32) {
      const int i = i0 + lane;
      const bool live = i < m;
      T p3[3] = {T(0), T(0), T(0)};
      int32_t o = 0;
      int cat = 3;
      if (live) {
        p3[0] = src.x[st + i];
        p3[1] = src.y[st + i];
        p3[2] = src.z[st + i];
        o = src.o[st + i];
        const int bn = bin_of<kBinsL>(ax == 0 ? p3[0] : (ax == 1 ? p3[1] : p3[2]), lo, inv);
        cat = bn < bstar ? 0 : (bn == bstar ? 1 : 2);
      }
      const unsigned mk0 = __ballot_sync(0xffffffffu, cat == 0);
      const unsigned mk1 = __ballot_sync(0xffffffffu, cat == 1);
      const unsigned mk2 = __ballot_sync(0xffffffffu, cat == 2);
      const unsigned below = (1u << lane) - 1u;
      int pos = 0;
      if (cat == 0) {
        pos = cl + __popc(mk0 & below);
      } else if (cat == 1) {
        const int t = cm + __popc(mk1 & below);
        pos = t < take ? lt + t : nl + (t - take);
      } else if (cat == 2) {
        pos = nl + (midc - take) + cr + __popc(mk2 & below);
      }
      cl += __popc(mk0);
      cm += __popc(mk1);
      cr += __popc(mk2);
      if (live) {
        dst.x[st + pos] = p3[0];
        dst.y[st + pos] = p3[1];
        dst.z[st + pos] = p3[2];
        dst.o[st + pos] = o;
        const bool left = pos < nl;  // registers only (no dynamic index)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const T al = p3[c] < a[0][c] ? p3[c] : a[0][c], ar = p3[c] < a[1][c] ? p3[c] : a[1][c];
          const T zl = p3[c] > z[0][c] ? p3[c] : z[0][c], zr = p3[c] > z[1][c] ? p3[c] : z[1][c];
          a[0][c] = left ? al : a[0][c];
          z[0][c] = left ? zl : z[0][c];
          a[1][c] = left ? a[1][c] : ar;
          z[1][c] = left ? z[1][c] : zr;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a[k][c] = bmin(a[k][c]);
        z[k][c] = bmax(z[k][c]);
      }
    if (top + 2 > kStack) __trap();  // depth <= log2(n / BS) + 1 < kStack
    if (lane == 0) {  // push right then left (left processed first; order is irrelevant)
      w_start[top] = st + nl;
      w_m[top] = m - nl;
      w_par[top] = pr ^ 1;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        w_box[top * 6 + c] = a[1][c];
        w_box[top * 6 + 3 + c] = z[1][c];
      }
      w_start[top + 1] = st;
      w_m[top + 1] = nl;
      w_par[top + 1] = pr ^ 1;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        w_box[(top + 1) * 6 + c] = a[0][c];
        w_box[(top + 1) * 6 + 3 + c] = z[0][c];
      }
    }
    top += 2;
    __syncwarp();
  }
}

// histograms of the CTA phase
size_t bucket_kd_smem() { return (size_t)kMaxSeg * kBins1 * sizeof(uint32_t); }

// largest segment the CTA phase hands over: the split sizes depend on n and
// the bucket size only (left_size), so the host replays the level loop
static int kd_max_segment(int64_t n, int64_t bs) {
  std::vector<int64_t> seg{n};
  for (;;) {
    bool any = false;
    for (int64_t m : seg) any |= m > bs;
    if (!any || 2 * seg.size() > (size_t)kMaxSeg) break;
    std::vector<int64_t> nx;
    for (int64_t m : seg) {
      if (m > bs) {
        const int64_t nl = ((m / bs + 1) / 2) * bs;
        nx.push_back(nl);
        nx.push_back(m - nl);
      } else {
        nx.push_back(m);
      }
    }
    seg.swap(nx);
  }
  int64_t mx = 0;
  for (int64_t m : seg) mx = m > mx ? m : mx;
  return (int)mx;
}

cudaError_t launch_bucket_kd(int dtype, const BucketBuildParams& p, int64_t batch,
                             cudaStream_t st) {
  const int esz = dtype == 0 ? 4 : 8;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  // leaf kernel: up to 4 warps (segments) per CTA with their segments staged
  // in shared memory; 2 or 1 for bigger segments; global arrays beyond that
  const int mmax = kd_max_segment(p.n, p.bs);
  int cap = (mmax + 31) / 32 * 32, wpc = 16;
  while (wpc > 1 && (size_t)wpc * kd_leaves_warp_bytes(cap, esz) > (size_t)optin) --wpc;
  if ((size_t)wpc * kd_leaves_warp_bytes(cap, esz) > (size_t)optin) {
    cap = 0;
    wpc = 4;
  }
  if (const char* v = getenv("FFPS_KD_STAGE"))  // A/B: 0 = leaves on the global arrays
    if (atoi(v) == 0) {
      cap = 0;
      wpc = 4;
    }
  const size_t leaves_smem = (size_t)wpc * kd_leaves_warp_bytes(cap, esz);
  // segment hand-off: [batch][2] header, [batch][kMaxSeg][2] (start, size),
  // [batch][kMaxSeg][6] boxes
  const size_t hdr_b = (size_t)batch * 2 * 4, sm_b = (size_t)batch * kMaxSeg * 2 * 4;
  const size_t box_b = (size_t)batch * kMaxSeg * 6 * esz;
  unsigned char* segs = nullptr;
  e = scratch_alloc(reinterpret_cast<void**>(&segs), hdr_b + sm_b + box_b + 64, st);
  if (e != cudaSuccess) return e;
  int32_t* seg_hdr = reinterpret_cast<int32_t*>(segs);
  int32_t* seg_sm = reinterpret_cast<int32_t*>(segs + hdr_b);
  void* seg_box = segs + ((hdr_b + sm_b + 15) / 16) * 16;
  // CTA phase: 2 CTAs per cloud (a cluster) while the batch fits the SMs twice
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  int cl = batch * 2 <= sms ? 2 : 1;
  if (const char* v = getenv("FFPS_KD_CL"))  // A/B: 1 or 2
    if (atoi(v) == 1 || atoi(v) == 2) cl = atoi(v);
  const void* f1 = dtype == 0 ? (cl == 2 ? reinterpret_cast<const void*>(&bucket_kd_kernel<float, 2>)
                                         : reinterpret_cast<const void*>(&bucket_kd_kernel<float, 1>))
                              : (cl == 2 ? reinterpret_cast<const void*>(&bucket_kd_kernel<double, 2>)
                                         : reinterpret_cast<const void*>(&bucket_kd_kernel<double, 1>));
  const void* f2 = dtype == 0 ? reinterpret_cast<const void*>(&bucket_kd_leaves_kernel<float>)
                              : reinterpret_cast<const void*>(&bucket_kd_leaves_kernel<double>);
  e = cudaFuncSetAttribute(f1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bucket_kd_smem());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(f2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)leaves_smem);
  if (e == cudaSuccess) {
    void* a1[] = {const_cast<BucketBuildParams*>(&p), &seg_hdr, &seg_sm, &seg_box};
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3((unsigned)(batch * cl), 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = bucket_kd_smem();
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelExC(&cfg, f1, a1);
  }
  if (e == cudaSuccess) {
    void* a2[] = {const_cast<BucketBuildParams*>(&p), &seg_hdr, &seg_sm, &seg_box, &cap, &wpc};
    e = cudaLaunchKernel(f2, dim3((unsigned)((kMaxSeg + wpc - 1) / wpc), (unsigned)batch),
                         dim3(32 * wpc), a2, leaves_smem, st);
  }
  cudaError_t e2 = scratch_free(segs, st);
  return e != cudaSuccess ? e : e2;
}

// K0 entry points of the bucketed schedules (K1b, K1g, K5): the kd build,
// two launches (CTA phase + leaf phase).  (The Morton-grid build of round 1
// was retired in round 2: kd leaves flag 2-4x fewer buckets per point.)
int bucket_build_launches(const BucketBuildParams&) { return 2; }

cudaError_t launch_bucket_build(int dtype, const BucketBuildParams& p, int64_t batch,
                                cudaStream_t st) {
  return launch_bucket_kd(dtype, p, batch, st);
}

}  // namespace ffps
