// K1 — persistent farthest-point-sampling kernel for sm_100a.
//
// Restates run_kernel (reference pkg/src/flashfps/fps_core.py:110-175) for a
// batch of clouds: one thread-block cluster per cloud runs the whole greedy
// loop on chip; the host is never involved between iterations.
//
// Data layout (per cluster = per cloud, C CTAs x NT threads):
//   * thread (rank, tid) owns the CONTIGUOUS point range
//         [base, base + Q),  base = (rank*NT + tid) * Q,  Q = P + S + G
//     so "lowest thread, then lowest slot" == "lowest point index", which is
//     the reference's tie rule (np.argmax first occurrence + chunk-order fold,
//     fps_core.py:94, :98-107).
//   * slots [0, P): x, y, z, dist in registers (pairs: float2 for FADD2/FMUL2);
//     slots [P, P+S): x, y, z in shared memory (16-byte vectors, SoA by
//     coordinate, conflict-free LDS.128), dist in registers;
//     slots [P+S, Q): {x, y, z, dist} streamed from a global spill buffer
//     (coalesced 16-byte loads) for clouds above on-chip capacity.
//   * padding slots (index >= n) and the selected points hold dist = -inf,
//     exactly like dist[best] = -inf in the reference (fps_core.py:169).
//   * slots are grouped by 8; each group keeps its running max, so the
//     winner search touches one group, not every slot.
//
// One iteration (everything below runs without host round trips):
//   1. update   d = ((dx*dx + dy*dy) + dz*dz), every op separately rounded
//               (RN, no FMA contraction — fps_core.py:74-83).  For fp32 two
//               points go through one packed f32x2 sub/mul/add (FADD2/FMUL2,
//               per-lane IEEE RN, bit-identical to the scalar ops);
//               dist = min(dist, d); group max via 3-input FMNMX.
//   2. warp     REDUX.MAX over the float bits (every live value is >= +0, so
//               the signed-int order is the float order; -inf is negative),
//               ballot for the lowest lane holding it, that lane finds its
//               lowest group/slot with the max (lazy argmax: no per-point
//               index bookkeeping) and the record {max, index, x, y, z} is
//               pushed by lanes 0..C-1 into EVERY cluster peer's shared
//               memory with st.async, completing the peer's mbarrier
//               transaction (DSMEM push; no __syncthreads, no cluster barrier).
//   3. combine  each warp waits on its CTA's mbarrier for the C*NW records,
//               reduces them (max value, then lowest index) with two warp
//               reductions and reads the winner's xyz; the owning thread marks
//               its slot dist = -inf.
// Records are double-buffered by iteration parity: a peer can only push
// iteration k+2 after every warp of this CTA pushed k+1, i.e. after they all
// consumed iteration k's records — one mbarrier wait per warp per iteration
// is the only synchronisation.
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"
#include "ffps_internal.h"
#include "ptx.cuh"

namespace ffps {

constexpr int kGroup = 8;  // slots per running-max group

// shared memory: [SG][3][NT] coordinate vectors, then 2 mbarriers (16 B),
// then the exchange records [2 parities][C ranks][NW warps] (sized per launch)
template <typename T, int NT>
__host__ __device__ constexpr size_t rec_bytes_per_rank() {
  return 2 * (size_t)(NT / 32) * Arith<T>::REC_STRIDE;
}

template <typename T, int NT, int P, int S, int MINB, bool SPILL>
__global__ void __launch_bounds__(NT, MINB) fps_greedy_kernel(const GreedyParams prm) {
  using A = Arith<T>;
  using bits_t = typename A::bits_t;
  using pair_t = typename A::pair_t;
  using vec_t = typename A::vec_t;
  constexpr int VW = A::VW;
  static_assert(P % 2 == 0, "register slots come in pairs");
  static_assert(S % VW == 0 && S % 2 == 0, "smem slots must fill whole 16-byte vectors");
  constexpr int SG = S / VW;      // smem vectors per coordinate
  constexpr int NW = NT / 32;
  constexpr int RS = A::REC_STRIDE;
  constexpr int GR = (P + kGroup - 1) / kGroup;  // register-slot groups
  constexpr int GM = (S + kGroup - 1) / kGroup;  // smem-slot groups
  constexpr int NG = (GR + GM) > 0 ? (GR + GM) : 1;

  extern __shared__ __align__(16) unsigned char smem[];
  vec_t* sv = reinterpret_cast<vec_t*>(smem);  // [SG][3][NT]
  unsigned char* tail = smem + (size_t)SG * 3 * NT * sizeof(vec_t);
  unsigned char* xch = tail + 16;               // [2][C][NW][RS]
  const uint32_t mbar0 = smem_u32(tail);        // 2 x u64

  const uint32_t C = cluster_nctarank();
  const uint32_t rank = cluster_ctarank();
  const int64_t b = cluster_id_x();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // all point positions are < 2^31 (checked by the C ABI): 32-bit loop state
  const int G = SPILL ? prm.spill_slots : 0;
  const int Q = P + S + G;
  const int base = ((int)rank * NT + tid) * Q;
  const int n = (int)prm.n;
  const int iters = (int)prm.iters;
  const T* X = static_cast<const T*>(prm.xyz) + b * prm.cloud_stride * 3;
  const int64_t* map = prm.index_map ? prm.index_map + b * prm.map_stride : nullptr;
  const int seed = (int)prm.seed_pos[b];
  vec_t* spill = nullptr;
  if (SPILL)
    spill = static_cast<vec_t*>(prm.spill) +
            (size_t)(b * C + rank) * (size_t)G * (sizeof(T) == 4 ? 1 : 2) * NT;

  // ---- load the owned range (fps_core.py:119-130: dist=+inf, dist[seed]=-inf)
  auto fetch = [&](int i, T& x, T& y, T& z, T& d) {
    if (i < n) {
      const int64_t src = map ? __ldg(map + i) : i;
      x = X[3 * src + 0];
      y = X[3 * src + 1];
      z = X[3 * src + 2];
      d = (i == seed) ? A::ninf() : A::pinf();
    } else {
      x = y = z = T(0);
      d = A::ninf();  // padding never wins
    }
  };

  constexpr int P2 = P > 0 ? P / 2 : 1;
  constexpr int S2 = S > 0 ? S / 2 : 1;
  pair_t rx[P2], ry[P2], rz[P2], rd[P2];
  pair_t sd[S2];
#pragma unroll
  for (int j = 0; j < P / 2; ++j) {
    T x0, y0, z0, d0, x1, y1, z1, d1;
    fetch(base + 2 * j, x0, y0, z0, d0);
    fetch(base + 2 * j + 1, x1, y1, z1, d1);
    rx[j] = A::mk(x0, x1);
    ry[j] = A::mk(y0, y1);
    rz[j] = A::mk(z0, z1);
    rd[j] = A::mk(d0, d1);
  }
#pragma unroll
  for (int q = 0; q < SG; ++q) {
    T xs[VW], ys[VW], zs[VW], ds[VW];
#pragma unroll
    for (int v = 0; v < VW; ++v) fetch(base + P + q * VW + v, xs[v], ys[v], zs[v], ds[v]);
#pragma unroll
    for (int v = 0; v < VW; v += 2) sd[(q * VW + v) / 2] = A::mk(ds[v], ds[v + 1]);
    T* sx = reinterpret_cast<T*>(&sv[(q * 3 + 0) * NT + tid]);
    T* sy = reinterpret_cast<T*>(&sv[(q * 3 + 1) * NT + tid]);
    T* sz = reinterpret_cast<T*>(&sv[(q * 3 + 2) * NT + tid]);
#pragma unroll
    for (int v = 0; v < VW; ++v) {
      sx[v] = xs[v];
      sy[v] = ys[v];
      sz[v] = zs[v];
    }
  }
  for (int s = 0; s < G; ++s) {
    T x, y, z, d;
    fetch(base + P + S + s, x, y, z, d);
    A::spill_store(spill, s, NT, tid, x, y, z, d);
  }

  T px, py, pz;
  {
    const int64_t src = map ? map[seed] : seed;
    px = X[3 * src + 0];
    py = X[3 * src + 1];
    pz = X[3 * src + 2];
  }
  if (rank == 0 && tid == 0) {
    prm.order[b * prm.out_stride] = seed;
    static_cast<T*>(prm.sel_d2)[b * prm.out_stride] = A::pinf();
  }
  if (tid == 0) {
    mbar_init(mbar0, 1);
    mbar_init(mbar0 + 8, 1);
    fence_mbar_init_cluster();
  }
  cluster_sync_all();  // mbarriers initialised cluster-wide; smem points visible

  const uint32_t xch0 = smem_u32(xch);
  const uint32_t nrec = C * NW;
  // optional phase trace (FFPS_TRACE_STREAM): cluster 0, lane 0 of every warp of
  // every rank: {start, update done, record pushed, records arrived, end}
  long long* trace = (prm.trace && b == 0 && lane == 0)
                         ? prm.trace + ((int64_t)rank * NW + warp) * prm.trace_iters * 8
                         : nullptr;
  for (int k = 1; k < iters; ++k) {
    long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    if (trace) t0 = clock64();
    const uint32_t par = (uint32_t)((k - 1) & 1);
    const uint32_t phase = (uint32_t)(((k - 1) >> 1) & 1);
    const uint32_t bar = mbar0 + 8 * par;
    if (tid == 0) mbar_arrive_expect_tx(bar, nrec * A::REC_TX);

    // 1. fused distance update + per-group running max --------------------------
    const pair_t ppx = A::mk(px, px), ppy = A::mk(py, py), ppz = A::mk(pz, pz);
    const pair_t nz = A::mk((T)prm.neg_zero, (T)prm.neg_zero);
    T gm[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) gm[g] = A::ninf();
#pragma unroll
    for (int j = 0; j < P / 2; ++j)
      A::upd2(rd[j], rx[j], ry[j], rz[j], ppx, ppy, ppz, nz, gm[(2 * j) / kGroup]);
#pragma unroll
    for (int q = 0; q < SG; ++q) {
      const vec_t vx = sv[(q * 3 + 0) * NT + tid];
      const vec_t vy = sv[(q * 3 + 1) * NT + tid];
      const vec_t vz = sv[(q * 3 + 2) * NT + tid];
      const T* ax = reinterpret_cast<const T*>(&vx);
      const T* ay = reinterpret_cast<const T*>(&vy);
      const T* az = reinterpret_cast<const T*>(&vz);
#pragma unroll
      for (int v = 0; v < VW; v += 2) {
        const int j = q * VW + v;  // smem slot
        A::upd2(sd[j / 2], A::mk(ax[v], ax[v + 1]), A::mk(ay[v], ay[v + 1]),
                A::mk(az[v], az[v + 1]), ppx, ppy, ppz, nz, gm[GR + j / kGroup]);
      }
    }
    T gsp = A::ninf();
    for (int s = 0; SPILL && s < G; ++s) {
      T x, y, z, d;
      A::spill_load(spill, s, NT, tid, x, y, z, d);
      const T nd = A::vmin(d, A::d2(x, y, z, px, py, pz));
      A::spill_store_d(spill, s, NT, tid, nd);
      gsp = A::vmax(gsp, nd);
    }
    T tm = gsp;
#pragma unroll
    for (int g = 0; g < NG; ++g) tm = A::vmax(tm, gm[g]);
    const bits_t tb = A::bits(tm);
    if (trace) t1 = clock64();

    // 2. warp max, lowest lane holding it finds its lowest slot ---------------
    const bits_t wb = A::warp_max(tb);
    const unsigned bal = __ballot_sync(0xffffffffu, tb == wb);
    const int wl = __ffs(bal) - 1;
    uint32_t widx = 0;
    T cx = T(0), cy = T(0), cz = T(0);
    if (lane == wl) {
      int gsel = NG;  // NG = spill group
#pragma unroll
      for (int g = NG - 1; g >= 0; --g)
        if (A::bits(gm[g]) == wb) gsel = g;
      int jj = -1;
#pragma unroll
      for (int g = 0; g < GR; ++g) {
        if (g == gsel) {
#pragma unroll
          for (int j = (g * kGroup + kGroup < P ? g * kGroup + kGroup : P) - 1; j >= g * kGroup;
               --j) {
            const pair_t dd = rd[j / 2];
            const T dv = (j & 1) ? dd.y : dd.x;
            if (A::bits(dv) == wb) {
              jj = j;
              cx = (j & 1) ? rx[j / 2].y : rx[j / 2].x;
              cy = (j & 1) ? ry[j / 2].y : ry[j / 2].x;
              cz = (j & 1) ? rz[j / 2].y : rz[j / 2].x;
            }
          }
        }
      }
#pragma unroll
      for (int g = 0; g < GM; ++g) {
        if (GR + g == gsel) {
          int js = -1;
#pragma unroll
          for (int j = (g * kGroup + kGroup < S ? g * kGroup + kGroup : S) - 1; j >= g * kGroup;
               --j) {
            const pair_t dd = sd[j / 2];
            const T dv = (j & 1) ? dd.y : dd.x;
            if (A::bits(dv) == wb) js = j;
          }
          if (js >= 0) {
            jj = P + js;
            const int q = js / VW, v = js % VW;
            const T* sc = reinterpret_cast<const T*>(sv);
            cx = sc[((size_t)(q * 3 + 0) * NT + tid) * VW + v];
            cy = sc[((size_t)(q * 3 + 1) * NT + tid) * VW + v];
            cz = sc[((size_t)(q * 3 + 2) * NT + tid) * VW + v];
          }
        }
      }
      if (SPILL && gsel == NG) {
        for (int s = 0; s < G; ++s) {
          T x, y, z, d;
          A::spill_load(spill, s, NT, tid, x, y, z, d);
          if (A::bits(d) == wb) {
            jj = P + S + s;
            cx = x;
            cy = y;
            cz = z;
            break;
          }
        }
      }
      widx = (uint32_t)(base + (jj < 0 ? 0 : jj));
    }
    // hand the record to lanes 0..C-1, which push it to the C peers in parallel
    widx = __shfl_sync(0xffffffffu, widx, wl);
    cx = __shfl_sync(0xffffffffu, cx, wl);
    cy = __shfl_sync(0xffffffffu, cy, wl);
    cz = __shfl_sync(0xffffffffu, cz, wl);
    if ((uint32_t)lane < C) {
      const uint32_t slot = xch0 + ((par * C + rank) * NW + warp) * RS;
      A::send(mapa(slot, lane), mapa(bar, lane), wb, widx, cx, cy, cz);
    }

    // 3. combine the C*NW records: max value, then lowest index ---------------
    if (trace) t2 = clock64();
    mbar_wait(bar, phase);
    if (trace) t3 = clock64();
    const unsigned char* recs = xch + (size_t)par * nrec * RS;
    bits_t lv = A::bits(A::ninf());
    uint32_t li = 0xffffffffu, lr = 0;
    for (uint32_t r = lane; r < nrec; r += 32) {
      bits_t v;
      uint32_t g;
      A::recv(recs + (size_t)r * RS, v, g);
      if (v > lv || (v == lv && g < li)) {
        lv = v;
        li = g;
        lr = r;
      }
    }
    const bits_t bv = A::warp_max(lv);
    const uint32_t bg = __reduce_min_sync(0xffffffffu, lv == bv ? li : 0xffffffffu);
    const int hl = __ffs(__ballot_sync(0xffffffffu, lv == bv && li == bg)) - 1;
    const uint32_t hr = __shfl_sync(0xffffffffu, lr, hl);
    A::recv_xyz(recs + (size_t)hr * RS, px, py, pz);
    if (rank == 0 && tid == 0) {  // fps_core.py:167-168
      prm.order[b * prm.out_stride + k] = bg;
      static_cast<T*>(prm.sel_d2)[b * prm.out_stride + k] = A::from_bits(bv);
    }
    const uint32_t off = bg - (uint32_t)base;
    if (off < (uint32_t)Q) {  // fps_core.py:169: dist[best] = -inf (one owner thread)
      const int jj = (int)off;
      if (jj < P) {
#pragma unroll
        for (int j = 0; j < P; ++j)
          if (jj == j) {
            if (j & 1) rd[j / 2].y = A::ninf();
            else rd[j / 2].x = A::ninf();
          }
      } else if (jj < P + S) {
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (jj == P + j) {
            if (j & 1) sd[j / 2].y = A::ninf();
            else sd[j / 2].x = A::ninf();
          }
      } else if (SPILL) {
        A::spill_store_d(spill, jj - P - S, NT, tid, A::ninf());
      }
    }
    if (trace && k < prm.trace_iters) {
      long long* r = trace + (int64_t)k * 8;
      r[0] = t0; r[1] = t1; r[2] = t2; r[3] = t3; r[4] = clock64();
    }
  }

  // positions -> original indices for restricted runs (fps_cache.py:197)
  if (map != nullptr && rank == 0) {
    __syncthreads();
    int64_t* order = prm.order + b * prm.out_stride;
    for (int k = tid; k < iters; k += NT) order[k] = __ldg(map + order[k]);
  }
  cluster_sync_all();  // no CTA leaves while peers may still push into it
}

template <typename T, int NT, int P, int S, int MINB, bool SPILL = false>
KernelInst make_inst() {
  constexpr int SG = S / Arith<T>::VW;
  KernelInst k;
  k.dtype = sizeof(T) == 4 ? 0 : 1;
  k.nt = NT;
  k.p = P;
  k.s = S;
  k.minb = MINB;
  k.spill = SPILL;
  k.fn = reinterpret_cast<const void*>(&fps_greedy_kernel<T, NT, P, S, MINB, SPILL>);
  k.smem_base = (size_t)SG * 3 * NT * 16 + 16;
  k.smem_per_rank = rec_bytes_per_rank<T, NT>();
  return k;
}

// Register budget: __launch_bounds__(NT, MINB) caps registers at
// 65536 / (NT * MINB) per thread; per thread a register slot costs 4 (f32) /
// 8 (f64) registers, an smem slot 1 / 2 registers plus 12 / 24 bytes of
// shared memory.
const KernelInst* greedy_instances(int* count) {
  static const KernelInst insts[] = {
      // float32, 2 CTAs per SM (another cloud's CTA hides the per-iteration sync)
      make_inst<float, 256, 2, 0, 2>(),
      make_inst<float, 256, 4, 0, 2>(),
      make_inst<float, 256, 8, 0, 2>(),
      make_inst<float, 256, 16, 0, 2>(),
      make_inst<float, 256, 16, 8, 2>(),
      make_inst<float, 256, 16, 16, 2>(),
      make_inst<float, 256, 16, 24, 2>(),
      make_inst<float, 256, 14, 36, 2>(),
      // float32, 3-4 CTAs per SM (smaller clouds / more clouds per SM)
      make_inst<float, 256, 8, 20, 3>(),
      make_inst<float, 256, 4, 16, 4>(),
      // float32, 128-thread CTAs: fewer threads -> less per-thread overhead,
      // more of the SM's register file + smem holds points (~25K per SM)
      make_inst<float, 128, 28, 72, 2>(),
      make_inst<float, 128, 10, 36, 4>(),
      // float32, 1 CTA per SM, 512 threads (largest clouds per cluster)
      make_inst<float, 512, 14, 36, 1>(),
      // spill variants: the rest of each thread's range streamed from HBM/L2
      make_inst<float, 256, 14, 36, 2, true>(),
      make_inst<float, 512, 14, 36, 1, true>(),
      // float64
      make_inst<double, 256, 2, 0, 2>(),
      make_inst<double, 256, 4, 0, 2>(),
      make_inst<double, 256, 8, 0, 2>(),
      make_inst<double, 256, 8, 8, 2>(),
      make_inst<double, 256, 6, 18, 2>(),
      make_inst<double, 512, 6, 18, 1>(),
      make_inst<double, 256, 6, 18, 2, true>(),
      make_inst<double, 512, 6, 18, 1, true>(),
  };
  *count = (int)(sizeof(insts) / sizeof(insts[0]));
  return insts;
}

}  // namespace ffps
