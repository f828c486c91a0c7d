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
//   * slots [0, P): x, y, z, dist in registers;
//     slots [P, P+S): x, y, z in shared memory (16-byte vectors, SoA by
//     coordinate, conflict-free LDS.128), dist in registers;
//     slots [P+S, Q): {x, y, z, dist} streamed from a global spill buffer
//     (coalesced 16-byte loads) for clouds above on-chip capacity.
//   * padding slots (index >= n) and the selected points hold dist = -inf,
//     exactly like dist[best] = -inf in the reference (fps_core.py:169).
//
// One iteration (everything below runs without host round trips):
//   1. update   d = ((dx*dx + dy*dy) + dz*dz), every op separately rounded
//               (RN, no FMA contraction — fps_core.py:74-83), dist = min(dist, d),
//               thread max tm (3-input FMNMX) — the only per-point work.
//   2. CTA max  REDUX.MAX over float bits (all live values are >= +0, so the
//               signed-int order is the float order; -inf is negative) into a
//               double-buffered smem slot, one __syncthreads.
//   3. winner   the lowest warp / lane holding the CTA max scans its own slots
//               for the lowest one equal to the max (lazy argmax: no per-point
//               index bookkeeping) and pushes a record {max, index, x, y, z}
//               into EVERY cluster peer's shared memory with st.async, which
//               completes the peer's mbarrier transaction (DSMEM push; no
//               cluster-wide barrier per iteration).
//   4. combine  every thread waits on its CTA's mbarrier for C records, takes
//               max value / lowest index, and gets the next point's xyz from
//               the record; the owning thread marks dist = -inf.
// Records and maxima are double-buffered by iteration parity, so a single
// __syncthreads + one mbarrier wait per iteration is all the synchronisation.
#include <cuda_runtime.h>

#include <cstdint>

#include "ffps_internal.h"
#include "ptx.cuh"

namespace ffps {

template <typename T>
struct Arith;

template <>
struct Arith<float> {
  using bits_t = int32_t;
  using vec_t = float4;
  static constexpr int VW = 4;             // slots per 16-byte vector
  static constexpr int REC_STRIDE = 32;    // bytes per exchange record in smem
  static constexpr uint32_t REC_TX = 20;   // bytes pushed per record
  __device__ static __forceinline__ float pinf() { return __int_as_float(0x7f800000); }
  __device__ static __forceinline__ float ninf() { return __int_as_float(0xff800000); }
  // fps_core.py:74-83: ((xs-px)^2 + (ys-py)^2) + (zs-pz)^2, separately rounded
  __device__ static __forceinline__ float d2(float x, float y, float z, float px, float py,
                                             float pz) {
    const float dx = __fsub_rn(x, px), dy = __fsub_rn(y, py), dz = __fsub_rn(z, pz);
    return __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
  }
  __device__ static __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
  __device__ static __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
  __device__ static __forceinline__ bits_t bits(float v) { return __float_as_int(v); }
  __device__ static __forceinline__ float from_bits(bits_t b) { return __int_as_float(b); }
  __device__ static __forceinline__ bits_t warp_max(bits_t v) {
    return __reduce_max_sync(0xffffffffu, v);
  }
  __device__ static __forceinline__ vec_t pack(const float* a) {
    return make_float4(a[0], a[1], a[2], a[3]);
  }
  __device__ static __forceinline__ void unpack(const vec_t& v, float* a) {
    a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
  }
  // spill slot s: one float4 {x, y, z, dist}
  __device__ static __forceinline__ void spill_load(const vec_t* sp, int s, int nt, int tid,
                                                    float& x, float& y, float& z, float& d) {
    const float4 v = sp[(size_t)s * nt + tid];
    x = v.x; y = v.y; z = v.z; d = v.w;
  }
  __device__ static __forceinline__ void spill_store(vec_t* sp, int s, int nt, int tid, float x,
                                                     float y, float z, float d) {
    sp[(size_t)s * nt + tid] = make_float4(x, y, z, d);
  }
  __device__ static __forceinline__ void spill_store_d(vec_t* sp, int s, int nt, int tid,
                                                       float d) {
    reinterpret_cast<float*>(sp + (size_t)s * nt + tid)[3] = d;
  }
  __device__ static __forceinline__ void send(uint32_t raddr, uint32_t rbar, bits_t v, int64_t g,
                                              float x, float y, float z) {
    st_async_v4(raddr, rbar, (uint32_t)v, (uint32_t)g, __float_as_uint(x), __float_as_uint(y));
    st_async_b32(raddr + 16, rbar, __float_as_uint(z));
  }
  __device__ static __forceinline__ void recv(const unsigned char* rec, bits_t& v, int64_t& g) {
    const int2 a = *reinterpret_cast<const int2*>(rec);
    v = a.x;
    g = (int64_t)(uint32_t)a.y;
  }
  __device__ static __forceinline__ void recv_xyz(const unsigned char* rec, float& x, float& y,
                                                  float& z) {
    const float2 a = *reinterpret_cast<const float2*>(rec + 8);
    x = a.x; y = a.y;
    z = *reinterpret_cast<const float*>(rec + 16);
  }
};

template <>
struct Arith<double> {
  using bits_t = long long;
  using vec_t = double2;
  static constexpr int VW = 2;
  static constexpr int REC_STRIDE = 48;
  static constexpr uint32_t REC_TX = 40;
  __device__ static __forceinline__ double pinf() { return __longlong_as_double(0x7ff0000000000000ll); }
  __device__ static __forceinline__ double ninf() { return __longlong_as_double((long long)0xfff0000000000000ull); }
  __device__ static __forceinline__ double d2(double x, double y, double z, double px,
                                              double py, double pz) {
    const double dx = __dsub_rn(x, px), dy = __dsub_rn(y, py), dz = __dsub_rn(z, pz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  }
  __device__ static __forceinline__ double vmin(double a, double b) { return fmin(a, b); }
  __device__ static __forceinline__ double vmax(double a, double b) { return fmax(a, b); }
  __device__ static __forceinline__ bits_t bits(double v) { return __double_as_longlong(v); }
  __device__ static __forceinline__ double from_bits(bits_t b) { return __longlong_as_double(b); }
  __device__ static __forceinline__ bits_t warp_max(bits_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const bits_t u = __shfl_xor_sync(0xffffffffu, v, o);
      v = u > v ? u : v;
    }
    return v;
  }
  __device__ static __forceinline__ vec_t pack(const double* a) { return make_double2(a[0], a[1]); }
  __device__ static __forceinline__ void unpack(const vec_t& v, double* a) {
    a[0] = v.x; a[1] = v.y;
  }
  // spill slot s: two double2 {x, y}, {z, dist}
  __device__ static __forceinline__ void spill_load(const vec_t* sp, int s, int nt, int tid,
                                                    double& x, double& y, double& z, double& d) {
    const double2 a = sp[(size_t)(2 * s) * nt + tid];
    const double2 b = sp[(size_t)(2 * s + 1) * nt + tid];
    x = a.x; y = a.y; z = b.x; d = b.y;
  }
  __device__ static __forceinline__ void spill_store(vec_t* sp, int s, int nt, int tid, double x,
                                                     double y, double z, double d) {
    sp[(size_t)(2 * s) * nt + tid] = make_double2(x, y);
    sp[(size_t)(2 * s + 1) * nt + tid] = make_double2(z, d);
  }
  __device__ static __forceinline__ void spill_store_d(vec_t* sp, int s, int nt, int tid,
                                                       double d) {
    reinterpret_cast<double*>(sp + (size_t)(2 * s + 1) * nt + tid)[1] = d;
  }
  __device__ static __forceinline__ void send(uint32_t raddr, uint32_t rbar, bits_t v, int64_t g,
                                              double x, double y, double z) {
    st_async_v2_b64(raddr, rbar, (uint64_t)v, (uint64_t)g);
    st_async_v2_b64(raddr + 16, rbar, (uint64_t)__double_as_longlong(x),
                    (uint64_t)__double_as_longlong(y));
    st_async_b64(raddr + 32, rbar, (uint64_t)__double_as_longlong(z));
  }
  __device__ static __forceinline__ void recv(const unsigned char* rec, bits_t& v, int64_t& g) {
    const longlong2 a = *reinterpret_cast<const longlong2*>(rec);
    v = a.x;
    g = a.y;
  }
  __device__ static __forceinline__ void recv_xyz(const unsigned char* rec, double& x, double& y,
                                                  double& z) {
    const double2 a = *reinterpret_cast<const double2*>(rec + 16);
    x = a.x; y = a.y;
    z = *reinterpret_cast<const double*>(rec + 32);
  }
};

constexpr int kMaxCluster = 16;

template <typename T, int NT>
__host__ __device__ constexpr size_t tail_offset_red() { return 16; }
template <typename T, int NT>
__host__ __device__ constexpr size_t tail_offset_xch() {
  return (16 + 2 * (NT / 32) * sizeof(typename Arith<T>::bits_t) + 15) / 16 * 16;
}
template <typename T, int NT>
__host__ __device__ constexpr size_t tail_bytes() {
  return tail_offset_xch<T, NT>() + 2 * kMaxCluster * Arith<T>::REC_STRIDE;
}

template <typename T, int NT, int P, int S, int MINB>
__global__ void __launch_bounds__(NT, MINB) fps_greedy_kernel(const GreedyParams prm) {
  using A = Arith<T>;
  using bits_t = typename A::bits_t;
  using vec_t = typename A::vec_t;
  constexpr int VW = A::VW;
  static_assert(S % VW == 0, "smem slots must fill whole 16-byte vectors");
  constexpr int SG = S / VW;
  constexpr int NW = NT / 32;
  constexpr int RS = A::REC_STRIDE;

  extern __shared__ __align__(16) unsigned char smem[];
  vec_t* sv = reinterpret_cast<vec_t*>(smem);  // [SG][3][NT]
  unsigned char* tail = smem + (size_t)SG * 3 * NT * sizeof(vec_t);
  bits_t* red = reinterpret_cast<bits_t*>(tail + tail_offset_red<T, NT>());  // [2][NW]
  unsigned char* xch = tail + tail_offset_xch<T, NT>();                      // [2][16][RS]
  const uint32_t mbar0 = smem_u32(tail);                                     // 2 x u64

  const uint32_t C = cluster_nctarank();
  const uint32_t rank = cluster_ctarank();
  const int64_t b = cluster_id_x();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = prm.spill_slots;
  const int64_t Q = P + S + G;
  const int64_t base = ((int64_t)rank * NT + tid) * Q;
  const int64_t n = prm.n;
  const T* X = static_cast<const T*>(prm.xyz) + b * prm.cloud_stride * 3;
  const int64_t* map = prm.index_map ? prm.index_map + b * prm.map_stride : nullptr;
  const int64_t seed = prm.seed_pos[b];
  int64_t* order = prm.order + b * prm.out_stride;
  T* sel = static_cast<T*>(prm.sel_d2) + b * prm.out_stride;
  vec_t* spill = nullptr;
  if (G > 0)
    spill = static_cast<vec_t*>(prm.spill) +
            (size_t)(b * C + rank) * (size_t)G * (sizeof(T) == 4 ? 1 : 2) * NT;

  // ---- load the owned range (fps_core.py:119-130: dist=+inf, dist[seed]=-inf)
  auto fetch = [&](int64_t i, T& x, T& y, T& z, T& d) {
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

  T rx[P > 0 ? P : 1], ry[P > 0 ? P : 1], rz[P > 0 ? P : 1], rd[P > 0 ? P : 1];
  T sd[S > 0 ? S : 1];
#pragma unroll
  for (int j = 0; j < P; ++j) fetch(base + j, rx[j], ry[j], rz[j], rd[j]);
#pragma unroll
  for (int q = 0; q < SG; ++q) {
    T xs[VW], ys[VW], zs[VW];
#pragma unroll
    for (int v = 0; v < VW; ++v) fetch(base + P + q * VW + v, xs[v], ys[v], zs[v], sd[q * VW + v]);
    sv[(q * 3 + 0) * NT + tid] = A::pack(xs);
    sv[(q * 3 + 1) * NT + tid] = A::pack(ys);
    sv[(q * 3 + 2) * NT + tid] = A::pack(zs);
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
    order[0] = seed;
    sel[0] = A::pinf();
  }
  if (tid == 0) {
    mbar_init(mbar0, 1);
    mbar_init(mbar0 + 8, 1);
    fence_mbar_init_cluster();
  }
  cluster_sync_all();  // mbarriers initialised cluster-wide; smem points visible

  const uint32_t xch0 = smem_u32(xch);
  for (int64_t k = 1; k < prm.iters; ++k) {
    const uint32_t par = (uint32_t)((k - 1) & 1);
    const uint32_t phase = (uint32_t)(((k - 1) >> 1) & 1);
    const uint32_t bar = mbar0 + 8 * par;

    // 1. fused distance update + thread max -----------------------------------
    T tm0 = A::ninf(), tm1 = A::ninf();
#pragma unroll
    for (int j = 0; j < P; ++j) {
      rd[j] = A::vmin(rd[j], A::d2(rx[j], ry[j], rz[j], px, py, pz));
      if (j & 1) tm1 = A::vmax(tm1, rd[j]);
      else tm0 = A::vmax(tm0, rd[j]);
    }
#pragma unroll
    for (int q = 0; q < SG; ++q) {
      T xs[VW], ys[VW], zs[VW];
      A::unpack(sv[(q * 3 + 0) * NT + tid], xs);
      A::unpack(sv[(q * 3 + 1) * NT + tid], ys);
      A::unpack(sv[(q * 3 + 2) * NT + tid], zs);
#pragma unroll
      for (int v = 0; v < VW; ++v) {
        T& d = sd[q * VW + v];
        d = A::vmin(d, A::d2(xs[v], ys[v], zs[v], px, py, pz));
        if (v & 1) tm1 = A::vmax(tm1, d);
        else tm0 = A::vmax(tm0, d);
      }
    }
    for (int s = 0; s < G; ++s) {
      T x, y, z, d;
      A::spill_load(spill, s, NT, tid, x, y, z, d);
      const T nd = A::vmin(d, A::d2(x, y, z, px, py, pz));
      A::spill_store_d(spill, s, NT, tid, nd);
      tm0 = A::vmax(tm0, nd);
    }
    const bits_t tb = A::bits(A::vmax(tm0, tm1));

    // 2. CTA max ----------------------------------------------------------------
    const bits_t wb = A::warp_max(tb);
    if (lane == 0) red[par * NW + warp] = wb;
    __syncthreads();
    bits_t cb = red[par * NW];
    int ws = 0;
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      const bits_t v = red[par * NW + w];
      if (v > cb) {
        cb = v;
        ws = w;
      }
    }
    if (tid == 0) mbar_arrive_expect_tx(bar, C * A::REC_TX);

    // 3. lowest holder of the CTA max finds its lowest slot and pushes the record
    if (warp == ws) {
      const unsigned bal = __ballot_sync(0xffffffffu, tb == cb);
      if (lane == __ffs(bal) - 1) {
        int jj = -1;
        T cx = T(0), cy = T(0), cz = T(0);
#pragma unroll
        for (int j = P - 1; j >= 0; --j)
          if (A::bits(rd[j]) == cb) {
            jj = j;
            cx = rx[j];
            cy = ry[j];
            cz = rz[j];
          }
        if (jj < 0) {
          int js = -1;
#pragma unroll
          for (int j = S - 1; j >= 0; --j)
            if (A::bits(sd[j]) == cb) js = j;
          if (js >= 0) {
            jj = P + js;
            const int q = js / VW, v = js % VW;
            const T* sc = reinterpret_cast<const T*>(sv);
            cx = sc[((size_t)(q * 3 + 0) * NT + tid) * VW + v];
            cy = sc[((size_t)(q * 3 + 1) * NT + tid) * VW + v];
            cz = sc[((size_t)(q * 3 + 2) * NT + tid) * VW + v];
          } else {
            for (int s = 0; s < G; ++s) {
              T x, y, z, d;
              A::spill_load(spill, s, NT, tid, x, y, z, d);
              if (A::bits(d) == cb) {
                jj = P + S + s;
                cx = x;
                cy = y;
                cz = z;
                break;
              }
            }
          }
        }
        const int64_t g = base + jj;
        const uint32_t slot = xch0 + (par * kMaxCluster + rank) * RS;
        for (uint32_t r = 0; r < C; ++r) A::send(mapa(slot, r), mapa(bar, r), cb, g, cx, cy, cz);
      }
    }

    // 4. combine the C records (max value, then lowest index) ------------------
    mbar_wait(bar, phase);
    const unsigned char* recs = xch + par * kMaxCluster * RS;
    bits_t bv;
    int64_t bg;
    A::recv(recs, bv, bg);
    uint32_t rw = 0;
    for (uint32_t r = 1; r < C; ++r) {
      bits_t v;
      int64_t g;
      A::recv(recs + r * RS, v, g);
      if (v > bv || (v == bv && g < bg)) {
        bv = v;
        bg = g;
        rw = r;
      }
    }
    A::recv_xyz(recs + rw * RS, px, py, pz);
    if (rank == 0 && tid == 0) {  // fps_core.py:167-168
      order[k] = bg;
      sel[k] = A::from_bits(bv);
    }
    if (bg >= base && bg < base + Q) {  // fps_core.py:169: dist[best] = -inf
      const int jj = (int)(bg - base);
#pragma unroll
      for (int j = 0; j < P; ++j)
        if (jj == j) rd[j] = A::ninf();
#pragma unroll
      for (int j = 0; j < S; ++j)
        if (jj == P + j) sd[j] = A::ninf();
      if (jj >= P + S) A::spill_store_d(spill, jj - P - S, NT, tid, A::ninf());
    }
  }

  // positions -> original indices for restricted runs (fps_cache.py:197)
  if (map != nullptr && rank == 0) {
    __syncthreads();
    for (int64_t k = tid; k < prm.iters; k += NT) order[k] = __ldg(map + order[k]);
  }
  cluster_sync_all();  // no CTA leaves while peers may still push into it
}

template <typename T, int NT, int P, int S, int MINB>
KernelInst make_inst() {
  constexpr int SG = S / Arith<T>::VW;
  KernelInst k;
  k.dtype = sizeof(T) == 4 ? 0 : 1;
  k.nt = NT;
  k.p = P;
  k.s = S;
  k.minb = MINB;
  k.fn = reinterpret_cast<const void*>(&fps_greedy_kernel<T, NT, P, S, MINB>);
  k.smem_bytes = (size_t)SG * 3 * NT * 16 + tail_bytes<T, NT>();
  return k;
}

// Register budget: __launch_bounds__(NT, MINB) caps registers at
// 65536 / (NT * MINB) = 128 for every instance below; per thread a register
// slot costs 4 (f32) / 8 (f64) registers, an smem slot 1 / 2 registers plus
// 12 / 24 bytes of shared memory.
const KernelInst* greedy_instances(int* count) {
  static const KernelInst insts[] = {
      // float32, 2 CTAs per SM (another cloud's CTA hides the per-iteration sync)
      make_inst<float, 256, 1, 0, 2>(),
      make_inst<float, 256, 2, 0, 2>(),
      make_inst<float, 256, 4, 0, 2>(),
      make_inst<float, 256, 8, 0, 2>(),
      make_inst<float, 256, 16, 0, 2>(),
      make_inst<float, 256, 16, 8, 2>(),
      make_inst<float, 256, 16, 16, 2>(),
      make_inst<float, 256, 16, 24, 2>(),
      make_inst<float, 256, 15, 36, 2>(),
      // float32, 1 CTA per SM, 512 threads (largest clouds per cluster)
      make_inst<float, 512, 15, 36, 1>(),
      // float64
      make_inst<double, 256, 1, 0, 2>(),
      make_inst<double, 256, 2, 0, 2>(),
      make_inst<double, 256, 4, 0, 2>(),
      make_inst<double, 256, 8, 0, 2>(),
      make_inst<double, 256, 8, 8, 2>(),
      make_inst<double, 256, 7, 18, 2>(),
      make_inst<double, 512, 7, 18, 1>(),
  };
  *count = (int)(sizeof(insts) / sizeof(insts[0]));
  return insts;
}

}  // namespace ffps
