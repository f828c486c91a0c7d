// Arithmetic traits shared by the greedy kernels (fps_greedy.cu, fps_bucket.cu):
// the reference's distance formula with every operation separately rounded
// (fps_core.py:74-83), the order-preserving bit view used for argmax keys,
// warp reductions, and the DSMEM record format of the cluster kernel.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

namespace ffps {

// ---- packed f32x2 arithmetic (sm_100: FADD2 / FMUL2, IEEE RN per lane) ----
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "sub.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
// a*a + z with z = -0.0 supplied at RUN time (GreedyParams::neg_zero): equal to
// the separately rounded square RN(a*a) for every a (adding -0 to the exact
// product changes nothing, and +0 + -0 = +0).  A plain mul.rn.f32x2 followed
// by add.rn.f32x2 is contracted into FFMA2 by ptxas 12.9 even with
// --fmad=false, which would round (a*a + b) once and break bit-exactness; an
// addend ptxas cannot prove to be -0 keeps the square a separate FFMA2.
__device__ __forceinline__ float2 sq2(float2 a, float2 z) {
  float2 r;
  asm("{.reg .b64 a, z, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 z, {%4, %5};\n\t"
      "fma.rn.f32x2 d, a, a, z;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(z.x), "f"(z.y));
  return r;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

template <typename T>
struct Arith;

template <>
struct Arith<float> {
  using bits_t = int32_t;
  using pair_t = float2;
  using vec_t = float4;
  static constexpr int VW = 4;             // slots per 16-byte smem vector
  static constexpr int REC_STRIDE = 32;    // bytes per exchange record in smem
  static constexpr uint32_t REC_TX = 20;   // bytes pushed per record
  __device__ static __forceinline__ float pinf() { return __int_as_float(0x7f800000); }
  __device__ static __forceinline__ float ninf() { return __int_as_float(0xff800000); }
  __device__ static __forceinline__ pair_t mk(float a, float b) { return make_float2(a, b); }
  // fps_core.py:74-83: ((xs-px)^2 + (ys-py)^2) + (zs-pz)^2, separately rounded
  __device__ static __forceinline__ float d2(float x, float y, float z, float px, float py,
                                             float pz) {
    const float dx = __fsub_rn(x, px), dy = __fsub_rn(y, py), dz = __fsub_rn(z, pz);
    return __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
  }
  // Lower bound of d2(x, p) over a box [lo, hi] with the SAME rounded ops: per
  // axis g = max(RN(lo - p), RN(p - hi), 0) <= |RN(x - p)| for every x in the
  // box (RN is monotone and odd), and RN square / RN sum are monotone, so the
  // computed d2(x, p) >= box_d2 exactly — skipping a box whose bound is >= its
  // max distance leaves every min(dist, d2) unchanged, bit for bit.
  __device__ static __forceinline__ float box_d2(float px, float py, float pz, const float* lo,
                                                 const float* hi) {
    const float gx = max3f(__fsub_rn(lo[0], px), __fsub_rn(px, hi[0]), 0.0f);
    const float gy = max3f(__fsub_rn(lo[1], py), __fsub_rn(py, hi[1]), 0.0f);
    const float gz = max3f(__fsub_rn(lo[2], pz), __fsub_rn(pz, hi[2]), 0.0f);
    return __fadd_rn(__fadd_rn(__fmul_rn(gx, gx), __fmul_rn(gy, gy)), __fmul_rn(gz, gz));
  }
  static constexpr bits_t kmin = (bits_t)0x80000000;  // below every key, -inf included
  // box_d2 with the box stored as per-axis pairs (lo, -hi) and pp = (-p, p):
  // one FADD2 gives (RN(lo - p), RN(p - hi)) — the same two rounded values.
  __device__ static __forceinline__ float box_d2_pairs(const float2* lnh, float2 ppx, float2 ppy,
                                                       float2 ppz, float2 nz) {
    const float2 ax = add2(lnh[0], ppx), ay = add2(lnh[1], ppy), az = add2(lnh[2], ppz);
    const float2 g = make_float2(max3f(ax.x, ax.y, 0.0f), max3f(ay.x, ay.y, 0.0f));
    const float gz = max3f(az.x, az.y, 0.0f);
    const float2 s = sq2(g, nz);
    return __fadd_rn(__fadd_rn(s.x, s.y), __fmul_rn(gz, gz));
  }
  // two points at once: d = min(d, d2(p)), gm = max(gm, d.x, d.y); nz = (-0, -0)
  __device__ static __forceinline__ void upd2(pair_t& d, pair_t x, pair_t y, pair_t z,
                                              pair_t px, pair_t py, pair_t pz, pair_t nz,
                                              float& gm) {
    const float2 dx = sub2(x, px), dy = sub2(y, py), dz = sub2(z, pz);
    const float2 s = add2(add2(sq2(dx, nz), sq2(dy, nz)), sq2(dz, nz));
    d.x = fminf(d.x, s.x);
    d.y = fminf(d.y, s.y);
    gm = max3f(gm, d.x, d.y);
  }
  __device__ static __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
  __device__ static __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
  __device__ static __forceinline__ bits_t bits(float v) { return __float_as_int(v); }
  __device__ static __forceinline__ float from_bits(bits_t b) { return __int_as_float(b); }
  __device__ static __forceinline__ bits_t warp_max(bits_t v) {
    return __reduce_max_sync(0xffffffffu, v);
  }
  __device__ static __forceinline__ bits_t shfl(bits_t v, int l) {
    return __shfl_sync(0xffffffffu, v, l);
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
  // record: {value bits, index, x, y} + {z}
  __device__ static __forceinline__ void send(uint32_t raddr, uint32_t rbar, bits_t v,
                                              uint32_t g, float x, float y, float z) {
    st_async_v4(raddr, rbar, (uint32_t)v, g, __float_as_uint(x), __float_as_uint(y));
    st_async_b32(raddr + 16, rbar, __float_as_uint(z));
  }
  __device__ static __forceinline__ void recv(const unsigned char* rec, bits_t& v, uint32_t& g) {
    const int2 a = *reinterpret_cast<const int2*>(rec);
    v = a.x;
    g = (uint32_t)a.y;
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
  using pair_t = double2;
  using vec_t = double2;
  static constexpr int VW = 2;
  static constexpr int REC_STRIDE = 48;
  static constexpr uint32_t REC_TX = 40;
  __device__ static __forceinline__ double pinf() { return __longlong_as_double(0x7ff0000000000000ll); }
  __device__ static __forceinline__ double ninf() { return __longlong_as_double((long long)0xfff0000000000000ull); }
  __device__ static __forceinline__ pair_t mk(double a, double b) { return make_double2(a, b); }
  __device__ static __forceinline__ double d2(double x, double y, double z, double px,
                                              double py, double pz) {
    const double dx = __dsub_rn(x, px), dy = __dsub_rn(y, py), dz = __dsub_rn(z, pz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  }
  __device__ static __forceinline__ double box_d2(double px, double py, double pz,
                                                  const double* lo, const double* hi) {
    const double gx = fmax(fmax(__dsub_rn(lo[0], px), __dsub_rn(px, hi[0])), 0.0);
    const double gy = fmax(fmax(__dsub_rn(lo[1], py), __dsub_rn(py, hi[1])), 0.0);
    const double gz = fmax(fmax(__dsub_rn(lo[2], pz), __dsub_rn(pz, hi[2])), 0.0);
    return __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
  }
  static constexpr bits_t kmin = (bits_t)0x8000000000000000ull;
  __device__ static __forceinline__ double box_d2_pairs(const double2* lnh, double2 ppx,
                                                        double2 ppy, double2 ppz, double2) {
    const double gx = fmax(fmax(__dadd_rn(lnh[0].x, ppx.x), __dadd_rn(lnh[0].y, ppx.y)), 0.0);
    const double gy = fmax(fmax(__dadd_rn(lnh[1].x, ppy.x), __dadd_rn(lnh[1].y, ppy.y)), 0.0);
    const double gz = fmax(fmax(__dadd_rn(lnh[2].x, ppz.x), __dadd_rn(lnh[2].y, ppz.y)), 0.0);
    return __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
  }
  __device__ static __forceinline__ void upd2(pair_t& d, pair_t x, pair_t y, pair_t z,
                                              pair_t px, pair_t py, pair_t pz, pair_t,
                                              double& gm) {
    d.x = fmin(d.x, d2(x.x, y.x, z.x, px.x, py.x, pz.x));
    d.y = fmin(d.y, d2(x.y, y.y, z.y, px.y, py.y, pz.y));
    gm = fmax(gm, fmax(d.x, d.y));
  }
  __device__ static __forceinline__ double vmin(double a, double b) { return fmin(a, b); }
  __device__ static __forceinline__ double vmax(double a, double b) { return fmax(a, b); }
  __device__ static __forceinline__ bits_t bits(double v) { return __double_as_longlong(v); }
  __device__ static __forceinline__ double from_bits(bits_t b) { return __longlong_as_double(b); }
  __device__ static __forceinline__ bits_t warp_max(bits_t v) {
    // max of signed 64-bit keys: high word first (signed), then low word
    const int hi = __reduce_max_sync(0xffffffffu, (int)(v >> 32));
    const unsigned lo_c = ((int)(v >> 32) == hi) ? (unsigned)(v & 0xffffffffu) : 0u;
    const unsigned lo = __reduce_max_sync(0xffffffffu, lo_c);
    return (long long)(((unsigned long long)(unsigned)hi << 32) | lo);
  }
  __device__ static __forceinline__ bits_t shfl(bits_t v, int l) {
    return __shfl_sync(0xffffffffu, v, l);
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
  // record: {value bits, index} + {x, y} + {z}
  __device__ static __forceinline__ void send(uint32_t raddr, uint32_t rbar, bits_t v,
                                              uint32_t g, double x, double y, double z) {
    st_async_v2_b64(raddr, rbar, (uint64_t)v, (uint64_t)g);
    st_async_v2_b64(raddr + 16, rbar, (uint64_t)__double_as_longlong(x),
                    (uint64_t)__double_as_longlong(y));
    st_async_b64(raddr + 32, rbar, (uint64_t)__double_as_longlong(z));
  }
  __device__ static __forceinline__ void recv(const unsigned char* rec, bits_t& v, uint32_t& g) {
    const longlong2 a = *reinterpret_cast<const longlong2*>(rec);
    v = a.x;
    g = (uint32_t)a.y;
  }
  __device__ static __forceinline__ void recv_xyz(const unsigned char* rec, double& x, double& y,
                                                  double& z) {
    const double2 a = *reinterpret_cast<const double2*>(rec + 16);
    x = a.x; y = a.y;
    z = *reinterpret_cast<const double*>(rec + 32);
  }
};


}  // namespace ffps
