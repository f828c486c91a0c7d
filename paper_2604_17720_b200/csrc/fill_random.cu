// K2r — budget fill, FillMode.SEEDED_RANDOM (reference
// pkg/src/flashfps/fps_prune.py:96-103): after a truncated greedy run of k
// iterations, append fill_n = m1 - k indices drawn by
//     np.random.default_rng(rng_seed).choice(pool, fill_n, replace=False)
// where pool is the ascending complement of the k picks in [0, n).  The draws
// follow NumPy's algorithm step for step (restated and pinned against NumPy in
// oracle/npchoice.py): PCG64 XSL-RR with buffered 32-bit halves, Lemire's
// bounded draw with rejection, then either the tail partial Fisher-Yates of
// arange(pop) (pop > 10000 and fill_n > pop // 50) or Floyd's algorithm over a
// linear-probing hash set followed by a Fisher-Yates of the picks.
//
// One CTA per cloud (all clouds start from the same generator state, as the
// reference seeds a fresh generator per call):
//   1. selection bitmap of [0, n) and the zero count before every word (block
//      scan) — the pool as ranks;
//   2. warp 0 runs the generator: the 32-bit value stream by a 32-step
//      jump-ahead of the 128-bit LCG per lane, the values mapped to draws 32
//      at a time (a Lemire rejection cuts the batch and shifts the later draws
//      by one value), then the tail shuffle 32 steps per batch (64 loads in
//      flight, in-batch aliasing resolved by a scan in step order, one store
//      per slot by its last writer); Floyd's branch (small fills) runs on
//      thread 0;
//   3. all threads map the drawn pool ranks to cloud indices (binary search of
//      the word prefix, then the rank-th zero bit of the word).
#include <cuda_runtime.h>

#include <cstdint>

#include "ffps_internal.h"

namespace ffps {

namespace {

constexpr int kRThreads = 512;

struct Pcg64 {
  uint64_t hi, lo, ihi, ilo;
  bool has32;
  uint32_t buf32;

  __device__ uint64_t next64() {
    constexpr uint64_t kMhi = 2549297995355413924ull, kMlo = 4865540595714422341ull;
    const uint64_t plo = lo * kMlo;
    const uint64_t phi = __umul64hi(lo, kMlo) + lo * kMhi + hi * kMlo;
    lo = plo + ilo;
    hi = phi + ihi + (lo < plo ? 1ull : 0ull);
    const uint64_t x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    return r ? (x >> r) | (x << (64u - r)) : x;
  }
  __device__ uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    const uint64_t v = next64();
    has32 = true;
    buf32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // random_bounded_uint64(off = 0, rng, mask = 0, use_masked = false), rng < 2^32
  __device__ uint32_t bounded(uint32_t rng) {
    if (rng == 0u) return 0u;
    if (rng == 0xffffffffu) return next32();
    const uint32_t excl = rng + 1u;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (0xffffffffu - rng) % excl;
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

// 128-bit LCG arithmetic for the jump-ahead of the PCG64 state
struct U128 {
  uint64_t hi, lo;
};
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {  // low 128 bits of a * b
  return U128{__umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo, a.lo * b.lo};
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  const uint64_t lo = a.lo + b.lo;
  return U128{a.hi + b.hi + (lo < a.lo ? 1ull : 0ull), lo};
}
__device__ __forceinline__ uint64_t pcg_output(U128 s) {  // XSL-RR
  const uint64_t x = s.hi ^ s.lo;
  const unsigned r = (unsigned)(s.hi >> 58);
  return r ? (x >> r) | (x << (64u - r)) : x;
}
constexpr uint64_t kMulHi = 2549297995355413924ull, kMulLo = 4865540595714422341ull;

// 32-bit values the generator will hand out, in order ([lo(o1), hi(o1),
// lo(o2), ...]: pcg64_next32 returns the low half of a fresh output and
// buffers the high half): nv / 2 outputs, lane l computes outputs l+1, l+33, ...
// by jumping 32 LCG steps at a time
__device__ void pcg_stream(uint32_t* v, int64_t nv, U128 s0, U128 inc, int lane,
                           uint64_t* sh_hi, uint64_t* sh_lo) {
  const U128 M{kMulHi, kMulLo};
  if (lane == 0) {  // states after 1..32 steps
    U128 st = s0;
    for (int l = 0; l < 32; ++l) {
      st = add128(mul128(st, M), inc);
      sh_hi[l] = st.hi;
      sh_lo[l] = st.lo;
    }
  }
  __syncwarp();
  U128 st{sh_hi[lane], sh_lo[lane]};
  U128 A = M, C = inc;  // (A, C) of 32 steps: s -> A s + C
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    C = add128(mul128(A, C), C);
    A = mul128(A, A);
  }
  for (int64_t o = lane; o < nv / 2; o += 32) {
    const uint64_t x = pcg_output(st);
    v[2 * o] = (uint32_t)x;
    v[2 * o + 1] = (uint32_t)(x >> 32);
    st = add128(mul128(A, st), C);
  }
  __syncwarp();
}

}  // namespace

// stream values allotted to a tail shuffle of nsteps draws: one per draw plus
// room for Lemire rejections (each costs one more value; expected count
// nsteps * pop / 2^32), rounded to whole warps of outputs
__host__ __device__ inline int64_t fill_stream_values(int64_t nsteps) {
  return ((nsteps + nsteps / 8 + 4096) + 63) / 64 * 64;
}

__global__ void __launch_bounds__(kRThreads) fill_random_kernel(
    int64_t* order_all, void* sel_all, int f64, int64_t out_stride, int64_t n, int64_t k,
    int64_t m1, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint32_t* scratch,
    int64_t scratch_words, int sequential) {
  __shared__ int64_t warp_tot[kRThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t* order = order_all + (int64_t)blockIdx.x * out_stride;
  const int64_t W = (n + 31) / 32;
  uint32_t* bitmap = scratch + (int64_t)blockIdx.x * scratch_words;
  uint32_t* zrank = bitmap + W;   // [W + 1]
  uint32_t* work = zrank + W + 1;  // tail: data[pop], drawn j [pop]; Floyd: hash set [mask + 1]
  const int64_t pop = n - k, size = m1 - k;
  const bool tail = pop > 10000 && size > pop / 50;
  uint64_t mask = 0;
  if (!tail) {  // smallest 2^b - 1 >= uint64(1.2 * size) (NumPy _gen_mask)
    mask = (uint64_t)(1.2 * (double)size);
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
  }

  // 1. bitmap of the picks, pool work array
  for (int64_t w = tid; w < W; w += kRThreads) bitmap[w] = 0u;
  if (tail)
    for (int64_t x = tid; x < pop; x += kRThreads) work[x] = (uint32_t)x;
  else
    for (int64_t x = tid; x <= (int64_t)mask; x += kRThreads) work[x] = 0xffffffffu;
  __syncthreads();
  for (int64_t i = tid; i < k; i += kRThreads) {
    const int64_t o = order[i];
    atomicOr(&bitmap[o >> 5], 1u << (o & 31));
  }
  __syncthreads();
  // zero bits before every word (contiguous word range per thread, block scan)
  {
    const int64_t wpt = (W + kRThreads - 1) / kRThreads;
    const int64_t w_lo = tid * wpt, w_hi = (w_lo + wpt) < W ? (w_lo + wpt) : W;
    uint32_t cnt = 0;
    for (int64_t w = w_lo; w < w_hi; ++w) {
      uint32_t f = ~bitmap[w];
      const int64_t valid = n - w * 32;
      if (valid < 32) f &= (1u << valid) - 1u;
      cnt += __popc(f);
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int64_t t = lane < kRThreads / 32 ? warp_tot[lane] : 0;
      int64_t ti = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, ti, o);
        if (lane >= o) ti += u;
      }
      if (lane < kRThreads / 32) warp_tot[lane] = ti - t;
    }
    __syncthreads();
    uint32_t run = (uint32_t)warp_tot[warp] + incl - cnt;
    for (int64_t w = w_lo; w < w_hi; ++w) {
      zrank[w] = run;
      uint32_t f = ~bitmap[w];
      const int64_t valid = n - w * 32;
      if (valid < 32) f &= (1u << valid) - 1u;
      run += __popc(f);
    }
    if (w_lo < W && w_hi == W) zrank[W] = run;
  }

  // 2. the generator: pool ranks into order[k, m1)
  int64_t* out = order + k;
  if (tail) {
    // tail partial Fisher-Yates: warp 0 produces the generator's values with
    // a 32-step jump-ahead per lane and maps them to the draws (Lemire's
    // rejections shift later draws by one value), then applies the swaps 32
    // steps at a time: all 64 loads in flight, the in-batch aliasing resolved by a scan
    // in step order (step b sees the slots written by steps a < b), one store
    // per slot by its last writer
    const int64_t first = (pop - size) > 1 ? (pop - size) : 1;
    const int64_t nsteps = pop - first;  // steps i = pop - 1, ..., first
    uint32_t* jarr = work + pop;          // [nsteps] drawn j of step t (i = pop - 1 - t)
    uint32_t* vstr = jarr + nsteps;       // [nv] the generator's 32-bit values
    const int64_t nv = fill_stream_values(nsteps);
    __shared__ uint64_t sh_hi[32], sh_lo[32];
    __shared__ int s_ovf;
    if (warp == 0 && sequential) {
      if (lane == 0) s_ovf = 1;  // test hook: the sequential generator below
    } else if (warp == 0) {
      pcg_stream(vstr, nv, U128{s_hi, s_lo}, U128{i_hi, i_lo}, lane, sh_hi, sh_lo);
      // draws -> values, 32 at a time: draw t takes value P + (t - t0) unless
      // an earlier draw of the batch was rejected; the first rejected draw is
      // redrawn by lane 0 and the next batch starts after it
      int64_t t0 = 0, P = 0;
      int ovf = 0;
      while (t0 < nsteps) {
        if (P + 32 > nv) {
          ovf = 1;
          break;
        }
        const int64_t t = t0 + lane;
        const bool live = t < nsteps;
        const uint32_t rng = live ? (uint32_t)(pop - 1 - t) : 1u, excl = rng + 1u;
        const uint64_t m = (uint64_t)vstr[P + lane] * excl;
        const uint32_t left = (uint32_t)m;
        bool rej = false;
        if (live && left < excl) rej = left < (0xffffffffu - rng) % excl;
        const unsigned rm = __ballot_sync(0xffffffffu, rej);
        const int f = rm ? __ffs(rm) - 1 : 32;
        if (live && lane < f) jarr[t] = (uint32_t)(m >> 32);
        if (f == 32) {
          t0 += 32;
          P += 32;
          continue;
        }
        int64_t p = P + f;
        if (lane == 0) {
          const uint32_t rf = (uint32_t)(pop - 1 - (t0 + f)), ef = rf + 1u;
          const uint32_t thr = (0xffffffffu - rf) % ef;
          uint64_t mm = 0;
          uint32_t lf = 0;
          do {
            ++p;
            if (p >= nv) break;
            mm = (uint64_t)vstr[p] * ef;
            lf = (uint32_t)mm;
          } while (lf < thr);
          if (p < nv) jarr[t0 + f] = (uint32_t)(mm >> 32);
        }
        p = __shfl_sync(0xffffffffu, p, 0);
        if (p >= nv) {
          ovf = 1;
          break;
        }
        t0 += f + 1;
        P = p + 1;
      }
      if (lane == 0) s_ovf = ovf;
    }
    __syncthreads();
    if (s_ovf && tid == 0) {  // more rejections than the stream allots: draw sequentially
      Pcg64 g{s_hi, s_lo, i_hi, i_lo, false, 0u};
      for (int64_t t = 0; t < nsteps; ++t) jarr[t] = g.bounded((uint32_t)(pop - 1 - t));
    }
    __syncthreads();
    if (warp == 0) {
      for (int64_t t0 = 0; t0 < nsteps; t0 += 32) {
        const int64_t t = t0 + lane;
        const bool live = t < nsteps;
        const uint32_t i = (uint32_t)(pop - 1 - (live ? t : 0));
        const uint32_t j = live ? jarr[t] : 0xffffffffu;
        uint32_t vj = live ? work[j] : 0u, vi = live ? work[i] : 0u;
#pragma unroll 4
        for (int a = 0; a < 31; ++a) {
          const uint32_t ja = __shfl_sync(0xffffffffu, j, a);
          const uint32_t wa = __shfl_sync(0xffffffffu, vi, a);  // value step a writes to slot ja
          if (lane > a) {
            if (j == ja) vj = wa;
            if (i == ja) vi = wa;
          }
        }
        if (live) out[i - (pop - size)] = vj;  // step: out = data[j]; data[j] = data[i]
        const unsigned same = __match_any_sync(0xffffffffu, j);
        if (live && lane == 31 - __clz(same)) work[j] = vi;
        __syncwarp();
      }
      if (lane == 0 && first > pop - size) out[0] = work[0];  // pop == size: slot 0 stays
    }
  } else if (tid == 0) {
    Pcg64 g{s_hi, s_lo, i_hi, i_lo, false, 0u};
    {
      // Floyd's algorithm, hash set of mask + 1 slots (empty = 0xffffffff)
      for (int64_t j = pop - size; j < pop; ++j) {
        const uint32_t val = g.bounded((uint32_t)j);
        uint64_t loc = val & mask;
        while (work[loc] != 0xffffffffu && work[loc] != val) loc = (loc + 1) & mask;
        if (work[loc] == 0xffffffffu) {
          work[loc] = val;
          out[j - pop + size] = val;
        } else {
          loc = (uint64_t)j & mask;
          while (work[loc] != 0xffffffffu) loc = (loc + 1) & mask;
          work[loc] = (uint32_t)j;
          out[j - pop + size] = j;
        }
      }
      for (int64_t i = size - 1; i >= 1; --i) {  // _shuffle_int(size, 1, picks)
        const uint32_t j = g.bounded((uint32_t)i);
        const int64_t t = out[j];
        out[j] = out[i];
        out[i] = t;
      }
    }
  }
  __syncthreads();

  // 3. pool ranks -> cloud indices; fill entries carry selection distance 0
  for (int64_t x = tid; x < size; x += kRThreads) {
    const uint32_t r = (uint32_t)order[k + x];
    int64_t lo = 0, hi = W - 1;  // largest w with zrank[w] <= r
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (zrank[mid] <= r) lo = mid;
      else hi = mid - 1;
    }
    uint32_t f = ~bitmap[lo];
    const int64_t valid = n - lo * 32;
    if (valid < 32) f &= (1u << valid) - 1u;
    order[k + x] = lo * 32 + (int64_t)__fns(f, 0u, (int)(r - zrank[lo]) + 1);
  }
  if (f64) {
    double* sel = static_cast<double*>(sel_all) + (int64_t)blockIdx.x * out_stride;
    for (int64_t i = tid; i < size; i += kRThreads) sel[k + i] = 0.0;
  } else {
    float* sel = static_cast<float*>(sel_all) + (int64_t)blockIdx.x * out_stride;
    for (int64_t i = tid; i < size; i += kRThreads) sel[k + i] = 0.0f;
  }
}

int64_t fill_random_scratch_words(int64_t n, int64_t k, int64_t m1) {
  const int64_t W = (n + 31) / 32, pop = n - k, size = m1 - k;
  const int64_t nsteps = pop - ((pop - size) > 1 ? (pop - size) : 1);
  int64_t work = pop + nsteps + fill_stream_values(nsteps);  // data, drawn j, values
  if (!(pop > 10000 && size > pop / 50)) {
    uint64_t mask = (uint64_t)(1.2 * (double)size);
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    work = (int64_t)mask + 1;
  }
  return ((W + W + 1 + work) + 31) / 32 * 32;  // 128-B aligned per cloud
}

cudaError_t launch_fill_random(int dtype, int64_t* order, void* sel_d2, int64_t batch,
                               int64_t out_stride, int64_t n, int64_t k, int64_t m1,
                               const uint64_t pcg[4], uint32_t* scratch, cudaStream_t st,
                               bool sequential) {
  if (m1 - k <= 0 || batch <= 0) return cudaSuccess;
  fill_random_kernel<<<(unsigned)batch, kRThreads, 0, st>>>(
      order, sel_d2, dtype == 1, out_stride, n, k, m1, pcg[0], pcg[1], pcg[2], pcg[3], scratch,
      fill_random_scratch_words(n, k, m1), sequential ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace ffps
