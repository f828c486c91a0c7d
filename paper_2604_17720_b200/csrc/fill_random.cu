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
//   2. thread 0 runs the generator; the tail shuffle works on a window of
//      kWin steps (8: larger windows thrash the instruction cache): draws
//      first, then all 2 * kWin loads in flight, aliasing
//      inside the window resolved in registers, then the stores (the only
//      reads a step can see from earlier steps of the window are the slots
//      they wrote, j_a == j_b or j_a == i_b);
//   3. all threads map the drawn pool ranks to cloud indices (binary search of
//      the word prefix, then the rank-th zero bit of the word).
#include <cuda_runtime.h>

#include <cstdint>

#include "ffps_internal.h"

namespace ffps {

namespace {

constexpr int kRThreads = 512;
#ifndef FFPS_FILL_WIN
#define FFPS_FILL_WIN 8
#endif
constexpr int kWin = FFPS_FILL_WIN;  // tail shuffle: steps per window

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
#ifdef FFPS_FILL_NOINLINE
  __device__ __noinline__ uint32_t bounded(uint32_t rng) {
#else
  __device__ uint32_t bounded(uint32_t rng) {
#endif
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

}  // namespace

__global__ void __launch_bounds__(kRThreads) fill_random_kernel(
    int64_t* order_all, void* sel_all, int f64, int64_t out_stride, int64_t n, int64_t k,
    int64_t m1, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, uint32_t* scratch,
    int64_t scratch_words) {
  __shared__ int64_t warp_tot[kRThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t* order = order_all + (int64_t)blockIdx.x * out_stride;
  const int64_t W = (n + 31) / 32;
  uint32_t* bitmap = scratch + (int64_t)blockIdx.x * scratch_words;
  uint32_t* zrank = bitmap + W;   // [W + 1]
  uint32_t* work = zrank + W + 1;  // tail: data[pop]; Floyd: hash set [mask + 1]
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

  // 2. the generator (thread 0): pool ranks into order[k, m1)
  if (tid == 0) {
    Pcg64 g{s_hi, s_lo, i_hi, i_lo, false, 0u};
    int64_t* out = order + k;
    if (tail) {
      const int64_t first = (pop - size) > 1 ? (pop - size) : 1;
      for (int64_t i0 = pop - 1; i0 >= first; i0 -= kWin) {
        const int cnt = (i0 - first + 1) < kWin ? (int)(i0 - first + 1) : kWin;
        uint32_t iu[kWin], ju[kWin], vj[kWin], vi[kWin];
#pragma unroll
        for (int u = 0; u < kWin; ++u) {
          iu[u] = (uint32_t)(i0 - u);
          ju[u] = u < cnt ? g.bounded(iu[u]) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kWin; ++u) {
          vj[u] = u < cnt ? work[ju[u]] : 0u;
          vi[u] = u < cnt ? work[iu[u]] : 0u;
        }
#pragma unroll
        for (int b = 0; b < kWin; ++b) {
#pragma unroll
          for (int a = 0; a < b; ++a) {  // slots written earlier in the window
            if (ju[a] == ju[b]) vj[b] = vi[a];
            if (ju[a] == iu[b]) vi[b] = vi[a];
          }
          // step b: out = data[j]; data[j] = data[i] (vi[b] now holds the value
          // written to slot j_b, read by later steps through the checks above)
          const uint32_t o = vj[b];
          if (b < cnt) out[iu[b] - (pop - size)] = o;
        }
#pragma unroll
        for (int b = 0; b < kWin; ++b)
          if (b < cnt) work[ju[b]] = vi[b];
      }
      if (first > pop - size) out[0] = work[0];  // pop == size: slot 0 keeps its value
    } else {
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
  int64_t work = pop;
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
                               const uint64_t pcg[4], uint32_t* scratch, cudaStream_t st) {
  if (m1 - k <= 0 || batch <= 0) return cudaSuccess;
  fill_random_kernel<<<(unsigned)batch, kRThreads, 0, st>>>(
      order, sel_d2, dtype == 1, out_stride, n, k, m1, pcg[0], pcg[1], pcg[2], pcg[3], scratch,
      fill_random_scratch_words(n, k, m1));
  return cudaGetLastError();
}

}  // namespace ffps
