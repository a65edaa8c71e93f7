// common.cuh -- shared device helpers of libedkm (sm_100a only).
//
// Layout conventions:
//   * A weight tensor is n 16-bit patterns; pattern u in [0, 65536) is the
//     index of the weight in the attention table (P:77, P:83 S2.2).
//   * Per-pattern tables are [nt][65536] arrays indexed by the pattern.
//   * The "magnitude page" of a pattern is (u >> 8) & 0x7F: 256 consecutive
//     patterns of one sign.  Per-weight kernels keep a window of np magnitude
//     pages (both signs) of a per-pattern table in shared memory; patterns
//     outside the window fall back to global memory (correct, slower).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace edkm {

constexpr int kPatterns = 65536;
constexpr int kMaxTensorsPerLaunch = 512;
constexpr int kMagPages = 128;

enum WDtype : int { kBF16 = 0, kFP16 = 1, kFP32 = 2, kU8 = 3 };

// ---------------------------------------------------------------- decoding
// Exact value of a 16-bit pattern ("16bit (e.g., BF16 or FP16)").
__device__ __forceinline__ double decode16(uint32_t u, int wdtype) {
  if (wdtype == kBF16) return (double)__uint_as_float(u << 16);
  return (double)__half2float(__ushort_as_half((unsigned short)u));
}
__device__ __forceinline__ float decode16f(uint32_t u, int wdtype) {
  if (wdtype == kBF16) return __uint_as_float(u << 16);
  return __half2float(__ushort_as_half((unsigned short)u));
}
// NaN/Inf patterns are counted but excluded from clustering (DESIGN R10).
__host__ __device__ __forceinline__ bool pattern_finite(uint32_t u, int wdtype) {
  return wdtype == kBF16 ? ((u & 0x7F80u) != 0x7F80u) : ((u & 0x7C00u) != 0x7C00u);
}
__device__ __forceinline__ uint16_t round16(double x, int wdtype) {
  if (wdtype == kBF16) return __bfloat16_as_ushort(__double2bfloat16(x));
  return __half_as_ushort(__double2half(x));
}
__device__ __forceinline__ uint16_t round16f(float x, int wdtype) {
  if (wdtype == kBF16) return __bfloat16_as_ushort(__float2bfloat16_rn(x));
  return __half_as_ushort(__float2half_rn(x));
}
__host__ __device__ __forceinline__ uint16_t nan16(int wdtype) { return wdtype == kBF16 ? 0x7FC0 : 0x7E00; }

// ---------------------------------------------------------------- streaming memory access
// 256-bit loads with an L2 evict-first hint: the weights/gradients are read
// once per pass and must not evict the per-pattern tables from L2.
struct V8 { uint32_t x[8]; };

__device__ __forceinline__ V8 ldg_stream8(const void* p) {
  V8 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.x[0]), "=r"(r.x[1]), "=r"(r.x[2]), "=r"(r.x[3]), "=r"(r.x[4]), "=r"(r.x[5]),
                 "=r"(r.x[6]), "=r"(r.x[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_stream8(void* p, const V8& v) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.x[0]),
               "r"(v.x[1]), "r"(v.x[2]), "r"(v.x[3]), "r"(v.x[4]), "r"(v.x[5]), "r"(v.x[6]), "r"(v.x[7])
               : "memory");
}
__device__ __forceinline__ void stg_stream4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void red_shared_add(uint32_t* addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(addr)), "r"(v) : "memory");
}

// ---------------------------------------------------------------- per-launch tensor lists
// Passed by value as kernel parameters (< 32 KB), so a launch needs no host->device copy.
struct StreamArgs {
  int nt;                     // tensors in this launch
  int t0;                     // index of the first tensor in the caller's [nt] arrays
  int wdtype;                 // kBF16 / kFP16
  int gdtype;                 // gradient dtype (kBF16/kFP16/kFP32) for B1/B2
  int odtype;                 // output dtype for F2/B2
  int mode;                   // F2 mode
  int64_t total;              // sum of n
  int64_t offs[kMaxTensorsPerLaunch + 1];
  const uint16_t* w[kMaxTensorsPerLaunch];
  const void* g[kMaxTensorsPerLaunch];
  void* out[kMaxTensorsPerLaunch];
};

// Static contiguous split of the concatenated element space over the grid,
// rounded to 512 elements so CTA boundaries inside a tensor stay vector-aligned.
__device__ __forceinline__ void cta_range(int64_t total, int64_t& lo, int64_t& hi) {
  const int64_t G = gridDim.x, c = blockIdx.x;
  const int64_t units = (total + 511) / 512;
  lo = (units * c / G) * 512;
  hi = (units * (c + 1) / G) * 512;
  if (lo > total) lo = total;
  if (hi > total) hi = total;
}

__device__ __forceinline__ int find_tensor(const StreamArgs& A, int64_t e) {
  int lo = 0, hi = A.nt;  // largest t with offs[t] <= e
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (A.offs[mid] <= e) lo = mid; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------- magnitude-page window
// page_cnt[256] (int64, per signed page u>>8, finite populated patterns only) is
// written by the forward table kernel.  Choose np <= cap consecutive magnitude
// pages [pbase, pbase+np) that hold the most weights.  Called by one warp.
__device__ __forceinline__ void choose_window(const int64_t* page_cnt, int cap, int* out_base, int* out_np) {
  const int lane = threadIdx.x & 31;
  // masses of magnitude pages lane, lane+32, lane+64, lane+96
  int64_t m[4];
  int pmin = 1 << 30, pmax = -1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int p = lane + 32 * q;
    m[q] = page_cnt[p] + page_cnt[p + 128];
    if (m[q] > 0) { pmin = min(pmin, p); pmax = max(pmax, p); }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    pmin = min(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
    pmax = max(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
  }
  if (pmax < 0) { *out_base = 0; *out_np = 0; return; }
  if (pmax - pmin + 1 <= cap) { *out_base = pmin; *out_np = pmax - pmin + 1; return; }
  // sliding window of `cap` pages maximising the mass (lane 0, 128 steps)
  __shared__ int64_t s_mass[kMagPages];
#pragma unroll
  for (int q = 0; q < 4; ++q) s_mass[lane + 32 * q] = m[q];
  __syncwarp();
  if (lane == 0) {
    int64_t cur = 0;
    for (int p = 0; p < cap; ++p) cur += s_mass[p];
    int64_t best = cur;
    int bb = 0;
    for (int p = cap; p < kMagPages; ++p) {
      cur += s_mass[p] - s_mass[p - cap];
      if (cur > best) { best = cur; bb = p - cap + 1; }
    }
    *out_base = bb;
    *out_np = cap;
  }
  __syncwarp();
}

// slot of pattern u in a window, or -1
__device__ __forceinline__ int window_slot(uint32_t u, int pbase, int np) {
  const uint32_t rel = ((u >> 8) & 0x7Fu) - (uint32_t)pbase;
  if (rel >= (uint32_t)np) return -1;
  return (int)((((u >> 15) * (uint32_t)np + rel) << 8) | (u & 0xFFu));
}
__device__ __forceinline__ uint32_t slot_pattern(int slot, int pbase, int np) {
  const uint32_t page = (uint32_t)slot >> 8, sign = page / (uint32_t)np, rel = page - sign * (uint32_t)np;
  return (sign << 15) | ((rel + (uint32_t)pbase) << 8) | ((uint32_t)slot & 0xFFu);
}

}  // namespace edkm
