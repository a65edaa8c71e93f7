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

// Bounds checks of shared- and global-memory indexing, compiled in only for a checking build
// (-DEDKM_BOUNDS, tools/bounds_check.sh): a failed check is a device assert.  The pool's
// compute-sanitizer is closed since the round-2 table changes; this is the substitute.
#ifdef EDKM_BOUNDS
#include <cassert>
#define EDKM_BCHECK(c) assert(c)
#else
#define EDKM_BCHECK(c) ((void)0)
#endif

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
  int64_t peer_delta;         // F1, NVLS emulate with a peer: byte offset of the peer's copy (0: none)
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

// Warp-parallel choice of the `cap` consecutive magnitude pages (of kMagPages = 128) with the
// largest total mass: lane l holds the masses of pages l, l+32, l+64, l+96 in m[0..3].  Returns
// (in every lane) the smallest start b maximising sum(mass[b .. b+cap)) and that sum in `best`
// -- the same window as a serial sliding-window scan that keeps the first maximum.  Called by
// one full warp; replaces a 128-step loop on one lane (~3 us of shared-memory latency per
// segment, paid by every per-weight kernel).
template <class T>
__device__ __forceinline__ int warp_best_window(const T (&m)[4], int cap, T& best) {
  const int lane = threadIdx.x & 31;
  // prefix sums in page order: page p = lane + 32 q; exclusive prefix over all pages
  T pre[4];  // mass of pages < lane + 32 q
  T carry = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    T inc = m[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    pre[q] = carry + inc - m[q];
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  // window starting at page b = lane + 32 q: prefix(b + cap) - prefix(b); prefix(128) = carry
  T bw = -1;
  int bs = 1 << 30;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int b = lane + 32 * q, e = b + cap;  // prefix(e) lives in lane e % 32, slot e / 32
    T pe = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const T x = __shfl_sync(0xffffffffu, pre[r], e & 31);
      if ((e >> 5) == r) pe = x;
    }
    if (e == kMagPages) pe = carry;
    if (e <= kMagPages) {
      const T w = pe - pre[q];
      if (w > bw) { bw = w; bs = b; }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const T ow = __shfl_xor_sync(0xffffffffu, bw, o);
    const int ob = __shfl_xor_sync(0xffffffffu, bs, o);
    if (ow > bw || (ow == bw && ob < bs)) { bw = ow; bs = ob; }
  }
  best = bw;
  return bs;
}

// ---------------------------------------------------------------- magnitude-page window
// page_cnt[256] (int64, weights per signed page u>>8, every present pattern) is written by the
// forward table kernel, which then chooses, once per tensor, the np <= cap consecutive
// magnitude pages [pbase, pbase+np) that the per-weight kernels keep in shared memory (both
// signs); patterns outside take a slower path.  Called by one full warp; every lane gets the
// result.  The window is the whole populated span when it fits in cap pages; otherwise the
// narrowest window that still holds all but ~1e-6 of the weights (a 16-vector with a pattern
// outside it takes the slow path, so that tail must be rare, while every page kept costs
// shared-memory set-up, staging and flushing in each segment of each per-weight kernel).
__device__ __forceinline__ void choose_window(const int64_t* page_cnt, int cap, int& pbase, int& np) {
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
  if (pmax < 0) { pbase = 0; np = 1; return; }  // keep np >= 1
  if (pmax - pmin + 1 <= cap) { pbase = pmin; np = pmax - pmin + 1; return; }
  int64_t tot = m[0] + m[1] + m[2] + m[3];
#pragma unroll
  for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  const int64_t need = tot - (tot >> 20);
  int64_t best;
  int lo = 1, hi = cap;  // smallest width whose best window reaches `need` (cap if none)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    warp_best_window(m, mid, best);
    if (best >= need) hi = mid; else lo = mid + 1;
  }
  pbase = warp_best_window(m, lo, best);
  np = lo;
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

namespace edkm {
// ---------------------------------------------------------------- shared-memory primitives (32-bit addresses)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_shared(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
  float2 r;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "r"(a));
  return r;
}

// Fast-path window addressing: the window holds every present pattern, so the
// shared address of pattern u is offP/offN + (u & 0x7FFF) * ES with no range
// check.  The clamp keeps a caller who breaks the contract (weights differing
// from those counted) inside the table: wrong values, never a stray write.
template <int ES>
struct FastWin {
  uint32_t offP, offN, lo, hi;
  __device__ void init(uint32_t base, int pbase, int np) {
    offP = base - (uint32_t)pbase * 256u * ES;
    offN = offP + (uint32_t)np * 256u * ES;
    lo = base;
    hi = base + (uint32_t)(2 * np * 256 - 1) * ES;
  }
  __device__ __forceinline__ uint32_t addr(uint32_t u) const {  // u: 16-bit pattern in the low half
    const uint32_t a = ((u & 0x8000u) ? offN : offP) + (u & 0x7FFFu) * ES;
    return min(max(a, lo), hi);
  }
};
}  // namespace edkm

namespace edkm {
// ---------------------------------------------------------------- windowed per-pattern lookups (predicated, no branch)
// Window of np magnitude pages from pbase: pattern u is in it iff
// rel = (u & 0x7FFF) - pbase*256 < np*256 (unsigned); its slot is rel in the
// positive half (u < 0x8000) or np*256 + rel in the negative half.
struct Win {
  uint32_t pb256, np256, baseP, baseN;  // baseP/baseN: shared byte address of slot 0 of each half
  template <int ES>
  __device__ void init(uint32_t base, int pbase, int np) {
    pb256 = (uint32_t)pbase << 8;
    np256 = (uint32_t)np << 8;
    baseP = base;
    baseN = base + np256 * ES;
  }
  __device__ __forceinline__ uint32_t rel(uint32_t u) const { return (u & 0x7FFFu) - pb256; }
  template <int ES>
  __device__ __forceinline__ uint32_t saddr(uint32_t u, uint32_t r) const { return ((u & 0x8000u) ? baseN : baseP) + r * ES; }
};

// Exact 64-bit fixed-point add into the shared bucket at saddr (lo u32) / saddr+HI_OFF (hi i32):
// lo += q; the lane whose add carried out of (or borrowed from) lo moves +-1 into hi.
template <uint32_t HI_OFF>
__device__ __forceinline__ void fixed_add(uint32_t saddr, int q) {
  asm volatile(
      "{\n\t.reg .pred c, n, f;\n\t.reg .u32 old, nw, d;\n\t"
      "atom.shared.add.u32 old, [%0], %1;\n\t"
      "add.u32 nw, old, %1;\n\t"
      "setp.lt.u32 c, nw, old;\n\t"
      "setp.lt.s32 n, %1, 0;\n\t"
      "xor.pred f, c, n;\n\t"
      "selp.u32 d, 1, 0xFFFFFFFF, c;\n\t"
      "@f red.shared.add.u32 [%0+%2], d;\n\t}"
      ::"r"(saddr), "r"(q), "n"(HI_OFF)
      : "memory");
}

// The same add in two halves so a thread can have many lo atomics in flight before it looks
// at any return value: fixed_lo issues lo += q, fixed_carry applies the carry/borrow.
__device__ __forceinline__ uint32_t fixed_lo(uint32_t saddr, int q) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(saddr), "r"(q));
  return old;
}
template <uint32_t HI_OFF>
__device__ __forceinline__ void fixed_carry(uint32_t saddr, int q, uint32_t old) {
  asm volatile(
      "{\n\t.reg .pred c, n, f;\n\t.reg .u32 nw, d;\n\t"
      "add.u32 nw, %1, %2;\n\t"
      "setp.lt.u32 c, nw, %1;\n\t"
      "setp.lt.s32 n, %2, 0;\n\t"
      "xor.pred f, c, n;\n\t"
      "selp.u32 d, 1, 0xFFFFFFFF, c;\n\t"
      "@f red.shared.add.u32 [%0+%3], d;\n\t}"
      ::"r"(saddr), "r"(old), "r"(q), "n"(HI_OFF));
}

// ---------------------------------------------------------------- TMA staging of per-pattern tables
// The per-segment tables (W~ table, index table, (phi, psi) window) are copied global -> shared
// by the bulk-copy engine (cp.async.bulk, completion counted in bytes on an mbarrier) instead of
// by the 1024 threads: one elected thread issues the copies, every thread waits on the phase.
struct TmaTable {
  uint64_t* bar;   // shared mbarrier (arrival count 1)
  uint32_t phase;  // parity of the next completion (uniform across the CTA)
  // called by every thread once per kernel, before the first stage()
  __device__ void init(uint64_t* b) {
    bar = b;
    phase = 0;
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(b)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
  }
  // Copy up to two contiguous global ranges into shared memory (bytes multiples of 16, both
  // addresses 16-byte aligned; the caller checks and otherwise uses plain loads) and wait.
  // Must be entered by every thread after a barrier that ended all reads of `dst0`/`dst1`.
  __device__ void stage(void* dst0, const void* src0, uint32_t bytes0, void* dst1 = nullptr,
                        const void* src1 = nullptr, uint32_t bytes1 = 0) {
    if (threadIdx.x == 0) {
      // the generic-proxy reads of the previous segment's table precede these async-proxy writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                   "r"(bytes0 + bytes1)
                   : "memory");
      copy(dst0, src0, bytes0);
      if (bytes1) copy(dst1, src1, bytes1);
    }
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TMA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TMA_WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
    phase ^= 1u;
  }
  __device__ void copy(void* dst, const void* src, uint32_t bytes) {
    constexpr uint32_t kPiece = 32768;
    for (uint32_t o = 0; o < bytes; o += kPiece) {
      const uint32_t n = bytes - o < kPiece ? bytes - o : kPiece;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_addr(dst) + o),
                   "l"((const char*)src + o), "r"(n), "r"(smem_addr(bar))
                   : "memory");
    }
  }
  static __device__ __forceinline__ bool aligned(const void* p) { return ((uintptr_t)p & 15u) == 0; }
};

// (phi, psi) of a pattern: shared window when `in` != 0, else the global table
// entry gtab[u] (its address is formed inside the predicated block).
__device__ __forceinline__ float2 lookup_f2(uint32_t in, uint32_t saddr, const float2* gtab, uint32_t u) {
  float2 r;
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .u64 ga;\n\tsetp.ne.u32 p, %2, 0;\n\t"
      "@p ld.shared.v2.f32 {%0, %1}, [%3];\n\t"
      "@!p mad.wide.u32 ga, %5, 8, %4;\n\t"
      "@!p ld.global.nc.v2.f32 {%0, %1}, [ga];\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "r"(in), "r"(saddr), "l"(gtab), "r"(u));
  return r;
}

// Exact 64-bit fixed-point bucket add: when `in` != 0, lo[slot] += q with the
// carry/borrow into hi[slot] (at saddr + HI_OFF) done by the lane that made it;
// otherwise the fp64 global bucket gB[u] gets g.  Predicated, no branch.
template <uint32_t HI_OFF>
__device__ __forceinline__ void bucket_add(uint32_t in, uint32_t saddr, int q, double* gB, uint32_t u, float g) {
  asm volatile(
      "{\n\t.reg .pred p, c, n, f;\n\t.reg .u32 old, nw, d;\n\t.reg .f64 gd;\n\t.reg .u64 ga;\n\t"
      "setp.ne.u32 p, %0, 0;\n\t"
      "mov.u32 old, 0;\n\t"
      "@p atom.shared.add.u32 old, [%1], %2;\n\t"
      "add.u32 nw, old, %2;\n\t"
      "setp.lt.u32 c, nw, old;\n\t"
      "setp.lt.s32 n, %2, 0;\n\t"
      "xor.pred f, c, n;\n\t"
      "and.pred f, f, p;\n\t"
      "selp.u32 d, 1, 0xFFFFFFFF, c;\n\t"
      "@f red.shared.add.u32 [%1+%6], d;\n\t"
      "@!p cvt.f64.f32 gd, %3;\n\t"
      "@!p mad.wide.u32 ga, %5, 8, %4;\n\t"
      "@!p red.global.add.f64 [ga], gd;\n\t}"
      ::"r"(in), "r"(saddr), "r"(q), "f"(g), "l"(gB), "r"(u), "n"(HI_OFF)
      : "memory");
}
}  // namespace edkm
