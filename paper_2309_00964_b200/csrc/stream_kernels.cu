// stream_kernels.cu -- the four per-weight passes of the eDKM hot path (S3).
//
//   F1  uniquify: counts[u] = #{i : bits(w_i) = u}            (Fig. 3)
//   F2  reconstruct: W~_i = table[bits(w_i)] (or hard modes)    (Fig. 1, "look-up")
//   B1  gradient buckets: B[u] = sum_{bits(w_i)=u} G_i          (DESIGN App. A)
//   B2  dW_i = G_i phi[bits(w_i)] + psi[bits(w_i)]               (DESIGN App. A)
//
// All four are HBM-streaming kernels: persistent grid (one 1024-thread CTA per
// SM, its shared memory holding one tensor's per-pattern table), a static
// contiguous split of the concatenated weight space, 256-bit evict-first loads,
// and the per-pattern table in shared memory.  No tensor cores: nothing here
// is a contraction.
#include <cstdio>

#include "common.cuh"
#include "launch.h"

namespace edkm {

constexpr int kThreads = 1024;   // F1, F2

constexpr int kF1Bins = 57344;  // patterns < 0xE000 counted in SMEM (224 KiB); the rest in L2
constexpr int kB1Pages = kWinPagesB;    // magnitude pages per sign kept by B1 (8 B/pattern)
constexpr int kB2Pages = kWinPagesB;    // B2 (float2 phi, psi)
constexpr int kF2Pages32 = kWinPagesF2; // F2 fp32 output (4 B/pattern)

// ----------------------------------------------------------------------------
// Generic visitor over this CTA's slice of the concatenated tensors.
// P::Vec is the register payload of one 16-element vector; vectors are
// processed two at a time so each thread keeps 2 x 32 B (or more) in flight.
// ----------------------------------------------------------------------------
template <class P>
__device__ __forceinline__ void for_each_segment(const StreamArgs& A, P& p) {
  int64_t lo, hi;
  cta_range(A.total, lo, hi);
  if (lo >= hi) return;
  int t = find_tensor(A, lo);
  const int tid = threadIdx.x, bs = blockDim.x;
  while (lo < hi) {
    while (A.offs[t + 1] <= lo) ++t;
    const int64_t a = lo - A.offs[t], b = min(hi, A.offs[t + 1]) - A.offs[t];
    p.begin(t, a, b);
    const uintptr_t wa = (uintptr_t)(A.w[t] + a);
    int64_t head = min((int64_t)(((32u - (uint32_t)(wa & 31u)) & 31u) >> 1), b - a);
    const int64_t va = a + head;
    int64_t nv = (b - va) >> 4;
    if (nv > 0 && !p.vec_ok(t, va)) { head = b - a; nv = 0; }
    for (int64_t i = a + tid; i < a + head; i += bs) p.scalar(t, i);
    int64_t v = tid;
    if (P::kLoop == 0) {
      // one vector per iteration: lowest register use, 1024 threads keep enough loads in flight
#pragma unroll 1
      for (; v < nv; v += bs) {
        typename P::Vec r0;
        p.load(t, va + 16 * v, r0);
        p.process(t, va + 16 * v, r0);
      }
    } else if (P::kLoop == 2) {
      // software pipeline: the next vector's loads are in flight while this one is processed
      typename P::Vec cur, nxt;
      if (v < nv) p.load(t, va + 16 * v, cur);
      for (; v < nv; v += bs) {
        const bool more = v + bs < nv;
        if (more) p.load(t, va + 16 * (v + bs), nxt);
        p.process(t, va + 16 * v, cur);
        if (more) cur = nxt;
      }
    } else {
      for (; v + bs < nv; v += 2 * bs) {
        typename P::Vec r0, r1;
        p.load(t, va + 16 * v, r0);
        p.load(t, va + 16 * (v + bs), r1);
        p.process(t, va + 16 * v, r0);
        p.process(t, va + 16 * (v + bs), r1);
      }
      if (v < nv) {
        typename P::Vec r0;
        p.load(t, va + 16 * v, r0);
        p.process(t, va + 16 * v, r0);
      }
    }
    for (int64_t i = va + 16 * nv + tid; i < b; i += bs) p.scalar(t, i);
    p.end(t);
    lo = A.offs[t] + b;
    ++t;
  }
}

__device__ __forceinline__ uint32_t pat(const V8& v, int e) { return (v.x[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu; }

// ============================================================================ F1
// Adds to the global counts: a plain L2 atomic, or (MC, NVLS mode) a multimem reduction on the
// multicast address of a symmetric buffer -- the NVSwitch adds v into every rank's copy, so the
// cross-rank sum of the counts happens inside F1's own flushes, with no separate collective.
// MC = 0: plain; 1: NVLS multicast; 2: the same protocol on ordinary memory (tests): the add goes
// to this rank's copy and, with a peer (peer != 0: byte offset of the peer's copy mapped by CUDA
// IPC), to the peer's copy too -- what the switch does for every rank's copy.
template <int MC>
__device__ __forceinline__ void cnt_add(int32_t* p, int v, int64_t peer = 0) {
  if (MC == 1) {
    asm volatile("multimem.red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  } else {
    atomicAdd(p, v);
    if (MC == 2 && peer) atomicAdd_system(reinterpret_cast<int32_t*>(reinterpret_cast<char*>(p) + peer), v);
  }
}

template <int MC>
struct F1Policy {
  static constexpr int kLoop = 1;  // two vectors per iteration (F1 is atomic-bound: more loads in flight)
  const StreamArgs& A;
  uint32_t* h;
  int32_t* counts;  // [nt_total][65536], this launch's tensors start at t0
  struct Vec { V8 w; };
  __device__ int32_t* cnt(int t) const { return counts + (int64_t)(A.t0 + t) * kPatterns; }
  __device__ void begin(int, int64_t, int64_t) {
    uint4* h4 = reinterpret_cast<uint4*>(h);
    for (int i = threadIdx.x; i < kF1Bins / 4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
  }
  __device__ bool vec_ok(int, int64_t) const { return true; }
  __device__ void load(int t, int64_t i, Vec& r) const { r.w = ldg_stream8(A.w[t] + i); }
  __device__ void count(int t, uint32_t u) {
    if (u < (uint32_t)kF1Bins) red_shared_add(&h[u], 1u);
    else cnt_add<MC>(&cnt(t)[u], 1, A.peer_delta);
  }
  __device__ void process(int t, int64_t, const Vec& r) {
#pragma unroll
    for (int e = 0; e < 16; ++e) count(t, pat(r.w, e));
  }
  __device__ void scalar(int t, int64_t i) { count(t, A.w[t][i]); }
  __device__ void end(int t) {
    __syncthreads();
    int32_t* c = cnt(t);
    for (int i = threadIdx.x; i < kF1Bins; i += blockDim.x) {
      const uint32_t v = h[i];
      if (v) cnt_add<MC>(&c[i], (int32_t)v, A.peer_delta);
    }
    __syncthreads();
  }
};

// ---------------------------------------------------------------------------- F1, lane-private
// One shared counter array makes F1 bound by shared-memory bank conflicts, not HBM: the 32
// random patterns of a warp's atomic land on the 32 banks like balls in bins (~3.8 wavefronts
// per instruction, S4).  Here every lane owns a private copy of the counters that
// lies entirely in its own bank (word = row * 32 + lane), so a warp's 32 atomics always hit 32
// distinct banks: one wavefront per instruction.  32 copies fit for a window of kF1LPages
// magnitude pages: word `row` = rel of a pattern (u & 0x7FFF) - pbase*256 counts both signs
// (word = P + 0xFF01 * N, see kF1NegInc).  A copy is shared by the 32 threads with the same
// lane id, so after 32 x kF1LChunkVec x 16 < 0xFF01 increments the copies are folded
// into per-thread 32-bit accumulators (each thread owns rows tid and tid + 1024) and zeroed.
// The window is chosen per segment from a sample; bf16 N(0, 0.02^2) keeps ~99.9% of the weights
// in it (patterns outside go to global atomics).  A segment whose sample is not covered well
// (fp16, whose pages are quarter binades, or unusual data) takes the shared-array path.
constexpr int kF1LPages = 7;
constexpr int kF1LRows = kF1LPages * 256;  // 1792 words per copy, 32 copies = 224 KiB
// vectors per thread between folds (32*127*16 < 65536); measured: 4x fewer folds would save
// only ~3% of F1, not worth an unsafe bound
constexpr int kF1LChunkVec = 127;
// patterns sampled per segment to place the window (4 per thread, one round of loads; 16K
// measured ~3% slower on CFG2's F1 and no better a window)
constexpr int kF1Sample = 4096;
// Lane-private counter word = P + kF1NegInc * N (P, N: counts of the positive and negative
// pattern of the row since the last fold, P + N <= 32 * kF1LChunkVec * 16 = 65024 < kF1NegInc,
// so the word is < 2^32 and decodes exactly).  The increment 1 or 0xFF01 is one PRMT.
constexpr uint32_t kF1NegInc = 0xFF01u;
static_assert(32u * kF1LChunkVec * 16u < kF1NegInc, "F1 lane-private counter decoding");
// dynamic shared memory of F1: the shared-array path's counters, or the lane-private copies
// plus one trash row (never folded) that absorbs the increments of patterns outside the window
constexpr size_t kF1Smem = (size_t)(kF1LRows + 1) * 128 > (size_t)kF1Bins * 4
                               ? (size_t)(kF1LRows + 1) * 128 : (size_t)kF1Bins * 4;

template <int MC>
__device__ __forceinline__ void f1_count_global(int32_t* c, uint32_t u, int64_t peer) { cnt_add<MC>(&c[u], 1, peer); }

// fold the 32 copies of rows tid and tid+1024 into acc (pos, neg per row) and zero them
__device__ __forceinline__ void f1l_fold(uint32_t* h, uint32_t acc[4]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int r = tid + j * 1024;
    if (r < kF1LRows) {
      uint4* row = reinterpret_cast<uint4*>(h + r * 32);
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int q = (tid + s) & 7;  // diagonal: the 8 threads of a quarter warp read 8 distinct bank groups
        const uint4 x = row[q];
        // word = P + kF1NegInc * N with P + N <= 65024 < kF1NegInc: N = word / kF1NegInc exactly
        const uint32_t n0 = x.x / kF1NegInc, n1 = x.y / kF1NegInc, n2 = x.z / kF1NegInc, n3 = x.w / kF1NegInc;
        hi += n0 + n1 + n2 + n3;
        lo += (x.x - n0 * kF1NegInc) + (x.y - n1 * kF1NegInc) + (x.z - n2 * kF1NegInc) + (x.w - n3 * kF1NegInc);
        row[q] = make_uint4(0, 0, 0, 0);
      }
      acc[2 * j] += lo;
      acc[2 * j + 1] += hi;
    }
  }
}

// F1's window: the kF1LPages consecutive magnitude pages holding most of a 4K-pattern sample of
// the segment [a, b), and whether the lane-private path pays (every thread calls it; the result
// is in *s_base / *s_lp after the closing barrier).
__device__ __forceinline__ void f1_choose_window(const uint16_t* w, int64_t a, int64_t b, int wdtype, uint32_t* s_pg,
                                              int* s_base, int* s_lp) {
  const int tid = threadIdx.x;
  if (tid < kMagPages) s_pg[tid] = 0;
  __syncthreads();
  if (wdtype == kBF16) {
    // (a vectorised sample with a warp-aggregated add measured 6% slower overall: its registers
    // changed the allocation of the hot loop)
    const int64_t se = min(b, a + kF1Sample);
#pragma unroll 4
    for (int64_t i = a + tid; i < se; i += blockDim.x) atomicAdd(&s_pg[(w[i] >> 8) & 0x7F], 1u);
  }
  __syncthreads();
  if (tid < 32) {
    long long m[4], tot = 0, best;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      m[q] = s_pg[tid + 32 * q];
      tot += m[q];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    const int bb = warp_best_window(m, kF1LPages, best);
    if (tid == 0) {
      *s_base = bb;
      // lane-private path when the window holds >= 98% of a non-trivial sample
      *s_lp = wdtype == kBF16 && tot >= 1024 && best * 50 >= tot * 49;
    }
  }
  __syncthreads();
}

template <int MC>
__device__ __forceinline__ void f1_body(const StreamArgs& A, int32_t* counts, uint32_t k16, uint32_t k128);

// MC: NVLS mode -- `counts` is a multicast address; every CTA (the grid is exactly the SM count on
// every rank) ends by adding 1 to its arrival counter flags_mc[blockIdx.x] with release semantics
// at system scope, after its own flushes (see f1_nvls_wait_kernel).
template <int MC>
__global__ void __launch_bounds__(kThreads, 1) f1_hist_kernel(const __grid_constant__ StreamArgs A, int32_t* counts,
                                                              uint32_t k16, uint32_t k128, uint32_t* flags_mc) {
  f1_body<MC>(A, counts, k16, k128);
  if (MC) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (MC == 1) {
        asm volatile("multimem.red.release.sys.global.add.u32 [%0], 1;" ::"l"(flags_mc + blockIdx.x) : "memory");
      } else {
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(flags_mc + blockIdx.x) : "memory");
        if (A.peer_delta)
          asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(reinterpret_cast<char*>(flags_mc + blockIdx.x) +
                                                                        A.peer_delta)
                       : "memory");
      }
    }
  }
}

// NVLS mode: wait until every CTA of every rank has arrived for this step (counter >= nranks *
// epoch, monotonic, never reset, so a fast rank's next-step arrivals cannot be lost), then
// advance this rank's epoch.  One CTA; the acquire loads order the reads of the counts after it.
// On timeout (a rank is gone, or multicast reductions do not arrive): trap -- fail loudly instead
// of hanging -- or, for a self-check that must be able to fall back (trap = 0), record the
// failure in g_nvls_failed (edkm_nvls_failed) and let the stream continue.
__device__ uint32_t g_nvls_failed;
__global__ void f1_nvls_wait_kernel(const uint32_t* flags, int nflags, uint32_t* epoch, uint32_t nranks,
                                    uint64_t timeout_ns, int trap) {
  const uint32_t e = *epoch + 1u, target = e * nranks;
  __shared__ int s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int c = threadIdx.x; c < nflags; c += blockDim.x) {
    uint32_t v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + c) : "memory");
      if ((int32_t)(v - target) >= 0) break;
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > timeout_ns || *(volatile int*)&s_fail) {
        if (trap) {
          printf("edkm: NVLS arrival barrier timed out (counter %d = %u, waiting for %u)\n", c, v, target);
          asm volatile("trap;");
        }
        s_fail = 1;
        break;
      }
      __nanosleep(64);
    }
  }
  // the counts were written through the multicast address and are read (here and by TF) through
  // the unicast one: order the aliased accesses after the acquire (virtual aliasing proxy)
  asm volatile("fence.proxy.alias;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_fail) atomicExch(&g_nvls_failed, 1u);
    *epoch = e;
  }
}

template <int MC>
__device__ __forceinline__ void f1_body(const StreamArgs& A, int32_t* counts, uint32_t k16, uint32_t k128) {
  extern __shared__ __align__(16) uint32_t smem_u32[];
  __shared__ uint32_t s_pg[kMagPages];
  __shared__ int s_base, s_lp;
  uint32_t* h = smem_u32;
  int64_t lo, hi;
  cta_range(A.total, lo, hi);
  if (lo >= hi) return;
  int t = find_tensor(A, lo);
  const int tid = threadIdx.x, bs = blockDim.x, lane = tid & 31;
  F1Policy<MC> gen{A, h, counts};
  while (lo < hi) {
    while (A.offs[t + 1] <= lo) ++t;
    const int64_t a = lo - A.offs[t], b = min(hi, A.offs[t + 1]) - A.offs[t];
    const uint16_t* w = A.w[t];
    int32_t* cnt = counts + (int64_t)(A.t0 + t) * kPatterns;
    // ---- choose the lane-private window from a sample of the segment
    f1_choose_window(w, a, b, A.wdtype, s_pg, &s_base, &s_lp);
    if (s_lp) {
      const uint32_t pb2 = ((0x10000u - ((uint32_t)s_base << 8)) & 0xFFFFu) * 0x10001u;  // -pbase*256, both halves
      const uint32_t base = smem_addr(h) + (uint32_t)lane * 4u;
      {
        uint4* z = reinterpret_cast<uint4*>(h);
        for (int i = tid; i < kF1LRows * 32 / 4; i += bs) z[i] = make_uint4(0, 0, 0, 0);
      }
      __syncthreads();
      uint32_t acc[4] = {0, 0, 0, 0};
      const uintptr_t wa = (uintptr_t)(w + a);
      const int64_t head = min((int64_t)(((32u - (uint32_t)(wa & 31u)) & 31u) >> 1), b - a);
      const int64_t va = a + head;
      const int64_t nv = (b - va) >> 4;
      for (int64_t i = a + tid; i < a + head; i += bs) f1_count_global<MC>(cnt, w[i], A.peer_delta);
      for (int64_t i = va + 16 * nv + tid; i < b; i += bs) f1_count_global<MC>(cnt, w[i], A.peer_delta);
      // one 16-pattern vector.  Every lane takes the same straight-line path: a pattern outside
      // the window is clamped to the trash row kF1LRows (never folded), and the lanes holding
      // such a pattern (~0.1% of bf16 N(0, 0.02^2) weights, but ~40% of warp iterations see one)
      // then add it to the global count in a short pass.  Before, a whole per-element slow path
      // ran divergently for those lanes (ncu: 26.9 of 32 threads active per warp).
      const uint32_t lim2 = (uint32_t)kF1LRows * 0x10001u;
      auto count_vec = [&](const V8& r) {
        uint32_t rmax2 = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t x = r.x[q];
          const uint32_t rel = __vadd2(x & 0x7FFF7FFFu, pb2);
          rmax2 = __vmaxu2(rmax2, rel);
          const uint32_t rc = __vminu2(rel, lim2);
          // row offsets by IMAD (k16, k128 are kernel parameters, opaque to ptxas, so the
          // multiplies stay on the FMA pipe); the increment 1 or 0x10000 (the sign selects the
          // counter half) from one PRMT sign-replicate + 1.  F1 is ALU-pipe bound otherwise.
          const uint32_t rh = __umulhi(rc, k16);
          const uint32_t rl = rc & 0xFFFFu;
          // increment 1 (positive pattern) or kF1NegInc = 0xFF01 (negative) in ONE PRMT: byte 0
          // from the constant 1, byte 1 the sign of the pattern replicated, bytes 2-3 zero
          uint32_t ilo, ihi;
          asm("prmt.b32 %0, %1, %2, 0x5594;" : "=r"(ilo) : "r"(x), "r"(1u));
          asm("prmt.b32 %0, %1, %2, 0x55B4;" : "=r"(ihi) : "r"(x), "r"(1u));
          red_add_shared(rl * k128 + base, ilo);
          red_add_shared(rh * k128 + base, ihi);
        }
        if (max(rmax2 & 0xFFFFu, rmax2 >> 16) >= (uint32_t)kF1LRows) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t x = r.x[q];
            const uint32_t rel = __vadd2(x & 0x7FFF7FFFu, pb2);
            if ((rel & 0xFFFFu) >= (uint32_t)kF1LRows) f1_count_global<MC>(cnt, x & 0xFFFFu, A.peer_delta);
            if ((rel >> 16) >= (uint32_t)kF1LRows) f1_count_global<MC>(cnt, x >> 16, A.peer_delta);
          }
        }
      };
      for (int64_t c0 = 0; c0 < nv; c0 += (int64_t)kF1LChunkVec * bs) {
        const int64_t c1 = min(nv, c0 + (int64_t)kF1LChunkVec * bs);
#pragma unroll 1
        for (int64_t v = c0 + tid; v < c1; v += 2 * bs) {
          V8 r[2];
          const bool two = v + bs < c1;
          r[0] = ldg_stream8(w + va + 16 * v);
          if (two) r[1] = ldg_stream8(w + va + 16 * (v + bs));
          count_vec(r[0]);
          if (two) count_vec(r[1]);
        }
        __syncthreads();
        f1l_fold(h, acc);
        __syncthreads();
      }
      // global counts of the window patterns: row r is rel, acc[2j] positive, acc[2j+1] negative
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = tid + j * 1024;
        if (r < kF1LRows) {
          const uint32_t u = ((uint32_t)s_base << 8) + (uint32_t)r;
          if (acc[2 * j]) cnt_add<MC>(&cnt[u], (int32_t)acc[2 * j], A.peer_delta);
          if (acc[2 * j + 1]) cnt_add<MC>(&cnt[u | 0x8000u], (int32_t)acc[2 * j + 1], A.peer_delta);
        }
      }
      __syncthreads();
    } else {
      // shared-array path (the generic visitor's body for this one segment)
      gen.begin(t, a, b);
      const uintptr_t wa = (uintptr_t)(w + a);
      const int64_t head = min((int64_t)(((32u - (uint32_t)(wa & 31u)) & 31u) >> 1), b - a);
      const int64_t va = a + head;
      const int64_t nv = (b - va) >> 4;
      for (int64_t i = a + tid; i < a + head; i += bs) gen.scalar(t, i);
      int64_t v = tid;
      for (; v + bs < nv; v += 2 * bs) {
        typename F1Policy<MC>::Vec r0, r1;
        gen.load(t, va + 16 * v, r0);
        gen.load(t, va + 16 * (v + bs), r1);
        gen.process(t, va + 16 * v, r0);
        gen.process(t, va + 16 * (v + bs), r1);
      }
      if (v < nv) {
        typename F1Policy<MC>::Vec r0;
        gen.load(t, va + 16 * v, r0);
        gen.process(t, va + 16 * v, r0);
      }
      for (int64_t i = va + 16 * nv + tid; i < b; i += bs) gen.scalar(t, i);
      gen.end(t);
    }
    lo = A.offs[t] + b;
    ++t;
  }
}

// ---------------------------------------------------------------- F1 for fp16 weights
// fp16 N(0, 0.02^2) weights spread over quarter-binade pages: the lane-private window (7 pages)
// holds about half of them, so fp16 segments always took f1_body's shared-array path -- whose
// per-element range test and branch (patterns >= 0xE000 go to the L2 counts) issued ~3x the
// instructions of the atomic itself.  This kernel runs that path alone (the bf16 kernel keeps its
// register allocation), branch-free: every pattern is clamped to the trash counter h[kF1Bins]
// (never flushed) and a vector holding one >= 0xE000 (|w| >= 512: not in trained weights) re-adds
// those to the global counts.  Still bound by shared-atomic bank conflicts (~7.7 wavefronts per
// warp instruction: DESIGN S9).
template <int MC>
struct F1SharedPolicy : F1Policy<MC> {
  static constexpr int kLoop = 0;
  using typename F1Policy<MC>::Vec;
  __device__ void begin(int t, int64_t a, int64_t b) {
    if (threadIdx.x == 0) this->h[kF1Bins] = 0;  // the trash counter (never read; initialised for initcheck)
    F1Policy<MC>::begin(t, a, b);
  }
  __device__ void process(int t, int64_t i, const Vec& r) {
    const uint32_t base = smem_addr(this->h);
    uint32_t mx2 = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t x = r.w.x[q];
      mx2 = __vmaxu2(mx2, x);
      const uint32_t c2 = __vminu2(x, (uint32_t)kF1Bins * 0x10001u);
      red_add_shared(base + (c2 & 0xFFFFu) * 4u, 1u);
      red_add_shared(base + (c2 >> 16) * 4u, 1u);
    }
    if (max(mx2 & 0xFFFFu, mx2 >> 16) >= (uint32_t)kF1Bins) {
      // rare: re-read the 16 patterns (dynamic indexing of the register vector would spill it)
#pragma unroll 1
      for (int e = 0; e < 16; ++e) {
        const uint32_t u = this->A.w[t][i + e];
        if (u >= (uint32_t)kF1Bins) cnt_add<MC>(&this->cnt(t)[u], 1, this->A.peer_delta);
      }
    }
  }
};

template <int MC>
__global__ void __launch_bounds__(kThreads, 1) f1_fp16_kernel(const __grid_constant__ StreamArgs A, int32_t* counts,
                                                              uint32_t* flags_mc) {
  extern __shared__ __align__(16) uint32_t smem_u32[];
  F1SharedPolicy<MC> p{{A, smem_u32, counts}};
  for_each_segment(A, p);
  if (MC) {  // NVLS arrival, as in f1_hist_kernel
    __syncthreads();
    if (threadIdx.x == 0) {
      if (MC == 1) {
        asm volatile("multimem.red.release.sys.global.add.u32 [%0], 1;" ::"l"(flags_mc + blockIdx.x) : "memory");
      } else {
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(flags_mc + blockIdx.x) : "memory");
        if (A.peer_delta)
          asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(reinterpret_cast<char*>(flags_mc + blockIdx.x) +
                                                                        A.peer_delta)
                       : "memory");
      }
    }
  }
}

// ============================================================================ F2
// mode: 0 soft 16-bit, 1 hard-value 16-bit, 2 soft fp32, 3 hard-value fp32, 4 hard index u8


template <int MODE>
struct F2Policy {
  static constexpr int kLoop = 0;  // one vector per iteration (measured faster for the gather)
  const StreamArgs& A;
  const F2Args& F;
  unsigned char* sm;
  TmaTable tma;
  int pbase, np;
  struct Vec { V8 w; };
  __device__ int gt(int t) const { return A.t0 + t; }
  __device__ void begin(int t, int64_t, int64_t) {
    const int T = gt(t);
    if (MODE == 0) {
      // the whole 16-bit W~ table (128 KiB), staged by TMA
      const uint16_t* src = F.table16 + (int64_t)T * kPatterns;
      if (TmaTable::aligned(src)) {
        tma.stage(sm, src, kPatterns * 2);
        return;
      }
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      uint4* dst = reinterpret_cast<uint4*>(sm);
      for (int i = threadIdx.x; i < kPatterns * 2 / 16; i += blockDim.x) dst[i] = __ldg(s4 + i);
    } else if (MODE == 1) {
      uint16_t* tab = reinterpret_cast<uint16_t*>(sm);
      const uint8_t* ix = F.idx8 + (int64_t)T * kPatterns;
      const float* C = F.C + (int64_t)T * F.k;
      for (int u = threadIdx.x; u < kPatterns; u += blockDim.x) {
        // index entries of absent finite patterns are not written by TF (never read for the output):
        // clamp before the centroid load so that a stale byte cannot index past C
        const uint32_t j = ix[u];
        tab[u] = pattern_finite(u, A.wdtype) && j < (uint32_t)F.k ? round16f(__ldg(C + j), A.wdtype)
                                                                   : nan16(A.wdtype);
      }
    } else if (MODE == 2) {
      pbase = F.state[T].win[2];  // chosen once per tensor by TF (table_windows)
      np = F.state[T].win[3];
      float* tab = reinterpret_cast<float*>(sm);
      const float* src = F.table + (int64_t)T * kPatterns;
      if (TmaTable::aligned(src)) {
        // the window's two halves are contiguous ranges of the table: patterns pbase*256.. of each sign
        const uint32_t half = (uint32_t)np * 256u;
        tma.stage(tab, src + pbase * 256, half * 4, tab + half, src + 0x8000 + pbase * 256, half * 4);
        return;
      }
      for (int s = threadIdx.x; s < 2 * np * 256; s += blockDim.x) tab[s] = __ldg(src + slot_pattern(s, pbase, np));
    } else {
      uint8_t* ix = reinterpret_cast<uint8_t*>(sm);
      const uint8_t* src = F.idx8 + (int64_t)T * kPatterns;
      if (MODE == 3) {  // the centroids, next to the index table (end() of the last segment synced)
        float* Cs = reinterpret_cast<float*>(sm + kPatterns);
        if (threadIdx.x < F.k) Cs[threadIdx.x] = F.C[(int64_t)T * F.k + threadIdx.x];
      }
      if (TmaTable::aligned(src)) {
        tma.stage(ix, src, kPatterns);
        if (MODE == 3) __syncthreads();  // Cs
        return;
      }
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      uint4* dst = reinterpret_cast<uint4*>(ix);
      for (int i = threadIdx.x; i < kPatterns / 16; i += blockDim.x) dst[i] = __ldg(s4 + i);
    }
    __syncthreads();
  }
  __device__ bool vec_ok(int t, int64_t i) const {
    const int osz = (MODE == 0 || MODE == 1) ? 2 : (MODE == 4 ? 1 : 4);
    const uintptr_t o = (uintptr_t)A.out[t] + (uintptr_t)i * osz;
    return (o & (MODE == 4 ? 15u : 31u)) == 0;
  }
  __device__ void load(int t, int64_t i, Vec& r) const { r.w = ldg_stream8(A.w[t] + i); }
  __device__ float f32_of(int t, uint32_t u) const {
    if (MODE == 2) {
      const int s = window_slot(u, pbase, np);
      return s >= 0 ? reinterpret_cast<const float*>(sm)[s] : __ldg(F.table + (int64_t)gt(t) * kPatterns + u);
    }
    // MODE 3: non-finite patterns have NaN value
    if (!pattern_finite(u, A.wdtype)) return __int_as_float(0x7FC00000);
    return reinterpret_cast<const float*>(sm + kPatterns)[sm[u]];
  }
  __device__ void process(int t, int64_t i, const Vec& r) {
    if (MODE == 0 || MODE == 1) {
      const uint16_t* tab = reinterpret_cast<const uint16_t*>(sm);
      V8 o;
#pragma unroll
      for (int q = 0; q < 8; ++q) o.x[q] = (uint32_t)tab[r.w.x[q] & 0xFFFFu] | ((uint32_t)tab[r.w.x[q] >> 16] << 16);
      stg_stream8(reinterpret_cast<uint16_t*>(A.out[t]) + i, o);
    } else if (MODE == 2 || MODE == 3) {
      V8 o0, o1;
#pragma unroll
      for (int e = 0; e < 8; ++e) o0.x[e] = __float_as_uint(f32_of(t, pat(r.w, e)));
#pragma unroll
      for (int e = 0; e < 8; ++e) o1.x[e] = __float_as_uint(f32_of(t, pat(r.w, 8 + e)));
      float* out = reinterpret_cast<float*>(A.out[t]) + i;
      stg_stream8(out, o0);
      stg_stream8(out + 8, o1);
    } else {
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t a = r.w.x[2 * q], b = r.w.x[2 * q + 1];
        o[q] = (uint32_t)sm[a & 0xFFFFu] | ((uint32_t)sm[a >> 16] << 8) | ((uint32_t)sm[b & 0xFFFFu] << 16) |
               ((uint32_t)sm[b >> 16] << 24);
      }
      stg_stream4(reinterpret_cast<uint8_t*>(A.out[t]) + i, o[0], o[1], o[2], o[3]);
    }
  }
  __device__ void scalar(int t, int64_t i) {
    const uint32_t u = A.w[t][i];
    if (MODE == 0 || MODE == 1) reinterpret_cast<uint16_t*>(A.out[t])[i] = reinterpret_cast<const uint16_t*>(sm)[u];
    else if (MODE == 2 || MODE == 3) reinterpret_cast<float*>(A.out[t])[i] = f32_of(t, u);
    else reinterpret_cast<uint8_t*>(A.out[t])[i] = sm[u];
  }
  __device__ void end(int) { __syncthreads(); }
};

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) f2_gather_kernel(const __grid_constant__ StreamArgs A, const F2Args F) {
  extern __shared__ __align__(128) unsigned char smem_u8[];
  __shared__ uint64_t s_bar;
  F2Policy<MODE> p{A, F, smem_u8, {}, 0, 0};
  p.tma.init(&s_bar);
  for_each_segment(A, p);
}

// ============================================================================ B1
// B[u] = sum G_i over this CTA's weights with pattern u, accumulated in 32-bit fixed point with
// native shared-memory integer atomics -- sm_100 has no native shared fp32 (or 64-bit integer)
// atomic add: ptxas emits a CAS loop for both.
//
// Two fixed-point banks per pattern slot (S4 "B1"): the per-segment scale 2^s maps the
// largest |G| of a 4K-element sample M to [2^21, 2^22).  An element with |G| >= 2^(24-s-f) goes
// to the coarse bank as q = rint(G 2^s); a smaller one to the fine bank as q = rint(G 2^(s+f)).
// Every |q| < 2^24.  For 16-bit G this is EXACT (no rounding at all) for every |G| in
// [2^(7-s-f), 2^(24-s)) ~ [M 2^-(15+f), 4..8 M): a bf16 (fp16) value with |G| >= 2^e has its
// last significand bit at 2^(e-7) (2^(e-10)), a multiple of 2^-s once e >= 7-s (10-s), which
// f <= 17 (14) guarantees for every coarse element.  For fp32 G each element is split into both
// banks: q_c = rint(G 2^s), and the exact residual G 2^s - q_c (|.| <= 1/2) as q_f = rint(. 2^f)
// with f = 24, so its rounding is below M 2^-46.  A scale set by the sample max alone (one bank,
// round 1) rounded every element to M 2^-22 in absolute terms: heavy-tailed G (Cauchy,
// Student-t, log-normal) then put dC_0 over the 1e-5 bar.
//
// lo[] starts at 2^31 (slot value = lo - 2^31 plus the carries): a zero-mean running sum then
// wraps lo only when it leaves (-2^31, 2^31).  The rare carry/borrow out of lo is added to the
// fp64 global bucket directly as +-2^32 of the bank's unit (exact: a power of two), so no
// high word is kept in shared memory.  A pattern outside the shared window, an element whose
// coarse |q| would reach 2^24 (|G| >= 4..8 M), or a non-finite G goes to the fp64 global bucket
// instead (predicated, correct, slower).  At the end of the segment the per-CTA bank values are
// converted to fp64 once and added to the global buckets.
// GDT: gradient dtype (kBF16, kFP16, kFP32).
#ifndef EDKM_B1_LOOP
#define EDKM_B1_LOOP 0
#endif
#ifndef EDKM_B2_LOOP
#define EDKM_B2_LOOP 0
#endif
#ifndef EDKM_B1_BATCH
#define EDKM_B1_BATCH 8
#endif
template <int GDT>
struct B1Policy {
  static constexpr int kLoop = EDKM_B1_LOOP;
  static constexpr int GF32 = GDT == kFP32;
  // fine-bank shift f (see above): bf16 <= 17, fp16 <= 14 keep every coarse element exact; at the
  // bound, thrF = 2^(24-s-f) is exactly the smallest |G| the coarse bank holds exactly, so the
  // fewest elements (and warps) need the fine bank
  static constexpr int kFine = GDT == kBF16 ? 17 : (GDT == kFP16 ? 14 : 24);
  static constexpr uint32_t kSlots = 2 * kB1Pages * 256;  // slots per bank
  static constexpr uint32_t kFOff = kSlots * 4;           // byte offset of the fine bank
  static constexpr uint32_t kLoBias = 0x80000000u;
  static constexpr int kB1Batch = EDKM_B1_BATCH;  // lo atomics in flight per thread
  const StreamArgs& A;
  const B1Args& Bq;
  uint32_t* lo;    // [2][kSlots]: coarse bank, fine bank
  int pbase, np;
  bool active;     // scale established (some finite nonzero G, representable scale)
  float scale;     // 2^s  (coarse)
  float scaleF;    // 2^(s+fe)  (fine)
  float thrF;      // 16-bit G: |G| < thrF -> fine bank (2^(24-s-fe)); fp32 G: 2^fe
  uint32_t glim;   // fp32 bits of 2^24 / 2^s: |G| below it has coarse |q| < 2^24 (fast path)
  uint32_t glim16; // the same bound for 16-bit G bit patterns (NaN/Inf excluded)
  uint32_t thrm1;  // 16-bit G: (smallest magnitude pattern >= thrF) - 1, or 0 if that is pattern 0
  uint32_t negpb2; // -pbase*256 in both 16-bit halves
  double unitC, unitF;  // 2^-s, 2^-(s+fe): the value of one unit of each bank
  Win win;
  struct Vec { V8 w; V8 g[GF32 ? 2 : 1]; };
  __device__ double* bucket(int t) const { return Bq.B + (int64_t)(A.t0 + t) * kPatterns; }
  __device__ float gval(int t, int64_t i) const {
    if (GF32) return reinterpret_cast<const float*>(A.g[t])[i];
    return decode16f(reinterpret_cast<const uint16_t*>(A.g[t])[i], GDT);
  }
  __device__ void begin(int t, int64_t a, int64_t b) {
    __shared__ unsigned s_max;
    if (threadIdx.x == 0) s_max = 0;
    pbase = Bq.state[A.t0 + t].win[0];  // chosen once per tensor by TF (table_windows)
    np = Bq.state[A.t0 + t].win[1];
    uint4* z = reinterpret_cast<uint4*>(lo);
    for (int s = threadIdx.x; s < 2 * np * 256 / 4; s += blockDim.x) {
      z[s] = make_uint4(kLoBias, kLoBias, kLoBias, kLoBias);
      z[s + kSlots / 4] = make_uint4(kLoBias, kLoBias, kLoBias, kLoBias);
    }
    __syncthreads();  // s_max = 0 before any atomicMax
    // scale from the max finite |G| of a sample (whole segment if the sample is all zero)
    unsigned m = 0;
    const int64_t sample_end = min(b, a + 4096);  // 16K measured 7% slower on CFG2's B1
    for (int pass = 0; pass < 2; ++pass) {
      const int64_t e_end = pass == 0 ? sample_end : b;
      for (int64_t i = (pass == 0 ? a : sample_end) + threadIdx.x; i < e_end; i += blockDim.x) {
        const unsigned ab = __float_as_uint(fabsf(gval(t, i)));
        if (ab < 0x7F800000u) m = max(m, ab);
      }
      m = __reduce_max_sync(0xffffffffu, m);
      if ((threadIdx.x & 31) == 0) atomicMax(&s_max, m);
      __syncthreads();
      if (s_max != 0) break;
      __syncthreads();
    }
    const unsigned mx = s_max;
    active = false;
    scale = scaleF = thrF = 0.0f;
    unitC = unitF = 0.0;
    glim = 0;
    glim16 = 0;
    thrm1 = 0;
    if (mx != 0) {
      int e;
      frexpf(__uint_as_float(mx), &e);  // mx in [2^(e-1), 2^e)
      const int s = 22 - e;              // mx * 2^s in [2^21, 2^22)
      if (s <= 126 && s >= -126) {
        active = true;
        // fine shift, capped so that 2^(s+fe) stays a normal fp32 (tiny gradients, s near 126)
        const int fe = min(kFine, 127 - s);
        scale = __int_as_float((127 + s) << 23);
        scaleF = __int_as_float((127 + s + fe) << 23);
        thrF = GF32 ? __int_as_float((127 + fe) << 23) : __int_as_float((127 + 24 - s - fe) << 23);
        unitC = __longlong_as_double((long long)(1023 - s) << 52);
        unitF = __longlong_as_double((long long)(1023 - s - fe) << 52);
        glim = __float_as_uint(16777216.0f * (float)unitC);  // exact: power-of-two scaling
        const float lim = __uint_as_float(glim);
        if (GDT == kBF16) glim16 = min((glim + 0xFFFFu) >> 16, 0x7F80u);
        else glim16 = lim >= 65504.0f ? 0x7C00u : (uint32_t)__half_as_ushort(__float2half_ru(lim));
        // thrF is a power of two: its exact bf16 pattern, or the fp16 pattern rounded up (0x0001 when
        // thrF is below the smallest fp16 subnormal, 0x7C00 = inf when above the largest finite)
        const uint32_t t16 = GDT == kBF16 ? (__float_as_uint(thrF) >> 16)
                                          : (uint32_t)__half_as_ushort(__float2half_ru(thrF));
        thrm1 = t16 ? t16 - 1u : 0u;
      }
    }
    win.init<4>(smem_addr(lo), pbase, np);
    negpb2 = ((0x10000u - win.pb256) & 0xFFFFu) * 0x10001u;
    __syncthreads();
  }
  __device__ bool vec_ok(int t, int64_t i) const {
    const uintptr_t g = (uintptr_t)A.g[t] + (uintptr_t)i * (GF32 ? 4 : 2);
    return (g & 31u) == 0;
  }
  __device__ void load(int t, int64_t i, Vec& r) const {
    r.w = ldg_stream8(A.w[t] + i);
    if (GF32) {
      r.g[0] = ldg_stream8(reinterpret_cast<const float*>(A.g[t]) + i);
      r.g[GF32] = ldg_stream8(reinterpret_cast<const float*>(A.g[t]) + i + 8);
    } else {
      r.g[0] = ldg_stream8(reinterpret_cast<const uint16_t*>(A.g[t]) + i);
    }
  }
  // the carry (+1) or borrow (-1) out of lo of an add of q that returned `old`: moved to the
  // global fp64 bucket as +-2^32 units of the bank (exact)
  __device__ __forceinline__ void carry(double* gB, uint32_t u, int q, uint32_t old, double unit) const {
    const bool c = old + (uint32_t)q < old;
    if (c != (q < 0)) atomicAdd(gB + u, c ? 4294967296.0 * unit : -4294967296.0 * unit);
  }
  // the bank (fine?) and integer q of a 16-bit-dtype element (|G| < 2^(24-s) assumed)
  __device__ __forceinline__ int q16(float g, bool& fine) const {
    fine = fabsf(g) < thrF;
    return __float2int_rn(g * (fine ? scaleF : scale));
  }
  // generic element (scalar head/tail, out-of-window vectors, segments without a scale)
  __device__ __forceinline__ void add_slow(int t, uint32_t u, float g) {
    const int slot = window_slot(u, pbase, np);
    if (active && slot >= 0 && __float_as_uint(fabsf(g)) < glim) {
      const uint32_t a = smem_addr(lo) + (uint32_t)slot * 4u;
      if (GF32) {
        const float x = g * scale, xr = rintf(x);
        const int qc = (int)xr, qf = __float2int_rn((x - xr) * thrF);
        carry(bucket(t), u, qc, atom_add_shared(a, (uint32_t)qc), unitC);
        carry(bucket(t), u, qf, atom_add_shared(a + kFOff, (uint32_t)qf), unitF);
      } else {
        bool fine;
        const int q = q16(g, fine);
        carry(bucket(t), u, q, atom_add_shared(a + (fine ? kFOff : 0u), (uint32_t)q), fine ? unitF : unitC);
      }
    } else if (g != 0.0f) {
      atomicAdd(&bucket(t)[u], (double)g);
    }
  }
  __device__ __forceinline__ float g_of(const Vec& r, int e) const {
    if (GF32) return __uint_as_float(r.g[e >> 3].x[e & 7]);
    if (GDT == kBF16) return __uint_as_float((e & 1) ? (r.g[0].x[e >> 1] & 0xFFFF0000u) : (r.g[0].x[e >> 1] << 16));
    return decode16f(pat(r.g[0], e), kFP16);
  }
  // The lo atomics of one vector, kB1Batch in flight per thread before any return value is looked
  // at, then the (rare) carries.  MODE 0: every element to the coarse bank (16-bit G, no nonzero
  // |G| below thrF: the common case, one FMUL + F2I + atomic per element); 1: per-element bank
  // choice (16-bit G with some small nonzero |G|); 2: both banks, split (fp32 G).
  template <int MODE>
  __device__ __forceinline__ void accumulate(int t, const Vec& r, const uint32_t (&slot2)[8]) {
    constexpr int kPer = MODE == 2 ? 2 : 1;  // atomics per element
    constexpr int kEl = kB1Batch / kPer;     // elements per batch
#pragma unroll
    for (int h = 0; h < 16; h += kEl) {
      uint32_t old[kB1Batch];
      int qv[kB1Batch];
#pragma unroll
      for (int e = h; e < h + kEl; ++e) {
        const uint32_t slot = (e & 1) ? (slot2[e >> 1] >> 16) : (slot2[e >> 1] & 0xFFFFu);
        const uint32_t a = win.baseP + slot * 4;
        const float g = g_of(r, e);
        if (MODE == 2) {
          const float x = g * scale, xr = rintf(x);
          qv[2 * (e - h)] = (int)xr;
          qv[2 * (e - h) + 1] = __float2int_rn((x - xr) * thrF);
          old[2 * (e - h)] = fixed_lo(a, qv[2 * (e - h)]);
          old[2 * (e - h) + 1] = fixed_lo(a + kFOff, qv[2 * (e - h) + 1]);
        } else if (MODE == 1) {
          bool fine;
          qv[e - h] = q16(g, fine);
          old[e - h] = fixed_lo(a + (fine ? kFOff : 0u), qv[e - h]);
        } else {
          qv[e - h] = __float2int_rn(g * scale);
          old[e - h] = fixed_lo(a, qv[e - h]);
        }
      }
      // |q| < 2^24 here, so lo can only have wrapped if the old value lay within 2^25 of the
      // 2^32 boundary; lo starts at 2^31 and a zero-mean sum of steps ~2^19 stays far from it,
      // so the exact carry pass below runs for almost no batch (one min per pair instead of
      // a carry test per element: B1 was issue-bound on the carry tests).
      uint32_t near = 0xFFFFFFFFu;
#pragma unroll
      for (int e = 0; e < kB1Batch; e += 2) near = min(near, min(old[e] + 0x02000000u, old[e + 1] + 0x02000000u));
      if (near < 0x04000000u) {
        double* gB = bucket(t);
#pragma unroll
        for (int e = h; e < h + kEl; ++e) {
          const uint32_t u = pat(r.w, e);
          if (MODE == 2) {
            carry(gB, u, qv[2 * (e - h)], old[2 * (e - h)], unitC);
            carry(gB, u, qv[2 * (e - h) + 1], old[2 * (e - h) + 1], unitF);
          } else if (MODE == 1) {
            carry(gB, u, qv[e - h], old[e - h], fabsf(g_of(r, e)) < thrF ? unitF : unitC);
          } else {
            carry(gB, u, qv[e - h], old[e - h], unitC);
          }
        }
      }
    }
  }
  __device__ void process(int t, int64_t i, const Vec& r) {
    // Window offsets of the 16 patterns two at a time (16x2 SIMD): rel = (u & 0x7FFF) - pbase*256
    // and slot = sign * np*256 + rel; one range check per vector (every rel < np*256 and every
    // |G| below the overflow limit, NaN/Inf included) selects the fast path.  For 16-bit G the
    // same pass takes the minimum of |G| - 1 per half (zero wraps to 0xFFFF: a zero G adds nothing
    // to either bank), so one compare tells whether every nonzero |G| is >= thrF (coarse bank only).
    uint32_t slot2[8];
    uint32_t rmax2 = 0, gmax = 0, gmin2 = 0xFFFFFFFFu;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t x = r.w.x[q];
      const uint32_t r2 = __vadd2(x & 0x7FFF7FFFu, negpb2);
      rmax2 = __vmaxu2(rmax2, r2);
      slot2[q] = ((x >> 15) & 0x00010001u) * win.np256 + r2;
      if (GF32) {
        gmax = max(gmax, max(r.g[q >> 2].x[(2 * q) & 7] & 0x7FFFFFFFu, r.g[q >> 2].x[(2 * q + 1) & 7] & 0x7FFFFFFFu));
      } else {
        const uint32_t m2 = r.g[0].x[q] & 0x7FFF7FFFu;
        gmax = __vmaxu2(gmax, m2);
        gmin2 = __vminu2(gmin2, __vsub2(m2, 0x00010001u));
      }
    }
    const bool ok = GF32 ? gmax < glim : (max(gmax & 0xFFFFu, gmax >> 16) < glim16);
    if (active && max(rmax2 & 0xFFFFu, rmax2 >> 16) < win.np256 && ok) {
      // the bank choice per element costs ~4 instructions per element, so it runs only for the warps
      // that need it, and for the whole warp: a divergent warp would issue both paths (Gaussian fp16 G
      // has a small element in ~1% of vectors, ~30% of warps: B1 4.37 -> 5.13 ms diverging, ncu r02)
      if (GF32) accumulate<2>(t, r, slot2);
      else if (__all_sync(__activemask(), min(gmin2 & 0xFFFFu, gmin2 >> 16) >= thrm1)) accumulate<0>(t, r, slot2);
      else accumulate<1>(t, r, slot2);
    } else {
      // rare: re-read the 16 elements (dynamic indexing of the register vector would spill it)
#pragma unroll 1
      for (int e = 0; e < 16; ++e) scalar(t, i + e);
    }
  }
  __device__ void scalar(int t, int64_t i) { add_slow(t, A.w[t][i], gval(t, i)); }
  __device__ void end(int t) {
    __syncthreads();
    if (active) {
      double* Bt = bucket(t);
      for (int s = threadIdx.x; s < 2 * np * 256; s += blockDim.x) {
        const int32_t vc = (int32_t)(lo[s] - kLoBias), vf = (int32_t)(lo[s + kSlots] - kLoBias);
        if (vc != 0 || vf != 0) atomicAdd(&Bt[slot_pattern(s, pbase, np)], (double)vc * unitC + (double)vf * unitF);
      }
    }
    __syncthreads();
  }
};

template <int GDT>
__global__ void __launch_bounds__(kThreads, 1) b1_bucket_kernel(const __grid_constant__ StreamArgs A, const B1Args Bq) {
  extern __shared__ __align__(16) uint32_t smem_b1[];
  B1Policy<GDT> p{A, Bq, smem_b1};
  for_each_segment(A, p);
}

// ============================================================================ B2
// dW_i = G_i phi[u_i] + psi[u_i]; (phi, psi) of the window's patterns in shared
// memory, the rest read from the global table (predicated).
// GDT: gradient dtype, ODT: dW dtype (kBF16, kFP16, kFP32).
template <int GDT, int ODT>
struct B2Policy {
  static constexpr int kLoop = EDKM_B2_LOOP;
  static constexpr int GF32 = GDT == kFP32, OF32 = ODT == kFP32;
  const StreamArgs& A;
  const B2Args& Bq;
  float2* tab;
  TmaTable tma;
  int pbase, np;
  uint32_t negpb2;  // -pbase*256 in both 16-bit halves
  Win win;
  struct Vec { V8 w; V8 g[GF32 ? 2 : 1]; };
  __device__ const float2* glob(int t) const { return Bq.phipsi + (int64_t)(A.t0 + t) * kPatterns; }
  __device__ float gval(int t, int64_t i) const {
    if (GF32) return reinterpret_cast<const float*>(A.g[t])[i];
    return decode16f(reinterpret_cast<const uint16_t*>(A.g[t])[i], GDT);
  }
  __device__ void begin(int t, int64_t, int64_t) {
    pbase = Bq.state[A.t0 + t].win[0];  // chosen once per tensor by TF (table_windows)
    np = Bq.state[A.t0 + t].win[1];
    const float2* src = glob(t);
    win.init<8>(smem_addr(tab), pbase, np);
    negpb2 = ((0x10000u - win.pb256) & 0xFFFFu) * 0x10001u;
    if (TmaTable::aligned(src)) {
      // the window's two halves are contiguous ranges of the (phi, psi) table, staged by TMA
      const uint32_t half = (uint32_t)np * 256u;
      tma.stage(tab, src + pbase * 256, half * 8, tab + half, src + 0x8000 + pbase * 256, half * 8);
      return;
    }
    for (int s = threadIdx.x; s < 2 * np * 256; s += blockDim.x) tab[s] = __ldg(src + slot_pattern(s, pbase, np));
    __syncthreads();
  }
  __device__ bool vec_ok(int t, int64_t i) const {
    const uintptr_t g = (uintptr_t)A.g[t] + (uintptr_t)i * (GF32 ? 4 : 2);
    const uintptr_t o = (uintptr_t)A.out[t] + (uintptr_t)i * (OF32 ? 4 : 2);
    return ((g | o) & 31u) == 0;
  }
  __device__ void load(int t, int64_t i, Vec& r) const {
    r.w = ldg_stream8(A.w[t] + i);
    if (GF32) {
      r.g[0] = ldg_stream8(reinterpret_cast<const float*>(A.g[t]) + i);
      r.g[GF32] = ldg_stream8(reinterpret_cast<const float*>(A.g[t]) + i + 8);
    } else {
      r.g[0] = ldg_stream8(reinterpret_cast<const uint16_t*>(A.g[t]) + i);
    }
  }
  __device__ __forceinline__ float g_of(const Vec& r, int e) const {
    if (GF32) return __uint_as_float(r.g[e >> 3].x[e & 7]);
    if (GDT == kBF16) return __uint_as_float((e & 1) ? (r.g[0].x[e >> 1] & 0xFFFF0000u) : (r.g[0].x[e >> 1] << 16));
    return decode16f(pat(r.g[0], e), kFP16);
  }
  __device__ __forceinline__ float dw_slow(int t, uint32_t u, float g) const {
    const int s = window_slot(u, pbase, np);
    const float2 pp = s >= 0 ? tab[s] : __ldg(glob(t) + u);
    return fmaf(g, pp.x, pp.y);
  }
  __device__ __forceinline__ uint32_t pack2(float a, float b) const {
    if (ODT == kBF16) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
      return *reinterpret_cast<const uint32_t*>(&h);
    }
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  __device__ void process(int t, int64_t i, const Vec& r) {
    // shared lookups issued speculatively with a clamped slot (16x2 SIMD offsets, as in B1);
    // one range check per 16 elements redoes the (rare) out-of-window vector via the generic path
    const uint32_t lim = win.np256 - 1u;
    const uint32_t lim2 = lim * 0x10001u;
    uint32_t rmax2 = 0;
    V8 o0, o1;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t x = r.w.x[q];
      const uint32_t r2 = __vadd2(x & 0x7FFF7FFFu, negpb2);
      rmax2 = __vmaxu2(rmax2, r2);
      const uint32_t s2 = ((x >> 15) & 0x00010001u) * win.np256 + __vminu2(r2, lim2);
      float d2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = 2 * q + h;
        const uint32_t slot = h ? (s2 >> 16) : (s2 & 0xFFFFu);
        const float2 pp = lds_f2(win.baseP + slot * 8);
        d2[h] = fmaf(g_of(r, e), pp.x, pp.y);
      }
      if (OF32) {
        V8& o = q < 4 ? o0 : o1;
        o.x[(2 * q) & 7] = __float_as_uint(d2[0]);
        o.x[(2 * q + 1) & 7] = __float_as_uint(d2[1]);
      } else {
        o0.x[q] = pack2(d2[0], d2[1]);
      }
    }
    const uint32_t rmax = max(rmax2 & 0xFFFFu, rmax2 >> 16);
    if (rmax > lim) {
      // rare: redo the 16 elements from memory (dynamic indexing of the register vector would spill it)
#pragma unroll 1
      for (int e = 0; e < 16; ++e) scalar(t, i + e);
      return;
    }
    if (OF32) {
      float* out = reinterpret_cast<float*>(A.out[t]) + i;
      stg_stream8(out, o0);
      stg_stream8(out + 8, o1);
    } else {
      stg_stream8(reinterpret_cast<uint16_t*>(A.out[t]) + i, o0);
    }
  }
  __device__ void scalar(int t, int64_t i) {
    const float d = dw_slow(t, A.w[t][i], gval(t, i));
    if (OF32) reinterpret_cast<float*>(A.out[t])[i] = d;
    else reinterpret_cast<uint16_t*>(A.out[t])[i] = round16f(d, ODT);
  }
  __device__ void end(int) { __syncthreads(); }
};

template <int GDT, int ODT>
__global__ void __launch_bounds__(kThreads, 1) b2_dw_kernel(const __grid_constant__ StreamArgs A, const B2Args Bq) {
  extern __shared__ __align__(128) float2 smem_b2[];
  __shared__ uint64_t s_bar;
  B2Policy<GDT, ODT> p{A, Bq, smem_b2, {}};
  p.tma.init(&s_bar);
  for_each_segment(A, p);
}

// ============================================================================ launchers
static int grid_for(int64_t total, int sms) {
  int64_t g = (total + 16383) / 16384;
  if (g > sms) g = sms;
  return g < 1 ? 1 : (int)g;
}

static cudaError_t set_smem(const void* fn, size_t bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t launch_f1(const StreamArgs& A, int32_t* counts, int sms, cudaStream_t s) {
  if (A.total == 0) return cudaSuccess;
  const size_t smem = kF1Smem;
  if (A.wdtype == kFP16) {
    cudaError_t e = set_smem((const void*)f1_fp16_kernel<0>, smem);
    if (e != cudaSuccess) return e;
    f1_fp16_kernel<0><<<grid_for(A.total, sms), kThreads, smem, s>>>(A, counts, nullptr);
    return cudaGetLastError();
  }
  cudaError_t e = set_smem((const void*)f1_hist_kernel<0>, smem);
  if (e != cudaSuccess) return e;
  f1_hist_kernel<0><<<grid_for(A.total, sms), kThreads, smem, s>>>(A, counts, 0x10000u, 128u, nullptr);
  return cudaGetLastError();
}

// NVLS mode: grid = `sms` CTAs on every rank (also when this rank's slice is empty), each
// signalling its arrival counter; then the wait kernel.
static double g_nvls_timeout_s = 20.0;
static int g_nvls_trap = 1;
void nvls_set_timeout(double seconds, int trap) {
  g_nvls_timeout_s = seconds;
  g_nvls_trap = trap;
}
cudaError_t nvls_failed(int* failed) {
  uint32_t v = 0, z = 0;
  cudaError_t e = cudaMemcpyFromSymbol(&v, g_nvls_failed, sizeof(v));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_nvls_failed, &z, sizeof(z));
  *failed = v != 0;
  return e;
}

cudaError_t launch_f1_nvls(const StreamArgs& A, int32_t* counts_mc, uint32_t* flags_mc, const uint32_t* flags,
                           uint32_t* epoch, int nranks, int emulate, int sms, cudaStream_t s) {
  const size_t smem = kF1Smem;
  const bool h = A.wdtype == kFP16;
  const void* fn = emulate ? (h ? (const void*)f1_fp16_kernel<2> : (const void*)f1_hist_kernel<2>)
                           : (h ? (const void*)f1_fp16_kernel<1> : (const void*)f1_hist_kernel<1>);
  cudaError_t e = set_smem(fn, smem);
  if (e != cudaSuccess) return e;
  if (h) {
    if (emulate) f1_fp16_kernel<2><<<sms, kThreads, smem, s>>>(A, counts_mc, flags_mc);
    else f1_fp16_kernel<1><<<sms, kThreads, smem, s>>>(A, counts_mc, flags_mc);
  } else {
    if (emulate) f1_hist_kernel<2><<<sms, kThreads, smem, s>>>(A, counts_mc, 0x10000u, 128u, flags_mc);
    else f1_hist_kernel<1><<<sms, kThreads, smem, s>>>(A, counts_mc, 0x10000u, 128u, flags_mc);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  f1_nvls_wait_kernel<<<1, 256, 0, s>>>(flags, sms, epoch, (uint32_t)nranks, (uint64_t)(g_nvls_timeout_s * 1e9),
                                        g_nvls_trap);
  return cudaGetLastError();
}

cudaError_t launch_f2(const StreamArgs& A, const F2Args& F, int mode, int sms, cudaStream_t s) {
  if (A.total == 0) return cudaSuccess;
  const void* fn;
  size_t smem;
  switch (mode) {
    case 0: fn = (const void*)f2_gather_kernel<0>; smem = kPatterns * 2; break;
    case 1: fn = (const void*)f2_gather_kernel<1>; smem = kPatterns * 2; break;
    case 2: fn = (const void*)f2_gather_kernel<2>; smem = 2 * kF2Pages32 * 256 * 4; break;
    case 3: fn = (const void*)f2_gather_kernel<3>; smem = kPatterns + 256 * 4; break;
    default: fn = (const void*)f2_gather_kernel<4>; smem = kPatterns; break;
  }
  cudaError_t e = set_smem(fn, smem);
  if (e != cudaSuccess) return e;
  const int g = grid_for(A.total, sms);
  switch (mode) {
    case 0: f2_gather_kernel<0><<<g, kThreads, smem, s>>>(A, F); break;
    case 1: f2_gather_kernel<1><<<g, kThreads, smem, s>>>(A, F); break;
    case 2: f2_gather_kernel<2><<<g, kThreads, smem, s>>>(A, F); break;
    case 3: f2_gather_kernel<3><<<g, kThreads, smem, s>>>(A, F); break;
    default: f2_gather_kernel<4><<<g, kThreads, smem, s>>>(A, F); break;
  }
  return cudaGetLastError();
}

template <int GDT>
static cudaError_t launch_b1_t(const StreamArgs& A, const B1Args& Bq, int sms, cudaStream_t s) {
  const size_t smem = 2 * kB1Pages * 256 * 8;
  cudaError_t e = set_smem((const void*)b1_bucket_kernel<GDT>, smem);
  if (e != cudaSuccess) return e;
  b1_bucket_kernel<GDT><<<grid_for(A.total, sms), kThreads, smem, s>>>(A, Bq);
  return cudaGetLastError();
}

cudaError_t launch_b1(const StreamArgs& A, const B1Args& Bq, int sms, cudaStream_t s) {
  if (A.total == 0) return cudaSuccess;
  switch (A.gdtype) {
    case kBF16: return launch_b1_t<kBF16>(A, Bq, sms, s);
    case kFP16: return launch_b1_t<kFP16>(A, Bq, sms, s);
    default: return launch_b1_t<kFP32>(A, Bq, sms, s);
  }
}

template <int GDT, int ODT>
static cudaError_t launch_b2_t(const StreamArgs& A, const B2Args& Bq, int sms, cudaStream_t s) {
  const size_t smem = 2 * kB2Pages * 256 * 8;
  cudaError_t e = set_smem((const void*)b2_dw_kernel<GDT, ODT>, smem);
  if (e != cudaSuccess) return e;
  b2_dw_kernel<GDT, ODT><<<grid_for(A.total, sms), kThreads, smem, s>>>(A, Bq);
  return cudaGetLastError();
}

template <int GDT>
static cudaError_t launch_b2_g(const StreamArgs& A, const B2Args& Bq, int sms, cudaStream_t s) {
  switch (A.odtype) {
    case kBF16: return launch_b2_t<GDT, kBF16>(A, Bq, sms, s);
    case kFP16: return launch_b2_t<GDT, kFP16>(A, Bq, sms, s);
    default: return launch_b2_t<GDT, kFP32>(A, Bq, sms, s);
  }
}

cudaError_t launch_b2(const StreamArgs& A, const B2Args& Bq, int sms, cudaStream_t s) {
  if (A.total == 0) return cudaSuccess;
  switch (A.gdtype) {
    case kBF16: return launch_b2_g<kBF16>(A, Bq, sms, s);
    case kFP16: return launch_b2_g<kFP16>(A, Bq, sms, s);
    default: return launch_b2_g<kFP32>(A, Bq, sms, s);
  }
}

}  // namespace edkm
