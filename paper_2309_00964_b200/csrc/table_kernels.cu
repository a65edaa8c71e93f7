// table_kernels.cu -- the table phase of the eDKM hot path (S4).
//
// The DKM attention map ("O(|W||C|)") is never formed per weight: by
// uniquification (P:77 S2.2, Fig. 3) every per-weight quantity depends on the
// weight only through its 16-bit pattern u, so the forward iterations and the
// backward loop run over the populated patterns ("rows") with their counts n_u.
//
//   TF      forward: rows <- counts; for t < T: A_t[u] = softmax(-(v_u-C_t)^2/tau),
//           S_t = sum_u n_u A_t[u], M_t = sum_u n_u A_t[u] v_u, C_{t+1} = M_t/S_t;
//           then the W~ table, its 16-bit rounding and the hard-index table.
//   TGAMMA  gamma_T[l] = sum_u B[u] A_T[u,l] (1 + (C_T[l]-W~_u) 2(v_u-C_T[l])/tau)
//   TB      reverse loop t = T-1..0 giving psi[u], dC_0; phi[u] = (2/tau) Var_{A_T[u]}(C_T).
//
// One thread-block cluster per tensor (cl CTAs); rows are split into cl
// contiguous pattern partitions.  Each CTA stages its rows (value v_u, count
// n_u, running psi) in shared memory once, so the T-loops touch no global
// memory; k-vector sums are reduced per thread in row order, then by warp
// shuffles, across warps in warp order and across the cluster through DSMEM in
// CTA order -- deterministic and identical on every CTA and every rank.
// The arithmetic of one row at one iteration is fp32 (the attention on an accurately reduced
// argument, attention_row; TB's terms re-centred on the nearest centroid, tb_row); every sum over
// rows, the centroids, S_t and the recursion across iterations are fp64 (R7).
// Cost O(U k T), independent of N.
#include <cooperative_groups.h>

#include "common.cuh"
#include "launch.h"
#include "table_common.cuh"

namespace cg = cooperative_groups;

namespace edkm {

#ifndef EDKM_FTHREADS
#define EDKM_FTHREADS 256
#endif
constexpr int kFThreads = EDKM_FTHREADS;  // TF, TGAMMA: small shared footprint, two CTAs per SM
// TB: 256 threads and two CTAs per SM (their per-iteration barriers interleave; CFG3 TB 0.29 ->
// 0.24 ms against one 512-thread CTA), with the staged rows sized by the weights' dtype (the
// host does not know U): 4608 rows (72 KiB) for bf16 (U ~ 5K per tensor, cl = 2), 6400 rows
// (100 KiB) for fp16 (U ~ 24K, cl = 4).  Rows beyond the stage are read from global memory,
// so the choice is a performance one only.
// TF: rows per CTA staged in shared memory (value f32, count i32): 4608 (36 KiB) for bf16 and
// 6400 (50 KiB) for fp16, with at most 64 registers (four CTAs per SM) except fp16 k = 16
// (two).  CFG3 TF 0.165 -> 0.142 ms, CFG4 k=4 1.04 -> 0.82 ms; rows beyond the stage take the
// global path, so never wrong.
constexpr int kStageFL = 6400, kStageFS = 4608;
constexpr int kBThreads = 256, kStageB16 = 4608, kStageB32 = 6400;  // TB: value (f32), count (i32), psi (f64)

// Centroids of one iteration in the forms the attention needs: fp64 values, fp32 values
// (to pick the nearest centroid), and per centroid pair (m, j) the fp64-derived difference
// (C_m - C_j) / tau * log2(e) (fp32) and sum C_m + C_j (float-float ph + pl).
template <int K>
struct CSet {
  double c[K];
  float hi[K];
  float sv[K];   // fp32 centroids in ascending order (ties by index) ...
  int sidx[K];   // ... and their indices: nearest-centroid search by bisection
  float dms[K][K];
  float ph[K][K], pl[K][K];
  float dpl[K][K];  // dms * pl (rounded once from fp64): the logit is one FFMA, fma(-dms, 2v - ph, dpl)
  // every thread of the block calls it; the caller synchronises before and after
  __device__ void prepare(const double* src, double inv_tau) {
    const int t = threadIdx.x;
    if (t < K * K) {
      const double a = src[t / K], b = src[t % K], p = a + b;
      const float d = (float)((a - b) * inv_tau * 1.4426950408889634);
      dms[t / K][t % K] = d;
      const float h = (float)p;
      ph[t / K][t % K] = h;
      const float l = (float)(p - (double)h);
      pl[t / K][t % K] = l;
      dpl[t / K][t % K] = (float)((double)d * (double)l);
    }
    if (t < K) {
      const double ct = src[t];
      c[t] = ct;
      hi[t] = (float)ct;
      int rank = 0;
      for (int l = 0; l < K; ++l) rank += (src[l] < ct) || (src[l] == ct && l < t);
      sv[rank] = (float)ct;
      sidx[rank] = t;
    }
  }
  // index of a nearest centroid to v (ties either way: any near-minimum keeps the
  // reduced logits in range; the attention itself is exact in the choice)
  __device__ __forceinline__ int nearest(float vf) const {
    if (K <= 4) {
      int jm = 0;
      float am = fabsf(vf - hi[0]);
#pragma unroll
      for (int j = 1; j < K; ++j) {
        const float a = fabsf(vf - hi[j]);
        if (a < am) { am = a; jm = j; }
      }
      return jm;
    }
    int pos = 0;
#pragma unroll
    for (int st = K / 2; st >= 1; st >>= 1)
      if (sv[pos + st - 1] < vf) pos += st;
    // candidates sv[pos-1], sv[pos]
    const int lo = pos > 0 ? pos - 1 : 0;
    EDKM_BCHECK(pos >= 0 && pos < K);
    return (fabsf(vf - sv[lo]) <= fabsf(vf - sv[pos])) ? sidx[lo] : sidx[pos];
  }
};

// Rows per thread whose per-row products are summed in fp32 before one fp64 add (TF, TB): the
// per-row arithmetic is fp32 (A itself carries ~2^-22 from ex2.approx), every sum over more rows
// is fp64 (R7; tools/exp_tb_fp32.py: dC_0 within 1e-6, C_T within 6e-8 of the oracle).
#ifndef EDKM_ROW_FLUSH
#define EDKM_ROW_FLUSH 32
#endif
constexpr int kRowFlush = EDKM_ROW_FLUSH;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// DKM attention of one pattern value v (exact in fp32: a 16-bit float) to the K centroids:
//   A_j = exp(-(d_j - d_min)/tau) / sum_l exp(-(d_l - d_min)/tau),  d_j = (v - C_j)^2.
// With m the nearest centroid, d_j - d_m = (C_m - C_j)(2v - C_m - C_j).  The second factor
// is 2v - (ph + pl) in fp32: exact where it is small (2v and ph within a factor 2,
// Sterbenz), so near a cluster boundary -- where A is most sensitive -- the logit carries a
// relative, not absolute, fp32 error (~1e-7); far from it the weight is tiny.  The
// exponential is MUFU ex2 (rel. error ~2^-22); A is normalised in fp32 and every sum over
// patterns is done by the callers in fp64 (R7).
template <int K>
__device__ __forceinline__ void attention_row(float vf, const CSet<K>& cs, float (&A)[K]) {
  const int jm = cs.nearest(vf);
  const float* dmr = cs.dms[jm];
  const float* phr = cs.ph[jm];
  const float* dplr = cs.dpl[jm];
  const float v2 = 2.0f * vf;
  float Z = 0.0f;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    // -(dms (2v - ph - pl)) = fma(-dms, 2v - ph, dms pl): 2v - ph exact where it is small
    // (Sterbenz, as before), dms pl a small correction rounded once
    A[j] = ex2(fmaf(-dmr[j], v2 - phr[j], dplr[j]));
    Z += A[j];
  }
  const float iz = 1.0f / Z;
#pragma unroll
  for (int j = 0; j < K; ++j) A[j] *= iz;
}

// Sum of K floats in four interleaved chains, then pairwise: a fixed order (deterministic) with a
// dependent chain of K/4 + 2 adds instead of K.
template <int K>
__device__ __forceinline__ float sum4(const float (&a)[K]) {
  if (K < 4) {
    float z = a[0];
#pragma unroll
    for (int j = 1; j < K; ++j) z += a[j];
    return z;
  }
  float z0 = a[0], z1 = a[1], z2 = a[2], z3 = a[3];
#pragma unroll
  for (int j = 4; j < K; j += 4) {
    z0 += a[j];
    z1 += a[j + 1];
    z2 += a[j + 2];
    z3 += a[j + 3];
  }
  return (z0 + z1) + (z2 + z3);
}

// sum_j a_j b_j in four interleaved FFMA chains, then pairwise (fixed order, as sum4)
template <int K>
__device__ __forceinline__ float dot4(const float (&a)[K], const float* b) {
  if (K < 4) {
    float z = a[0] * b[0];
#pragma unroll
    for (int j = 1; j < K; ++j) z = fmaf(a[j], b[j], z);
    return z;
  }
  float z0 = a[0] * b[0], z1 = a[1] * b[1], z2 = a[2] * b[2], z3 = a[3] * b[3];
#pragma unroll
  for (int j = 4; j < K; j += 4) {
    z0 = fmaf(a[j], b[j], z0);
    z1 = fmaf(a[j + 1], b[j + 1], z1);
    z2 = fmaf(a[j + 2], b[j + 2], z2);
    z3 = fmaf(a[j + 3], b[j + 3], z3);
  }
  return (z0 + z1) + (z2 + z3);
}

// 1/Z for Z >= 1 (the nearest centroid's term is ex2(0) = 1): MUFU rcp, ~1 ulp
__device__ __forceinline__ float rcp_ge1(float z) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(z));
  return y;
}

// The same without the normalisation: fills A with the unnormalised terms and returns 1 / sum_j A[j]
// (the callers apply it to the sums that use A); `m` receives the nearest centroid's index.
template <int K>
__device__ __forceinline__ float attention_row_raw(float vf, const CSet<K>& cs, float (&A)[K], int& m) {
  const int jm = cs.nearest(vf);
  m = jm;
  const float* dmr = cs.dms[jm];
  const float* phr = cs.ph[jm];
  const float* dplr = cs.dpl[jm];
  const float v2 = 2.0f * vf;
#pragma unroll
  for (int j = 0; j < K; ++j) A[j] = ex2(fmaf(-dmr[j], v2 - phr[j], dplr[j]));
  return rcp_ge1(sum4<K>(A));
}

// Warp sum of N doubles per lane (N a power of two <= 32) by a transposing butterfly: at the
// level of xor offset o each lane keeps one half of its remaining values, sends the other half to
// its partner and adds what it receives, so the N values shrink to one while the lanes fan out;
// a lane ends with the whole warp's sum of value (lane >> (5 - log2 N)).  N + N/2 + ... = 2N - 1
// shuffled doubles instead of 5N for N independent xor reductions (ncu r02: the per-iteration
// reduction of TF<16>'s 32 sums was 320 SHFL + 160 DADD, 21% of the kernel's samples).  The
// addition order is fixed: results are deterministic and identical on every CTA and every rank.
template <int N>
__device__ __forceinline__ double warp_transpose_sum(double (&v)[N]) {
  static_assert(N >= 1 && N <= 32 && (N & (N - 1)) == 0, "N: a power of two <= 32");
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int m = N, o = 16; m > 1; m >>= 1, o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < m / 2; ++i) {
      const double send = upper ? v[i] : v[i + m / 2];
      const double keep = upper ? v[i + m / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  double x = v[0];
  // the lanes that share a value index: the low 5 - log2 N bits
#pragma unroll
  for (int o = 16 / N; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
template <int N>
__device__ __forceinline__ constexpr int log2i() { return N <= 1 ? 0 : 1 + log2i<N / 2>(); }

// Sum N doubles over the CTA then over the cluster; result in tot[0..N) of every CTA.
// `part` is a [2][N] shared buffer used with alternating parity so one cluster
// barrier per call suffices.  cluster_allreduce_red starts from per-warp sums already in
// red[warp * N + i] (warp_flush); cluster_allreduce from one N-vector per thread.
template <int N, int NW>
__device__ __forceinline__ void cluster_allreduce_red(const double* red, double* part, double* tot, int parity,
                                                      cg::cluster_group& cluster) {
  __syncthreads();
  double* mine = part + parity * N;
  if (threadIdx.x < N) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += red[w * N + threadIdx.x];
    mine[threadIdx.x] = s;
  }
  cluster.sync();
  if (threadIdx.x < N) {
    double s = 0.0;
    for (unsigned r = 0; r < cluster.num_blocks(); ++r) s += cluster.map_shared_rank(mine, r)[threadIdx.x];
    tot[threadIdx.x] = s;
  }
  __syncthreads();
}

template <int N, int NW>
__device__ __forceinline__ void cluster_allreduce(double (&v)[N], double* red, double* part, double* tot, int parity,
                                                  cg::cluster_group& cluster) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kShift = 5 - log2i<N>();
  const double x = warp_transpose_sum<N>(v);
  if ((lane & ((1 << kShift) - 1)) == 0) red[warp * N + (lane >> kShift)] = x;
  cluster_allreduce_red<N, NW>(red, part, tot, parity, cluster);
}

// Warp-uniform: add the warp's fp32 per-lane partials af[0..N) (in fp64) to the warp's own
// accumulator red_w[0..N) in shared memory (zeroed by warp_zero).  No fp64 accumulators stay
// live in registers across the row loops.
template <int N>
__device__ __forceinline__ void warp_flush(float (&af)[N], double* red_w) {
  __syncwarp();
  const int lane = threadIdx.x & 31;
  constexpr int kShift = 5 - log2i<N>();
  double v[N];
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = (double)af[i];
  const double x = warp_transpose_sum<N>(v);
  if ((lane & ((1 << kShift) - 1)) == 0) red_w[lane >> kShift] += x;
  __syncwarp();
}
template <int N>
__device__ __forceinline__ void warp_zero(double* red_w) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < N; i += 32) red_w[i] = 0.0;
  __syncwarp();
}

// Rows of one partition: patterns in rows[]; value (exact in fp32), count and the running psi
// staged in shared memory for r < kStage, read from global memory beyond (U > kStage per CTA).
struct RowStage {
  const uint16_t* rows;
  const int32_t* cnt;
  float* sv;     // [kStage] value v_u
  int32_t* sn;   // [kStage] count n_u
  double* spsi;  // [kStage] psi accumulator (TB)
  double* gpsi;  // global psi for r >= kStage
  int nr, wdtype, ns;  // ns: staged capacity
  __device__ __forceinline__ double v(int r) const {
    EDKM_BCHECK(r >= 0 && r < nr);
    return r < ns ? (double)sv[r] : decode16(rows[r], wdtype);
  }
  __device__ __forceinline__ double n(int r) const { return (double)(r < ns ? sn[r] : cnt[rows[r]]); }
  __device__ __forceinline__ double& psi(int r) const {
    EDKM_BCHECK(r >= 0 && r < nr);
    return r < ns ? spsi[r] : gpsi[r];
  }
  __device__ __forceinline__ float vf(int r) const { return r < ns ? sv[r] : decode16f(rows[r], wdtype); }
  __device__ __forceinline__ float nf(int r) const { return (float)(r < ns ? sn[r] : cnt[rows[r]]); }
  // four rows per thread per step: their pattern loads, then their count gathers, are issued
  // together (a dependent rows[r] -> cnt[u] pair per row measured 12% of CFG3's TB)
  __device__ void stage() {
    const int lim = min(nr, ns), bd = blockDim.x;
    for (int r0 = threadIdx.x; r0 < lim; r0 += 4 * bd) {
      uint32_t u[4];
      int32_t c[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = r0 + q * bd < lim ? (uint32_t)rows[r0 + q * bd] : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) c[q] = r0 + q * bd < lim ? cnt[u[q]] : 0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (r0 + q * bd < lim) {
          EDKM_BCHECK(r0 + q * bd < ns && u[q] < (uint32_t)kPatterns);
          sv[r0 + q * bd] = decode16f(u[q], wdtype);
          sn[r0 + q * bd] = c[q];
        }
    }
    __syncthreads();
  }
};

// ============================================================================ TF
template <int K, int kStage, int kMinBlocks>
__global__ void __launch_bounds__(kFThreads, kMinBlocks) tf_kernel(const TableArgs P) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double stage_mem[];
  const int cl = P.cl, crank = (int)cluster.block_rank(), t = blockIdx.x / cl, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  __shared__ double sCb[2][K], sCf[K], sDelta[K];  // C_t / C_{t+1}, alternating by iteration parity
  __shared__ double red[(kFThreads / 32) * 2 * K], part[2 * 2 * K];
  __shared__ CSet<K> cs;
  __shared__ int s_scan[(kFThreads / 32)];
  __shared__ long long s_nf[(kFThreads / 32)];

  __shared__ int s_pg[256], s_pref[257], s_pb[kMaxCluster + 1];

  const int32_t* cnt = P.counts + (int64_t)t * kPatterns;
  TensorState* st = P.state + t;
  float* tab = P.table + (int64_t)t * kPatterns;
  uint16_t* tab16 = P.table16 + (int64_t)t * kPatterns;
  uint8_t* idx = P.idx8 + (int64_t)t * kPatterns;

  // ---- 0. partition bounds (identical on every CTA): the two signs for cl = 2 (balanced for a
  //         symmetric law, and page masses come from the compaction loop), else row-balanced ranges
  //         (which also writes the page masses)
  const bool sign_split = cl == 2;
  if (sign_split) {
    if (tid == 0) {
      s_pb[0] = 0;
      s_pb[1] = kPatterns / 2;
      s_pb[2] = kPatterns;
    }
    __syncthreads();
  } else {
    table_partitions<kFThreads>(cnt, P.wdtype, P.page_cnt + (int64_t)t * 256, cl, crank, cluster, s_pg, s_pref, s_pb);
  }
  const int base = s_pb[crank], end = s_pb[crank + 1];
  uint16_t* rows = P.rows + (int64_t)t * kPatterns + base;
  float* stage_v = reinterpret_cast<float*>(stage_mem);                // [kStage] value v_u
  int32_t* stage_n = reinterpret_cast<int32_t*>(stage_mem) + kStage;  // [kStage] count n_u

  // ---- 1. compact populated finite patterns of this partition (ascending u), 16 per thread per step;
  //         non-finite counts, NaN entries of the non-finite patterns in the W~ tables
  int nr = 0;
  long long nonfin = 0;
  for (int off = 0; off < end - base; off += kFThreads * 16) {
    const int u0 = base + off + tid * 16;
    const bool in = u0 < end;
    int c[16];
    const int4* c4 = reinterpret_cast<const int4*>(cnt + (in ? u0 : 0));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int4 x = in ? __ldg(c4 + q) : make_int4(0, 0, 0, 0);
      c[4 * q] = x.x;
      c[4 * q + 1] = x.y;
      c[4 * q + 2] = x.z;
      c[4 * q + 3] = x.w;
    }
    unsigned popmask = 0;
    long long pm = 0;
    // the non-finite patterns form aligned blocks (bf16: 128, fp16: 1,024 per sign), so a 16-aligned
    // group is finite or not as a whole
    const bool fin = pattern_finite(u0, P.wdtype);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      if (fin && c[e] > 0) popmask |= 1u << e;
      pm += c[e];
    }
    if (!fin) nonfin += pm;
    if (sign_split) {  // one signed page = 256 patterns = 16 threads (the ranges are page-aligned)
#pragma unroll
      for (int o = 8; o; o >>= 1) pm += __shfl_xor_sync(0xffffffffu, pm, o);
      if ((lane & 15) == 0 && in) P.page_cnt[(int64_t)t * 256 + (u0 >> 8)] = pm;
    }
    if (in && !fin) {
      // NaN/Inf patterns: W~ = NaN, hard index 0 (R10).  Finite patterns are written in phase 3 when
      // populated; absent ones are never read (round 1 NaN-filled all 65,536 entries of the three
      // tables of every tensor: 104 MB of stores per CFG3 step)
      const float nanf = __int_as_float(0x7FC00000);
      float4* t4 = reinterpret_cast<float4*>(tab + u0);
#pragma unroll
      for (int q = 0; q < 4; ++q) t4[q] = make_float4(nanf, nanf, nanf, nanf);
      const uint32_t n16 = nan16(P.wdtype) * 0x10001u;
      uint4* h4 = reinterpret_cast<uint4*>(tab16 + u0);
      h4[0] = make_uint4(n16, n16, n16, n16);
      h4[1] = make_uint4(n16, n16, n16, n16);
      *reinterpret_cast<uint4*>(idx + u0) = make_uint4(0, 0, 0, 0);
    }
    // block exclusive scan of the per-thread populated counts
    const int np = __popc(popmask);
    int incl = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_scan[warp] = incl;
    __syncthreads();
    int woff = 0, btot = 0;
    for (int w = 0; w < (kFThreads / 32); ++w) {
      const int x = s_scan[w];
      woff += (w < warp) ? x : 0;
      btot += x;
    }
    int pos = nr + woff + incl - np;
    if (popmask) {  // the rows, and their value and count staged in shared memory (no re-read)
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (popmask & (1u << e)) {
          EDKM_BCHECK(pos < end - base && u0 + e < end);
          rows[pos] = (uint16_t)(u0 + e);
          if (pos < kStage) {
            stage_v[pos] = decode16f(u0 + e, P.wdtype);
            stage_n[pos] = c[e];
          }
          ++pos;
        }
    }
    nr += btot;
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) nonfin += __shfl_xor_sync(0xffffffffu, nonfin, o);
  if (lane == 0) s_nf[warp] = nonfin;
  __syncthreads();  // also orders the rows[] writes before staging
  if (tid == 0) {
    long long s = 0;
    for (int w = 0; w < (kFThreads / 32); ++w) s += s_nf[w];
    st->nonfinite[crank] = s;
    EDKM_BCHECK(nr >= 0 && nr <= end - base);
    st->nrows[crank] = nr;
    if (crank == 0) {
      st->cl = cl;
      for (int r = 0; r <= cl; ++r) st->pbase[r] = s_pb[r];
    }
  }
  if (P.layout_only) {  // a rank that does not own this tensor: its layout, from the global counts
    cluster.sync();
    table_windows(P.page_cnt + (int64_t)t * 256, st, crank);
    return;
  }
  RowStage R{rows, cnt, stage_v, stage_n, nullptr, nullptr, nr, P.wdtype, kStage};  // staged by the compaction

  // ---- 2. unrolled centroid updates
  const int stride_c = (P.max_iter + 1) * K, stride_s = (P.max_iter > 0 ? P.max_iter : 1) * K;
  double* ctraj = P.ctraj + (int64_t)t * stride_c;
  double* straj = P.straj + (int64_t)t * stride_s;
  if (tid < K) {
    sCb[0][tid] = (double)P.C0[(int64_t)t * K + tid];
    if (crank == 0) ctraj[tid] = sCb[0][tid];
  }
  __syncthreads();
  int T = P.max_iter;
  if (P.max_iter > 0) cs.prepare(sCb[0], P.inv_tau);
  __syncthreads();
  // Per iteration: the row loop, one CTA barrier + one cluster barrier for the sums, the centroid
  // update by K threads straight from the cluster's partial sums, one barrier, the next
  // iteration's tables, one barrier (round 2: five CTA barriers before).
  for (int it = 0; it < P.max_iter; ++it) {
    const double* sC = sCb[it & 1];
    double* sCn = sCb[(it + 1) & 1];
    double* red_w = red + warp * 2 * K;
    warp_zero<2 * K>(red_w);
    // warp-uniform blocks of at most kRowFlush rows per lane: S_j, M_j partials in fp32, then
    // fp64 (R7); lane l of warp w takes rows w*32 + l + i*kFThreads
    for (int rb = warp * 32; rb < nr; rb += kRowFlush * kFThreads) {
      float af[2 * K];
#pragma unroll
      for (int j = 0; j < 2 * K; ++j) af[j] = 0.0f;
      const int r1 = min(nr, rb + kRowFlush * kFThreads);
      auto row = [&](float v, float n) {
        float A[K];
        int m;
        // 1/Z applied to the count (n/Z, n v/Z) instead of to each A_j
        const float nz = n * attention_row_raw<K>(v, cs, A, m), nvz = nz * v;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          af[j] = fmaf(A[j], nz, af[j]);
          af[K + j] = fmaf(A[j], nvz, af[K + j]);
        }
      };
      if (r1 <= R.ns) {  // staged rows (the usual case): shared memory only
        for (int r = rb + lane; r < r1; r += kFThreads) {
          EDKM_BCHECK(r < R.ns && r < nr);
          row(R.sv[r], (float)R.sn[r]);
        }
      } else {
        for (int r = rb + lane; r < r1; r += kFThreads) row(R.vf(r), R.nf(r));
      }
      warp_flush<2 * K>(af, red_w);
    }
    // the CTA's sums (warp order), then the cluster's (CTA order) read by the K updating threads
    __syncthreads();
    double* mine = part + (it & 1) * 2 * K;
    if (tid < 2 * K) {
      double x = 0.0;
      for (int w = 0; w < kFThreads / 32; ++w) x += red[w * 2 * K + tid];
      mine[tid] = x;
    }
    cluster.sync();
    if (tid < K) {
      double S = 0.0, M = 0.0;
      for (unsigned r = 0; r < cluster.num_blocks(); ++r) {
        const double* q = cluster.map_shared_rank(mine, r);
        S += q[tid];
        M += q[K + tid];
      }
      const double cn = (S != 0.0) ? M / S : sC[tid];
      sCn[tid] = cn;
      sDelta[tid] = fabs(cn - sC[tid]);
      if (crank == 0) {
        ctraj[(int64_t)(it + 1) * K + tid] = cn;
        straj[(int64_t)it * K + tid] = S;
      }
    }
    __syncthreads();
    double dmax = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) dmax = fmax(dmax, sDelta[j]);
    if (P.eps > 0.0 && dmax <= P.eps) {  // identical on every CTA of the cluster
      T = it + 1;
      break;
    }
    if (it + 1 < P.max_iter) cs.prepare(sCn, P.inv_tau);  // sDelta is rewritten only after the next barrier
    __syncthreads();
  }
  const double* sC = sCb[T & 1];
  if (crank == 0 && tid == 0) st->T = T;
  if (tid < K) {
    const float cf = (float)sC[tid];
    if (crank == 0) P.C_out[(int64_t)t * K + tid] = cf;
    sCf[tid] = (double)cf;  // the deployable fp32 lookup table (R9)
  }
  cs.prepare(sC, P.inv_tau);
  __syncthreads();

  // ---- 3. per populated pattern: W~ (fp32 and 16-bit), hard index vs the fp32 C_out
  for (int r = tid; r < nr; r += kFThreads) {
    const uint32_t u = rows[r];
    EDKM_BCHECK((int)u >= base && (int)u < end);
    const double v = R.v(r);
    int best = 0;
    double bd = (v - sCf[0]) * (v - sCf[0]);
#pragma unroll
    for (int j = 1; j < K; ++j) {
      const double d = (v - sCf[j]) * (v - sCf[j]);
      if (d < bd) { bd = d; best = j; }
    }
    idx[u] = (uint8_t)best;
    float A[K];
    attention_row<K>((float)v, cs, A);
    double wt = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) wt = fma((double)A[j], cs.c[j], wt);
    tab[u] = (float)wt;
    tab16[u] = round16(wt, P.wdtype);
  }
  cluster.sync();  // keep this CTA's shared memory alive until the cluster is done with it; page masses complete
  table_windows(P.page_cnt + (int64_t)t * 256, st, crank);
}

// ============================================================================ TGAMMA
template <int K>
#ifndef EDKM_TG_MB16
#define EDKM_TG_MB16 3  // k = 16: three CTAs per SM (CFG4 TGAMMA 0.116 -> 0.106 ms; 4: 0.111, spills)
#endif
#ifndef EDKM_TG_BATCH
#define EDKM_TG_BATCH 4
#endif
__global__ void __launch_bounds__(kFThreads, K <= 8 ? 4 : EDKM_TG_MB16) tgamma_kernel(const TableArgs P) {
  cg::cluster_group cluster = cg::this_cluster();
  const int cl = P.cl, crank = (int)cluster.block_rank(), t = blockIdx.x / cl, tid = threadIdx.x;
  __shared__ double red[(kFThreads / 32) * K], part[2 * K], tot[K];
  __shared__ CSet<K> cs;
  const TensorState* st = P.state + t;
  const int T = st->T, pcl = st->cl;
  cs.prepare(P.ctraj + (int64_t)t * (P.max_iter + 1) * K + (int64_t)T * K, P.inv_tau);
  __syncthreads();
  const double* sC = cs.c;
  const double* Bt = P.B + (int64_t)t * kPatterns;
  double acc[K];
#pragma unroll
  for (int l = 0; l < K; ++l) acc[l] = 0.0;
  for (int p = crank; p < pcl; p += cl) {
    const uint16_t* rows = P.rows + (int64_t)t * kPatterns + st->pbase[p];
    const int nr = st->nrows[p];
    // NB rows per thread per step: their pattern and bucket loads are issued together (the
    // kernel is bound by these dependent global loads otherwise)
    constexpr int NB = EDKM_TG_BATCH;
    for (int r0 = tid; r0 < nr; r0 += NB * kFThreads) {
      uint32_t uq[NB];
      double Bq[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) uq[q] = r0 + q * kFThreads < nr ? (uint32_t)rows[r0 + q * kFThreads] : 0u;
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        EDKM_BCHECK(uq[q] < (uint32_t)kPatterns);
        Bq[q] = r0 + q * kFThreads < nr ? Bt[uq[q]] : 0.0;
      }
#pragma unroll 1
      for (int q = 0; q < NB; ++q) {
        const uint32_t u = uq[q];
        const double B = Bq[q];
        if (B == 0.0) continue;
        const double v = decode16(u, P.wdtype);
        float Af[K];
        attention_row<K>((float)v, cs, Af);
        double A[K], wt = 0.0;
#pragma unroll
        for (int l = 0; l < K; ++l) {
          A[l] = (double)Af[l];
          wt = fma(A[l], sC[l], wt);
        }
#pragma unroll
        for (int l = 0; l < K; ++l) acc[l] += B * A[l] * (1.0 + (sC[l] - wt) * 2.0 * (v - sC[l]) * P.inv_tau);
      }
    }
  }
  cluster_allreduce<K, kFThreads / 32>(acc, red, part, tot, 0, cluster);
  if (crank == 0 && tid < K) P.gamma[(int64_t)t * K + tid] = tot[tid];
  cluster.sync();
}

// ============================================================================ TB
// Per-iteration constants of the reverse loop in the forms one row needs, all derived in fp64 and
// rounded once.  With m the row's nearest centroid (the one attention_row reduces against):
//   gh'_j = gh_j - gh_m = (g1_j - g1_m) v - (g2_j - g2_m),  gh_j = g1_j v - g2_j = dL/dA_t[u][j],
//   dz_l  = h1 (v - C_t[l]) = dzm + h1 (C_t[m] - C_t[l]),    dzm = h1 (v - C_t[m]) (float-float),
// g1_j = G_j / S_j, g2_j = g1_j C_{t+1}[j], h1 = 2/tau.  The softmax Jacobian only sees gh up to a
// constant, so gh' gives the same rr_l = A_l (gh_l - sum_j A_j gh_j) when sum_j A_j = 1 -- and when
// it is not (fp32 normalisation) the constant gh_m no longer leaks in; gh'_m = 0 exactly and dzm is
// accurate where v is near C_t[m], the row's largest attention (R7; tools/exp_tb_fp32.py).
template <int K>
struct BSet {
  float g1[K];
  float g1d[K][K], g2d[K][K], dh[K][K];
  float h2hi[K], h2lo[K];
  // every thread of the block calls it; the caller synchronises before and after
  __device__ void prepare(const double* G, const double* cn, const double* S, const double* c, float h1f) {
    const int t = threadIdx.x;
    if (t < K * K) {
      const int m = t / K, j = t % K;
      const double ism = S[m] != 0.0 ? 1.0 / S[m] : 0.0, isj = S[j] != 0.0 ? 1.0 / S[j] : 0.0;
      const double g1m = G[m] * ism, g1j = G[j] * isj;
      g1d[m][j] = (float)(g1j - g1m);
      g2d[m][j] = (float)(g1j * cn[j] - g1m * cn[m]);
      dh[m][j] = (float)((double)h1f * (c[m] - c[j]));
    }
    if (t < K) {
      const double is = S[t] != 0.0 ? 1.0 / S[t] : 0.0;
      g1[t] = (float)(G[t] * is);
      const double h = (double)h1f * c[t];
      h2hi[t] = (float)h;
      h2lo[t] = (float)(h - (double)h2hi[t]);
    }
  }
};

// One row of the reverse loop at iteration t, in fp32 (R7): adds n * q_l to af[l] (the row's
// contribution to dL/dC_t[l]) and returns the row's psi increment (dL/dv through A_t and M_t).
//   A = softmax attention (unnormalised here, 1/Z applied to the three sums that use it)
//   rr_l = A_l (gh_l - sum_j A_j gh_j),  q_l = rr_l dz_l,  dpsi = sum_j A_j g1_j - sum_l q_l
template <int K>
__device__ __forceinline__ float tb_row(float v, float n, const CSet<K>& cs, const BSet<K>& bs, float h1f,
                                        float (&af)[K]) {
  float A[K];
  int m;
  const float iz = attention_row_raw<K>(v, cs, A, m);
  const float* g1r = bs.g1d[m];
  const float* g2r = bs.g2d[m];
  const float* dhr = bs.dh[m];
  float gh[K], p[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    gh[j] = fmaf(g1r[j], v, -g2r[j]);  // gh'_j (zero where S_t[j] = 0 and S_t[m] = 0)
    p[j] = A[j] * gh[j];
  }
  const float dsum = dot4<K>(A, bs.g1);  // sum_j A_j g1_j: the direct path of v through M_t
  const float s = sum4<K>(p) * iz;
  const float dzm = fmaf(h1f, v, -bs.h2hi[m]) - bs.h2lo[m];
  const float niz = n * iz;
#pragma unroll
  for (int l = 0; l < K; ++l) {
    const float q = fmaf(-A[l], s, p[l]) * (dzm + dhr[l]);  // Z * rr_l * dz_l
    p[l] = q;
    af[l] = fmaf(niz, q, af[l]);
  }
  return iz * (dsum - sum4<K>(p));
}

// Reverse loop t = T-1..0: psi[u] and dC_0; then the (phi, psi) table.  The running psi is kept
// in shared memory next to the staged rows (kPsiShared, 16 B per staged row: k = 16, two CTAs
// per SM at 128 registers) or in global memory (8 B per staged row, L2-resident: k <= 8, four
// CTAs per SM; CFG3 k = 8 TB 0.241 -> 0.217 ms, CFG4 k = 4 1.79 -> 1.43 ms in round 2).
template <int K, int kStageB, int kMinBlocks, bool kPsiShared>
__global__ void __launch_bounds__(kBThreads, kMinBlocks) tb_kernel(const TableArgs P) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double stage_mem[];
  const int cl = P.cl, crank = (int)cluster.block_rank(), t = blockIdx.x / cl, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  __shared__ double sG[K], sInvS[K], red[(kBThreads / 32) * K], part[2 * K];
  __shared__ CSet<K> cs;
  __shared__ BSet<K> bs;
  const double* sCt = cs.c;
  const TensorState* st = P.state + t;
  const int T = st->T, pcl = st->cl;
  const int32_t* cnt = P.counts + (int64_t)t * kPatterns;
  const double* ctraj = P.ctraj + (int64_t)t * (P.max_iter + 1) * K;
  const double* straj = P.straj + (int64_t)t * (P.max_iter > 0 ? P.max_iter : 1) * K;
  double* psi = P.psi + (int64_t)t * kPatterns;
  // this CTA owns partitions p = crank, crank + cl, ...; with pcl == cl (always, same
  // heuristic in TF) that is the single partition `crank`, staged in shared memory
  const bool one = pcl == cl;
  const int pb0 = one ? st->pbase[crank] : 0;
  double* vn_mem = kPsiShared ? stage_mem + kStageB : stage_mem;
  RowStage R{P.rows + (int64_t)t * kPatterns + pb0, cnt, reinterpret_cast<float*>(vn_mem),
             reinterpret_cast<int32_t*>(vn_mem) + kStageB, kPsiShared ? stage_mem : nullptr, psi + pb0,
             one ? st->nrows[crank] : 0, P.wdtype, kStageB};
  if (one) R.stage();
  if (tid < K) sG[tid] = P.gamma[(int64_t)t * K + tid];
  // the iteration's C_t, C_{t+1} and S_t, copied to shared memory one iteration ahead (cp.async,
  // no registers held across the row loop): the per-iteration tables are then built from shared
  // memory instead of from dependent L2 loads (ncu r02: 8% of TB<16>'s stall samples)
  __shared__ __align__(16) double sTr[2][3 * K];
  auto fetch = [&](int it, int buf) {
    if (tid < 3 * K) {
      EDKM_BCHECK(buf == 0 || buf == 1);
      const double* src = tid < K ? ctraj + (int64_t)it * K + tid
                                  : tid < 2 * K ? ctraj + (int64_t)(it + 1) * K + (tid - K) : straj + (int64_t)it * K + (tid - 2 * K);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(&sTr[buf][tid])), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (T > 0) fetch(T - 1, 0);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const float h1f = (float)(2.0 * P.inv_tau);
  for (int it = T - 1; it >= 0; --it) {
    const int buf = (T - 1 - it) & 1;
    if (it > 0) fetch(it - 1, buf ^ 1);  // the other buffer: last read by the previous iteration's tables
    const double* tr = sTr[buf];
    cs.prepare(tr, P.inv_tau);
    bs.prepare(sG, tr + K, tr + 2 * K, tr, h1f);
    if (tid < K) {
      const double S = tr[2 * K + tid];
      sInvS[tid] = S != 0.0 ? 1.0 / S : 0.0;
    }
    __syncthreads();
    double* red_w = red + warp * K;
    warp_zero<K>(red_w);
    for (int p = crank; p < pcl; p += cl) {
      const uint16_t* rows = P.rows + (int64_t)t * kPatterns + st->pbase[p];
      double* gpsi = psi + st->pbase[p];
      const int nr = one ? R.nr : st->nrows[p];
      // warp-uniform blocks of at most kRowFlush rows per lane: the n-weighted sums in fp32,
      // then fp64 (R7); lane l of warp w takes rows w*32 + l + i*kBThreads
      for (int rb = warp * 32; rb < nr; rb += kRowFlush * kBThreads) {
        float af[K];
#pragma unroll
        for (int l = 0; l < K; ++l) af[l] = 0.0f;
        const int r1 = min(nr, rb + kRowFlush * kBThreads);
        if (one && r1 <= R.ns) {  // staged rows (the usual case)
          for (int r = rb + lane; r < r1; r += kBThreads) {
            EDKM_BCHECK(r < R.ns && r < R.nr);
            double& ps = kPsiShared ? R.spsi[r] : gpsi[r];
            const double ps_old = it == T - 1 ? 0.0 : ps;  // issued before the row's arithmetic
            ps = ps_old + (double)tb_row<K>(R.sv[r], (float)R.sn[r], cs, bs, h1f, af);
          }
        } else {
          for (int r = rb + lane; r < r1; r += kBThreads) {
            const float v = one ? R.vf(r) : decode16f(rows[r], P.wdtype);
            const float n = one ? R.nf(r) : (float)cnt[rows[r]];
            double& ps = (kPsiShared && one) ? R.psi(r) : gpsi[r];
            const double ps_old = it == T - 1 ? 0.0 : ps;
            ps = ps_old + (double)tb_row<K>(v, n, cs, bs, h1f, af);
          }
        }
        warp_flush<K>(af, red_w);
      }
    }
    // the CTA's sums (warp order), then the cluster's (CTA order) read by the K updating threads
    __syncthreads();
    double* mine = part + (it & 1) * K;
    if (tid < K) {
      double x = 0.0;
      for (int w = 0; w < kBThreads / 32; ++w) x += red[w * K + tid];
      mine[tid] = x;
    }
    cluster.sync();
    if (tid < K) {
      double g = 0.0;
      for (unsigned r = 0; r < cluster.num_blocks(); ++r) g += cluster.map_shared_rank(mine, r)[tid];
      sG[tid] = g + (sInvS[tid] == 0.0 ? sG[tid] : 0.0);  // C_{t+1} = C_t where S_t = 0
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // the next iteration's trajectories
    __syncthreads();
  }
  if (crank == 0 && tid < K) P.dC0[(int64_t)t * K + tid] = (float)sG[tid];
  // (phi, psi) table: phi[u] = (2/tau) sum_l A_T[u,l] (C_T[l] - W~_u)^2
  cs.prepare(ctraj + (int64_t)T * K, P.inv_tau);
  __syncthreads();
  float2* pp = P.phipsi + (int64_t)t * kPatterns;
  for (int p = crank; p < pcl; p += cl) {
    const uint16_t* rows = P.rows + (int64_t)t * kPatterns + st->pbase[p];
    double* gpsi = psi + st->pbase[p];
    const int nr = one ? R.nr : st->nrows[p];
    for (int r = tid; r < nr; r += kBThreads) {
      const uint32_t u = rows[r];
      EDKM_BCHECK((int)u >= st->pbase[p] && (int)u < st->pbase[p + 1]);
      const double v = one ? R.v(r) : decode16(u, P.wdtype);
      float Af[K];
      attention_row<K>((float)v, cs, Af);
      double wt = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) wt = fma((double)Af[l], sCt[l], wt);
      double var = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) var += (double)Af[l] * (sCt[l] - wt) * (sCt[l] - wt);
      const double ps = T > 0 ? ((kPsiShared && one) ? R.psi(r) : gpsi[r]) : 0.0;
      pp[u] = make_float2((float)(2.0 * P.inv_tau * var), (float)ps);
    }
    // NaN/Inf patterns: (phi, psi) = NaN, so dW = NaN (R10).  Absent finite patterns are left as
    // they are: B2 gathers only the patterns of its weights (round 1 NaN-filled every absent
    // pattern, reading all 65,536 counts per tensor: ~28 us of CFG3's 0.18 ms TB).
    const float2 nan2 = make_float2(__int_as_float(0x7FC00000), __int_as_float(0x7FC00000));
    const int nf0 = P.wdtype == kBF16 ? 0x7F80 : 0x7C00;  // first non-finite pattern of each sign
    for (int h = 0; h < 2; ++h) {
      const int lo = max(st->pbase[p], h * 0x8000 + nf0), hi = min(st->pbase[p + 1], h * 0x8000 + 0x8000);
      for (int u = lo + tid; u < hi; u += kBThreads) {
        EDKM_BCHECK(u >= st->pbase[p] && u < st->pbase[p + 1] && !pattern_finite(u, P.wdtype));
        pp[u] = nan2;
      }
    }
  }
  cluster.sync();
}

// ============================================================================ launchers
// CTAs per tensor (row partitions, <= the portable cluster size 8): fill the GPU for small nt,
// else 2 for bf16 and 4 for fp16.  Rows are balanced across the partitions, but each CTA pays
// fixed costs per iteration (centroid tables, cluster reduction), so for bf16 (U ~ 5K per
// tensor) more, smaller partitions measured slower for 226 tensors (cl = 5: TF 0.15 -> 0.26 ms,
// TB 0.27 -> 0.47 ms on CFG3).  fp16 tensors have ~5x the rows (U ~ 24K): with cl = 4 and TB's
// two-CTAs-per-SM shape, CFG4 (k = 16) TB 4.06 -> 3.76 ms, k = 4 TB 1.93 -> 1.79 ms.
#ifndef EDKM_CL_FP16
#define EDKM_CL_FP16 4
#endif
#ifndef EDKM_CL_BF16
#define EDKM_CL_BF16 2
#endif
int table_cluster_size(int nt, int wdtype) {
  if (nt <= 18) return 8;
  if (nt <= 37) return 4;
  return wdtype == kFP16 ? EDKM_CL_FP16 : EDKM_CL_BF16;
}

template <class Fn>
static cudaError_t launch_table(const TableArgs& P, cudaStream_t s, Fn fn, size_t smem, int threads) {
  if (P.nt == 0) return cudaSuccess;
  if (smem) {
    cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P.nt * P.cl));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)P.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, P);
}

#define EDKM_TABLE_LAUNCH(NAME, KERNEL, SMEM, NT)              \
  cudaError_t NAME(const TableArgs& P, cudaStream_t s) {         \
    switch (P.k) {                                               \
      case 2: return launch_table(P, s, KERNEL<2>, SMEM, NT);    \
      case 4: return launch_table(P, s, KERNEL<4>, SMEM, NT);    \
      case 8: return launch_table(P, s, KERNEL<8>, SMEM, NT);    \
      case 16: return launch_table(P, s, KERNEL<16>, SMEM, NT);  \
      default: return cudaErrorInvalidValue;                     \
    }                                                            \
  }

#ifndef EDKM_TF16_MB
#define EDKM_TF16_MB 3
#endif
template <int K>
static cudaError_t launch_tf_k(const TableArgs& P, cudaStream_t s) {
  if (P.wdtype == kBF16)
    return launch_table(P, s, tf_kernel<K, kStageFS, 4>, (size_t)kStageFS * 8, kFThreads);
  // fp16: ~6K rows per CTA at cl = 4; four CTAs per SM where k <= 8 fits 64 registers
  return launch_table(P, s, tf_kernel<K, kStageFL, (K <= 8 ? 4 : EDKM_TF16_MB)>, (size_t)kStageFL * 8, kFThreads);
}

cudaError_t launch_tf(const TableArgs& P, cudaStream_t s) {
  switch (P.k) {
    case 2: return launch_tf_k<2>(P, s);
    case 4: return launch_tf_k<4>(P, s);
    case 8: return launch_tf_k<8>(P, s);
    case 16: return launch_tf_k<16>(P, s);
    default: return cudaErrorInvalidValue;
  }
}
EDKM_TABLE_LAUNCH(launch_tgamma, tgamma_kernel, 0, kFThreads)
// TB variant per k (measured, S4): k <= 8 keep psi in global memory and run four CTAs
// per SM; k = 16 (128 registers) keeps psi staged in shared memory at two CTAs per SM.
#ifndef EDKM_TB16_MB
#define EDKM_TB16_MB 2
#endif
template <int K>
static cudaError_t launch_tb_k(const TableArgs& P, cudaStream_t s) {
  if constexpr (K <= 8) {
    if (P.wdtype == kBF16)
      return launch_table(P, s, tb_kernel<K, kStageB16, 4, false>, (size_t)kStageB16 * 8, kBThreads);
    return launch_table(P, s, tb_kernel<K, kStageB32, 4, false>, (size_t)kStageB32 * 8, kBThreads);
  } else {
    constexpr int MB = EDKM_TB16_MB;
    constexpr bool PS = MB <= 2;  // psi staged next to the rows only at two CTAs per SM
    if (P.wdtype == kBF16)
      return launch_table(P, s, tb_kernel<K, kStageB16, MB, PS>, (size_t)kStageB16 * (PS ? 16 : 8), kBThreads);
    return launch_table(P, s, tb_kernel<K, kStageB32, MB, PS>, (size_t)kStageB32 * (PS ? 16 : 8), kBThreads);
  }
}

cudaError_t launch_tb(const TableArgs& P, cudaStream_t s) {
  switch (P.k) {
    case 2: return launch_tb_k<2>(P, s);
    case 4: return launch_tb_k<4>(P, s);
    case 8: return launch_tb_k<8>(P, s);
    case 16: return launch_tb_k<16>(P, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace edkm
