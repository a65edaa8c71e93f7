// table_wide.cu -- table phase for k = 32..256 centroids (bits 5..8; the paper compresses the
// embeddings at 8 bits, P:91 S3.1).  Same mathematics as table_kernels.cu (S4), laid
// out one warp per pattern row: lane l owns centroids j = l, l+32, ..., so per-centroid state
// stays in registers for any k, and the k-wide sums of a row are warp shuffles.
//
//   TF      forward iterations + W~ table + hard-index table
//   TGAMMA  gamma_T from the gradient buckets
//   TB      reverse loop -> (phi, psi) per pattern and dC_0
//
// Reductions: per lane in row order, across warps in warp order, across the cluster in CTA
// order -- deterministic.  Precision as in table_kernels.cu (R7): logit differences from fp64
// centroid sums/differences, exp2 of the fraction in fp32, the power of two and all sums fp64.
#include <cooperative_groups.h>

#include "common.cuh"
#include "launch.h"
#include "table_common.cuh"

namespace cg = cooperative_groups;

namespace edkm {

constexpr int kWThreads = 512;
constexpr int kWWarps = kWThreads / 32;
constexpr int kWStage = 2048;  // rows per CTA staged in shared memory (v, n, psi)

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ float warp_sumf(float x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Attention of value v (fp32-exact) to the K centroids c[] (fp64 in shared memory); lane owns
// j = lane + 32 q.  Returns normalised fp64 A[q].
template <int K>
__device__ __forceinline__ void attention_w(double v, const double* c, const float* chi, float sc,
                                            double (&A)[K / 32]) {
  constexpr int J = K / 32;
  const int lane = threadIdx.x & 31;
  const float vf = (float)v;
  float am = INFINITY;
  int jm = 0;
#pragma unroll
  for (int q = 0; q < J; ++q) {
    const float a = fabsf(vf - chi[lane + 32 * q]);
    if (a < am) { am = a; jm = lane + 32 * q; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {  // warp argmin, lowest index on ties
    const float a2 = __shfl_xor_sync(0xffffffffu, am, o);
    const int j2 = __shfl_xor_sync(0xffffffffu, jm, o);
    if (a2 < am || (a2 == am && j2 < jm)) { am = a2; jm = j2; }
  }
  const double cm = c[jm], v2 = 2.0 * v;
  float a[J];
  int ne[J];
  float zp = 0.0f;
#pragma unroll
  for (int q = 0; q < J; ++q) {
    const double cj = c[lane + 32 * q];
    const float y = (float)((cm - cj) * (v2 - cm - cj)) * sc;  // (d_j - d_m)/tau in base 2
    const float n = floorf(y);
    ne[q] = (int)n;
    a[q] = exp2f(n - y);
    zp += ne[q] < 126 ? __int_as_float((127 - ne[q]) << 23) * a[q] : 0.0f;
  }
  const float iz = 1.0f / warp_sumf(zp);
#pragma unroll
  for (int q = 0; q < J; ++q) {
    const double p2 = ne[q] > 1022 ? 0.0 : __longlong_as_double((long long)(1023 - ne[q]) << 52);
    A[q] = (double)(a[q] * iz) * p2;
  }
}

// Sum NV per-lane vectors of J doubles (entry j = lane + 32 q of vector w at v[w][q]) over the
// block and the cluster; result tot[w * K + j] on every CTA.  red: [kWWarps][NV*K], part: [2][NV*K].
template <int K, int NV>
__device__ __forceinline__ void cluster_allreduce_w(double (&v)[NV][K / 32], double* red, double* part, double* tot,
                                                    int parity, cg::cluster_group& cluster) {
  constexpr int J = K / 32, N = NV * K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int w = 0; w < NV; ++w)
#pragma unroll
    for (int q = 0; q < J; ++q) red[warp * N + w * K + lane + 32 * q] = v[w][q];
  __syncthreads();
  double* mine = part + parity * N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kWWarps; ++w) s += red[w * N + i];
    mine[i] = s;
  }
  cluster.sync();
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double s = 0.0;
    for (unsigned r = 0; r < cluster.num_blocks(); ++r) s += cluster.map_shared_rank(mine, r)[i];
    tot[i] = s;
  }
  __syncthreads();
}

template <int K>
struct WideSmem {
  double c[K], cn[K], cf[K], invS[K], g[K];
  float chi[K];
  double red[kWWarps * 2 * K];
  double part[2 * 2 * K];
  double tot[2 * K];
  double sv[kWStage], sn[kWStage], spsi[kWStage];
  int scan[kWWarps];
  long long nf[kWWarps];
  int flag;
};

template <int K>
__device__ __forceinline__ void load_c(WideSmem<K>& S, const double* src) {
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    S.c[j] = src[j];
    S.chi[j] = (float)src[j];
  }
}

// ============================================================================ TF (wide)
template <int K>
__global__ void __launch_bounds__(kWThreads) tf_wide_kernel(const TableArgs P) {
  constexpr int J = K / 32;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char wsm[];
  WideSmem<K>& S = *reinterpret_cast<WideSmem<K>*>(wsm);
  const int cl = P.cl, crank = (int)cluster.block_rank(), t = blockIdx.x / cl, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  __shared__ int s_pg[256], s_pref[257], s_pb[kMaxCluster + 1];
  const int32_t* cnt = P.counts + (int64_t)t * kPatterns;
  table_partitions<kWThreads>(cnt, P.wdtype, P.page_cnt + (int64_t)t * 256, cl, crank, cluster, s_pg, s_pref, s_pb);
  const int base = s_pb[crank], end = s_pb[crank + 1];
  uint16_t* rows = P.rows + (int64_t)t * kPatterns + base;
  TensorState* st = P.state + t;
  float* tab = P.table + (int64_t)t * kPatterns;
  uint16_t* tab16 = P.table16 + (int64_t)t * kPatterns;
  uint8_t* idx = P.idx8 + (int64_t)t * kPatterns;
  const float nanf = __int_as_float(0x7FC00000);

  // ---- 1. compaction of this partition (one pattern per thread per step), NaN entries of the non-finite patterns
  int nr = 0;
  long long nonfin = 0;
  for (int off = 0; off < end - base; off += kWThreads) {
    const int u = base + off + tid;
    const bool in = u < end;
    const int c = in ? cnt[u] : 0;
    const bool fin = pattern_finite(u, P.wdtype);
    const bool pop = in && fin && c > 0;
    if (!fin) nonfin += c;
    if (in && !fin) {  // NaN/Inf patterns (R10); populated finite ones are set in phase 3, absent ones never read
      idx[u] = 0;
      tab[u] = nanf;
      tab16[u] = nan16(P.wdtype);
    }
    const unsigned b = __ballot_sync(0xffffffffu, pop);
    if (lane == 0) S.scan[warp] = __popc(b);
    __syncthreads();
    int woff = 0, btot = 0;
    for (int w = 0; w < kWWarps; ++w) {
      woff += (w < warp) ? S.scan[w] : 0;
      btot += S.scan[w];
    }
    if (pop) rows[nr + woff + __popc(b & ((1u << lane) - 1u))] = (uint16_t)u;
    nr += btot;
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) nonfin += __shfl_xor_sync(0xffffffffu, nonfin, o);
  if (lane == 0) S.nf[warp] = nonfin;
  __syncthreads();
  if (tid == 0) {
    long long s = 0;
    for (int w = 0; w < kWWarps; ++w) s += S.nf[w];
    st->nonfinite[crank] = s;
    st->nrows[crank] = nr;
    if (crank == 0) {
      st->cl = cl;
      for (int r = 0; r <= cl; ++r) st->pbase[r] = s_pb[r];
    }
  }
  if (P.layout_only) {  // a rank that does not own this tensor: its layout, from the global counts
    cluster.sync();
    table_windows(P.page_cnt + (int64_t)t * 256, P.state + t, crank);
    return;
  }
  for (int r = tid; r < nr && r < kWStage; r += kWThreads) {
    const uint32_t u = rows[r];
    S.sv[r] = decode16(u, P.wdtype);
    S.sn[r] = (double)cnt[u];
  }

  // ---- 2. iterations (warp per row)
  const int stride_c = (P.max_iter + 1) * K, stride_s = (P.max_iter > 0 ? P.max_iter : 1) * K;
  double* ctraj = P.ctraj + (int64_t)t * stride_c;
  double* straj = P.straj + (int64_t)t * stride_s;
  for (int j = tid; j < K; j += kWThreads) {
    const double c0 = (double)P.C0[(int64_t)t * K + j];
    S.c[j] = c0;
    S.chi[j] = (float)c0;
    if (crank == 0) ctraj[j] = c0;
  }
  __syncthreads();
  const float sc = (float)(P.inv_tau * 1.4426950408889634);
  int T = P.max_iter;
  for (int it = 0; it < P.max_iter; ++it) {
    double acc[2][J];
#pragma unroll
    for (int q = 0; q < J; ++q) acc[0][q] = acc[1][q] = 0.0;
    for (int r = warp; r < nr; r += kWWarps) {
      const double v = r < kWStage ? S.sv[r] : decode16(rows[r], P.wdtype);
      const double n = r < kWStage ? S.sn[r] : (double)cnt[rows[r]];
      double A[J];
      attention_w<K>(v, S.c, S.chi, sc, A);
#pragma unroll
      for (int q = 0; q < J; ++q) {
        acc[0][q] = fma(A[q], n, acc[0][q]);
        acc[1][q] = fma(A[q], n * v, acc[1][q]);
      }
    }
    cluster_allreduce_w<K, 2>(acc, S.red, S.part, S.tot, it & 1, cluster);
    // identical on every thread: new centroids, max shift
    double dmax = 0.0;
    for (int j = 0; j < K; ++j) {
      const double Sj = S.tot[j];
      const double cn = (Sj != 0.0) ? S.tot[K + j] / Sj : S.c[j];
      dmax = fmax(dmax, fabs(cn - S.c[j]));
    }
    __syncthreads();
    for (int j = tid; j < K; j += kWThreads) {
      const double Sj = S.tot[j];
      const double cn = (Sj != 0.0) ? S.tot[K + j] / Sj : S.c[j];
      if (crank == 0) {
        ctraj[(int64_t)(it + 1) * K + j] = cn;
        straj[(int64_t)it * K + j] = Sj;
      }
      S.cn[j] = cn;
    }
    __syncthreads();
    load_c<K>(S, S.cn);
    __syncthreads();
    if (P.eps > 0.0 && dmax <= P.eps) {
      T = it + 1;
      break;
    }
  }
  if (crank == 0 && tid == 0) st->T = T;
  for (int j = tid; j < K; j += kWThreads) {
    const float cf = (float)S.c[j];
    if (crank == 0) P.C_out[(int64_t)t * K + j] = cf;
    S.cf[j] = (double)cf;  // deployable fp32 lookup table (R9)
  }
  __syncthreads();

  // ---- 3. per populated pattern (warp per row): W~, 16-bit W~, hard index (lowest j on ties)
  for (int r = warp; r < nr; r += kWWarps) {
    const uint32_t u = rows[r];
    const double v = r < kWStage ? S.sv[r] : decode16(u, P.wdtype);
    double bd = INFINITY;
    int best = 0;
#pragma unroll
    for (int q = 0; q < J; ++q) {
      const int j = lane + 32 * q;
      const double d = (v - S.cf[j]) * (v - S.cf[j]);
      if (d < bd) { bd = d; best = j; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double d2 = __shfl_xor_sync(0xffffffffu, bd, o);
      const int j2 = __shfl_xor_sync(0xffffffffu, best, o);
      if (d2 < bd || (d2 == bd && j2 < best)) { bd = d2; best = j2; }
    }
    double A[J];
    attention_w<K>(v, S.c, S.chi, sc, A);
    double wt = 0.0;
#pragma unroll
    for (int q = 0; q < J; ++q) wt = fma(A[q], S.c[lane + 32 * q], wt);
    wt = warp_sum(wt);
    if (lane == 0) {
      idx[u] = (uint8_t)best;
      tab[u] = (float)wt;
      tab16[u] = round16(wt, P.wdtype);
    }
  }
  cluster.sync();  // page masses complete
  table_windows(P.page_cnt + (int64_t)t * 256, P.state + t, crank);
}

// ============================================================================ TGAMMA (wide)
template <int K>
__global__ void __launch_bounds__(kWThreads) tgamma_wide_kernel(const TableArgs P) {
  constexpr int J = K / 32;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char wsm[];
  WideSmem<K>& S = *reinterpret_cast<WideSmem<K>*>(wsm);
  const int cl = P.cl, crank = (int)cluster.block_rank(), t = blockIdx.x / cl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const TensorState* st = P.state + t;
  const int T = st->T, pcl = st->cl;
  load_c<K>(S, P.ctraj + (int64_t)t * (P.max_iter + 1) * K + (int64_t)T * K);
  __syncthreads();
  const float sc = (float)(P.inv_tau * 1.4426950408889634);
  const double* Bt = P.B + (int64_t)t * kPatterns;
  double acc[1][J];
#pragma unroll
  for (int q = 0; q < J; ++q) acc[0][q] = 0.0;
  for (int p = crank; p < pcl; p += cl) {
    const uint16_t* rows = P.rows + (int64_t)t * kPatterns + st->pbase[p];
    const int nr = st->nrows[p];
    for (int r = warp; r < nr; r += kWWarps) {
      const uint32_t u = rows[r];
      const double B = Bt[u];
      if (B == 0.0) continue;  // warp-uniform
      const double v = decode16(u, P.wdtype);
      double A[J];
      attention_w<K>(v, S.c, S.chi, sc, A);
      double wt = 0.0;
#pragma unroll
      for (int q = 0; q < J; ++q) wt = fma(A[q], S.c[lane + 32 * q], wt);
      wt = warp_sum(wt);
#pragma unroll
      for (int q = 0; q < J; ++q) {
        const double cl_ = S.c[lane + 32 * q];
        acc[0][q] += B * A[q] * (1.0 + (cl_ - wt) * 2.0 * (v - cl_) * P.inv_tau);
      }
    }
  }
  cluster_allreduce_w<K, 1>(acc, S.red, S.part, S.tot, 0, cluster);
  if (crank == 0)
    for (int j = threadIdx.x; j < K; j += kWThreads) P.gamma[(int64_t)t * K + j] = S.tot[j];
  cluster.sync();
}

// ============================================================================ TB (wide)
template <int K>
__global__ void __launch_bounds__(kWThreads) tb_wide_kernel(const TableArgs P) {
  constexpr int J = K / 32;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char wsm[];
  WideSmem<K>& S = *reinterpret_cast<WideSmem<K>*>(wsm);
  const int cl = P.cl, crank = (int)cluster.block_rank(), t = blockIdx.x / cl, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const TensorState* st = P.state + t;
  const int T = st->T, pcl = st->cl;
  const int32_t* cnt = P.counts + (int64_t)t * kPatterns;
  const double* ctraj = P.ctraj + (int64_t)t * (P.max_iter + 1) * K;
  const double* straj = P.straj + (int64_t)t * (P.max_iter > 0 ? P.max_iter : 1) * K;
  double* psi = P.psi + (int64_t)t * kPatterns;
  const bool one = pcl == cl;
  const uint16_t* rows0 = P.rows + (int64_t)t * kPatterns + (one ? st->pbase[crank] : 0);
  const int nr0 = one ? st->nrows[crank] : 0;
  for (int r = tid; r < nr0 && r < kWStage; r += kWThreads) {
    const uint32_t u = rows0[r];
    S.sv[r] = decode16(u, P.wdtype);
    S.sn[r] = (double)cnt[u];
  }
  for (int j = tid; j < K; j += kWThreads) S.g[j] = P.gamma[(int64_t)t * K + j];
  __syncthreads();
  const float sc = (float)(P.inv_tau * 1.4426950408889634);
  for (int it = T - 1; it >= 0; --it) {
    load_c<K>(S, ctraj + (int64_t)it * K);
    for (int j = tid; j < K; j += kWThreads) {
      S.cn[j] = ctraj[(int64_t)(it + 1) * K + j];
      const double Sj = straj[(int64_t)it * K + j];
      S.invS[j] = Sj != 0.0 ? 1.0 / Sj : 0.0;
    }
    __syncthreads();
    double acc[1][J];
#pragma unroll
    for (int q = 0; q < J; ++q) acc[0][q] = 0.0;
    for (int p = crank; p < pcl; p += cl) {
      const uint16_t* rows = P.rows + (int64_t)t * kPatterns + st->pbase[p];
      double* gpsi = psi + st->pbase[p];
      const int nr = one ? nr0 : st->nrows[p];
      for (int r = warp; r < nr; r += kWWarps) {
        const bool staged = one && r < kWStage;
        const double v = staged ? S.sv[r] : decode16(rows[r], P.wdtype);
        const double n = staged ? S.sn[r] : (double)cnt[rows[r]];
        double A[J], gh[J];
        attention_w<K>(v, S.c, S.chi, sc, A);
        double s = 0.0, dpsi = 0.0;
#pragma unroll
        for (int q = 0; q < J; ++q) {
          const int j = lane + 32 * q;
          gh[q] = S.g[j] * (v - S.cn[j]) * S.invS[j];
          s = fma(A[q], gh[q], s);
          dpsi += S.g[j] * A[q] * S.invS[j];
        }
        s = warp_sum(s);
#pragma unroll
        for (int q = 0; q < J; ++q) {
          const double rr = A[q] * (gh[q] - s);
          const double dz = 2.0 * (v - S.c[lane + 32 * q]) * P.inv_tau;
          dpsi -= rr * dz;
          acc[0][q] += n * rr * dz;
        }
        dpsi = warp_sum(dpsi);
        if (lane == 0) {
          double& ps = staged ? S.spsi[r] : gpsi[r];
          ps = (it == T - 1 ? 0.0 : ps) + dpsi;
        }
      }
    }
    cluster_allreduce_w<K, 1>(acc, S.red, S.part, S.tot, it & 1, cluster);
    for (int j = tid; j < K; j += kWThreads) S.g[j] = S.tot[j] + (S.invS[j] == 0.0 ? S.g[j] : 0.0);
    __syncthreads();
  }
  if (crank == 0)
    for (int j = tid; j < K; j += kWThreads) P.dC0[(int64_t)t * K + j] = (float)S.g[j];
  load_c<K>(S, ctraj + (int64_t)T * K);
  __syncthreads();
  float2* pp = P.phipsi + (int64_t)t * kPatterns;
  for (int p = crank; p < pcl; p += cl) {
    const uint16_t* rows = P.rows + (int64_t)t * kPatterns + st->pbase[p];
    double* gpsi = psi + st->pbase[p];
    const int nr = one ? nr0 : st->nrows[p];
    for (int r = warp; r < nr; r += kWWarps) {
      const bool staged = one && r < kWStage;
      const uint32_t u = rows[r];
      const double v = staged ? S.sv[r] : decode16(u, P.wdtype);
      double A[J];
      attention_w<K>(v, S.c, S.chi, sc, A);
      double wt = 0.0;
#pragma unroll
      for (int q = 0; q < J; ++q) wt = fma(A[q], S.c[lane + 32 * q], wt);
      wt = warp_sum(wt);
      double var = 0.0;
#pragma unroll
      for (int q = 0; q < J; ++q) {
        const double d = S.c[lane + 32 * q] - wt;
        var += A[q] * d * d;
      }
      var = warp_sum(var);
      if (lane == 0) {
        const double ps = T > 0 ? (staged ? S.spsi[r] : gpsi[r]) : 0.0;
        pp[u] = make_float2((float)(2.0 * P.inv_tau * var), (float)ps);
      }
    }
    // NaN/Inf patterns: NaN (R10); absent finite patterns are never read (as in tb_kernel)
    const int nf0 = P.wdtype == kBF16 ? 0x7F80 : 0x7C00;
    for (int h = 0; h < 2; ++h) {
      const int lo = max(st->pbase[p], h * 0x8000 + nf0), hi = min(st->pbase[p + 1], h * 0x8000 + 0x8000);
      for (int u = lo + tid; u < hi; u += kWThreads)
        pp[u] = make_float2(__int_as_float(0x7FC00000), __int_as_float(0x7FC00000));
    }
  }
  cluster.sync();
}

// ============================================================================ launchers
template <class Fn>
static cudaError_t launch_wide(const TableArgs& P, cudaStream_t s, Fn fn, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P.nt * P.cl));
  cfg.blockDim = dim3(kWThreads);
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

#define EDKM_WIDE_LAUNCH(NAME, KERNEL)                                                    \
  cudaError_t NAME(const TableArgs& P, cudaStream_t s) {                                    \
    if (P.nt == 0) return cudaSuccess;                                                      \
    switch (P.k) {                                                                          \
      case 32: return launch_wide(P, s, KERNEL<32>, sizeof(WideSmem<32>));                  \
      case 64: return launch_wide(P, s, KERNEL<64>, sizeof(WideSmem<64>));                  \
      case 128: return launch_wide(P, s, KERNEL<128>, sizeof(WideSmem<128>));               \
      case 256: return launch_wide(P, s, KERNEL<256>, sizeof(WideSmem<256>));               \
      default: return cudaErrorInvalidValue;                                                \
    }                                                                                       \
  }

EDKM_WIDE_LAUNCH(launch_tf_wide, tf_wide_kernel)
EDKM_WIDE_LAUNCH(launch_tgamma_wide, tgamma_wide_kernel)
EDKM_WIDE_LAUNCH(launch_tb_wide, tb_wide_kernel)

}  // namespace edkm
