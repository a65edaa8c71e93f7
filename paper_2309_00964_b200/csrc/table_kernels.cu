// table_kernels.cu -- the table phase of the eDKM hot path (S3).
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
// contiguous pattern partitions; k-vector sums are reduced per thread in row
// order, then by warp shuffles, across warps in warp order and across the
// cluster through DSMEM in CTA order -- deterministic, identical on every CTA.
// All arithmetic is fp64 (exp included): DESIGN.md R7 shows fp32 table-phase
// arithmetic misses the 1e-5 parity bound.  Cost is O(U k T), independent of N.
#include <cooperative_groups.h>

#include "common.cuh"
#include "launch.h"

namespace cg = cooperative_groups;

namespace edkm {

constexpr int kTThreads = 512;
constexpr int kTWarps = kTThreads / 32;

template <int K>
__device__ __forceinline__ void attention_row(double v, const double* C, double inv_tau, double (&A)[K]) {
  double d[K];
  double dmin = d[0] = (v - C[0]) * (v - C[0]);
#pragma unroll
  for (int j = 1; j < K; ++j) {
    d[j] = (v - C[j]) * (v - C[j]);
    dmin = fmin(dmin, d[j]);
  }
  double Z = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    A[j] = exp(-(d[j] - dmin) * inv_tau);
    Z += A[j];
  }
  const double iz = 1.0 / Z;
#pragma unroll
  for (int j = 0; j < K; ++j) A[j] *= iz;
}

// Sum N doubles over the CTA then over the cluster; result in tot[0..N) of every CTA.
// `part` is a [2][N] shared buffer used with alternating parity so one cluster
// barrier per call suffices.
template <int N>
__device__ __forceinline__ void cluster_allreduce(double (&v)[N], double* red, double* part, double* tot, int parity,
                                                  cg::cluster_group& cluster) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int n = 0; n < N; ++n) {
    double x = v[n];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp * N + n] = x;
  }
  __syncthreads();
  double* mine = part + parity * N;
  if (threadIdx.x < N) {
    double s = 0.0;
    for (int w = 0; w < kTWarps; ++w) s += red[w * N + threadIdx.x];
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

// ============================================================================ TF
template <int K>
__global__ void __launch_bounds__(kTThreads) tf_kernel(const TableArgs P) {
  cg::cluster_group cluster = cg::this_cluster();
  const int cl = P.cl, crank = (int)cluster.block_rank(), t = blockIdx.x / cl, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  __shared__ double sC[K], sCn[K], sCf[K], sDelta[K];
  __shared__ double red[kTWarps * 2 * K], part[2 * 2 * K], tot[2 * K];
  __shared__ int s_scan[kTWarps];
  __shared__ long long s_pg[kTWarps], s_nf[kTWarps];

  const int32_t* cnt = P.counts + (int64_t)t * kPatterns;
  const int chunk = kPatterns / cl, base = crank * chunk;
  uint16_t* rows = P.rows + (int64_t)t * kPatterns + base;
  TensorState* st = P.state + t;

  // ---- 1. compact populated finite patterns of this partition (ascending u); page masses
  int nr = 0;
  long long nonfin = 0;
  for (int off = 0; off < chunk; off += kTThreads) {
    const uint32_t u = (uint32_t)(base + off + tid);
    const int c = cnt[u];
    const bool fin = pattern_finite(u, P.wdtype);
    const bool pop = fin && c > 0;
    if (!fin) nonfin += c;
    const unsigned b = __ballot_sync(0xffffffffu, pop);
    long long pm = c;  // all present patterns (finite or not) pick the per-weight windows
#pragma unroll
    for (int o = 16; o; o >>= 1) pm += __shfl_xor_sync(0xffffffffu, pm, o);
    if (lane == 0) { s_scan[warp] = __popc(b); s_pg[warp] = pm; }
    __syncthreads();
    int woff = 0, btot = 0;
    for (int w = 0; w < kTWarps; ++w) {
      const int x = s_scan[w];
      woff += (w < warp) ? x : 0;
      btot += x;
    }
    if (pop) rows[nr + woff + __popc(b & ((1u << lane) - 1u))] = (uint16_t)u;
    if (tid < kTThreads / 256) {  // one signed page = 256 patterns = 8 warps
      long long s = 0;
      for (int w = 0; w < 8; ++w) s += s_pg[tid * 8 + w];
      P.page_cnt[(int64_t)t * 256 + ((base + off) >> 8) + tid] = s;
    }
    nr += btot;
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) nonfin += __shfl_xor_sync(0xffffffffu, nonfin, o);
  if (lane == 0) s_nf[warp] = nonfin;
  __syncthreads();
  if (tid == 0) {
    long long s = 0;
    for (int w = 0; w < kTWarps; ++w) s += s_nf[w];
    st->nonfinite[crank] = s;
    st->nrows[crank] = nr;
    if (crank == 0) st->cl = cl;
  }

  // ---- 2. unrolled centroid updates
  const int stride_c = (P.max_iter + 1) * K, stride_s = (P.max_iter > 0 ? P.max_iter : 1) * K;
  double* ctraj = P.ctraj + (int64_t)t * stride_c;
  double* straj = P.straj + (int64_t)t * stride_s;
  if (tid < K) {
    sC[tid] = (double)P.C0[(int64_t)t * K + tid];
    if (crank == 0) ctraj[tid] = sC[tid];
  }
  __syncthreads();
  int T = P.max_iter;
  for (int it = 0; it < P.max_iter; ++it) {
    double acc[2 * K];
#pragma unroll
    for (int j = 0; j < 2 * K; ++j) acc[j] = 0.0;
    for (int r = tid; r < nr; r += kTThreads) {
      const uint32_t u = rows[r];
      const double v = decode16(u, P.wdtype), n = (double)cnt[u];
      double A[K];
      attention_row<K>(v, sC, P.inv_tau, A);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const double na = n * A[j];
        acc[j] += na;
        acc[K + j] += na * v;
      }
    }
    cluster_allreduce<2 * K>(acc, red, part, tot, it & 1, cluster);
    if (tid < K) {
      const double S = tot[tid], M = tot[K + tid];
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
    if (tid < K) sC[tid] = sCn[tid];
    __syncthreads();
    if (P.eps > 0.0 && dmax <= P.eps) {  // identical on every CTA of the cluster
      T = it + 1;
      break;
    }
  }
  if (crank == 0 && tid == 0) st->T = T;
  if (tid < K) {
    const float cf = (float)sC[tid];
    if (crank == 0) P.C_out[(int64_t)t * K + tid] = cf;
    sCf[tid] = (double)cf;  // the deployable fp32 lookup table (R9)
  }
  __syncthreads();

  // ---- 3. W~ table (populated patterns), 16-bit rounding, hard index (all finite patterns)
  float* tab = P.table + (int64_t)t * kPatterns;
  uint16_t* tab16 = P.table16 + (int64_t)t * kPatterns;
  uint8_t* idx = P.idx8 + (int64_t)t * kPatterns;
  for (int u = base + tid; u < base + chunk; u += kTThreads) {
    const bool fin = pattern_finite(u, P.wdtype);
    const double v = decode16(u, P.wdtype);
    int best = 0;
    if (fin) {
      double bd = (v - sCf[0]) * (v - sCf[0]);
#pragma unroll
      for (int j = 1; j < K; ++j) {
        const double d = (v - sCf[j]) * (v - sCf[j]);
        if (d < bd) { bd = d; best = j; }
      }
    }
    idx[u] = (uint8_t)best;
    if (fin && cnt[u] > 0) {
      double A[K];
      attention_row<K>(v, sC, P.inv_tau, A);
      double wt = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) wt += A[j] * sC[j];
      tab[u] = (float)wt;
      tab16[u] = round16(wt, P.wdtype);
    } else {
      tab[u] = __int_as_float(0x7FC00000);
      tab16[u] = nan16(P.wdtype);
    }
  }
  cluster.sync();  // keep this CTA's shared memory alive until the cluster is done with it
}

// ============================================================================ TGAMMA
template <int K>
__global__ void __launch_bounds__(kTThreads) tgamma_kernel(const TableArgs P) {
  cg::cluster_group cluster = cg::this_cluster();
  const int cl = P.cl, crank = (int)cluster.block_rank(), t = blockIdx.x / cl, tid = threadIdx.x;
  __shared__ double sC[K], red[kTWarps * K], part[2 * K], tot[K];
  const TensorState* st = P.state + t;
  const int T = st->T, pcl = st->cl;
  if (tid < K) sC[tid] = P.ctraj[(int64_t)t * (P.max_iter + 1) * K + (int64_t)T * K + tid];
  __syncthreads();
  const double* Bt = P.B + (int64_t)t * kPatterns;
  double acc[K];
#pragma unroll
  for (int l = 0; l < K; ++l) acc[l] = 0.0;
  for (int p = crank; p < pcl; p += cl) {
    const uint16_t* rows = P.rows + (int64_t)t * kPatterns + p * (kPatterns / pcl);
    const int nr = st->nrows[p];
    for (int r = tid; r < nr; r += kTThreads) {
      const uint32_t u = rows[r];
      const double B = Bt[u];
      if (B == 0.0) continue;
      const double v = decode16(u, P.wdtype);
      double A[K];
      attention_row<K>(v, sC, P.inv_tau, A);
      double wt = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) wt += A[l] * sC[l];
#pragma unroll
      for (int l = 0; l < K; ++l) acc[l] += B * A[l] * (1.0 + (sC[l] - wt) * 2.0 * (v - sC[l]) * P.inv_tau);
    }
  }
  cluster_allreduce<K>(acc, red, part, tot, 0, cluster);
  if (crank == 0 && tid < K) P.gamma[(int64_t)t * K + tid] = tot[tid];
  cluster.sync();
}

// ============================================================================ TB
template <int K>
__global__ void __launch_bounds__(kTThreads) tb_kernel(const TableArgs P) {
  cg::cluster_group cluster = cg::this_cluster();
  const int cl = P.cl, crank = (int)cluster.block_rank(), t = blockIdx.x / cl, tid = threadIdx.x;
  __shared__ double sG[K], sCt[K], sCn[K], sInvS[K], red[kTWarps * K], part[2 * K], tot[K];
  const TensorState* st = P.state + t;
  const int T = st->T, pcl = st->cl;
  const int32_t* cnt = P.counts + (int64_t)t * kPatterns;
  const double* ctraj = P.ctraj + (int64_t)t * (P.max_iter + 1) * K;
  const double* straj = P.straj + (int64_t)t * (P.max_iter > 0 ? P.max_iter : 1) * K;
  double* psi = P.psi + (int64_t)t * kPatterns;
  if (tid < K) sG[tid] = P.gamma[(int64_t)t * K + tid];
  __syncthreads();
  for (int it = T - 1; it >= 0; --it) {
    if (tid < K) {
      sCt[tid] = ctraj[(int64_t)it * K + tid];
      sCn[tid] = ctraj[(int64_t)(it + 1) * K + tid];
      const double S = straj[(int64_t)it * K + tid];
      sInvS[tid] = S != 0.0 ? 1.0 / S : 0.0;
    }
    __syncthreads();
    double acc[K];
#pragma unroll
    for (int l = 0; l < K; ++l) acc[l] = 0.0;
    for (int p = crank; p < pcl; p += cl) {
      const uint16_t* rows = P.rows + (int64_t)t * kPatterns + p * (kPatterns / pcl);
      double* psi_p = psi + p * (kPatterns / pcl);
      const int nr = st->nrows[p];
      for (int r = tid; r < nr; r += kTThreads) {
        const uint32_t u = rows[r];
        const double v = decode16(u, P.wdtype), n = (double)cnt[u];
        double A[K], gh[K];
        attention_row<K>(v, sCt, P.inv_tau, A);
        double s = 0.0, dpsi = 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          gh[j] = sG[j] * (v - sCn[j]) * sInvS[j];  // dL/dA_t[u][j] (zero where S_t[j] = 0)
          s += A[j] * gh[j];
          dpsi += sG[j] * A[j] * sInvS[j];           // direct path of v through M_t
        }
#pragma unroll
        for (int l = 0; l < K; ++l) {
          const double rr = A[l] * (gh[l] - s);      // softmax Jacobian applied to gh
          const double dz = 2.0 * (v - sCt[l]) * P.inv_tau;
          dpsi -= rr * dz;
          acc[l] += n * rr * dz;
        }
        psi_p[r] = (it == T - 1 ? 0.0 : psi_p[r]) + dpsi;
      }
    }
    cluster_allreduce<K>(acc, red, part, tot, it & 1, cluster);
    if (tid < K) sG[tid] = tot[tid] + (sInvS[tid] == 0.0 ? sG[tid] : 0.0);  // C_{t+1} = C_t where S_t = 0
    __syncthreads();
  }
  if (crank == 0 && tid < K) P.dC0[(int64_t)t * K + tid] = (float)sG[tid];
  // (phi, psi) table: phi[u] = (2/tau) sum_l A_T[u,l] (C_T[l] - W~_u)^2
  if (tid < K) sCt[tid] = ctraj[(int64_t)T * K + tid];
  __syncthreads();
  float2* pp = P.phipsi + (int64_t)t * kPatterns;
  for (int p = crank; p < pcl; p += cl) {
    const uint16_t* rows = P.rows + (int64_t)t * kPatterns + p * (kPatterns / pcl);
    const double* psi_p = psi + p * (kPatterns / pcl);
    const int nr = st->nrows[p];
    for (int r = tid; r < nr; r += kTThreads) {
      const uint32_t u = rows[r];
      const double v = decode16(u, P.wdtype);
      double A[K];
      attention_row<K>(v, sCt, P.inv_tau, A);
      double wt = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) wt += A[l] * sCt[l];
      double var = 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) var += A[l] * (sCt[l] - wt) * (sCt[l] - wt);
      pp[u] = make_float2((float)(2.0 * P.inv_tau * var), T > 0 ? (float)psi_p[r] : 0.0f);
    }
    // NaN/Inf patterns: dW = NaN (R10)
    const int chunk = kPatterns / pcl;
    for (int u = p * chunk + tid; u < (p + 1) * chunk; u += kTThreads)
      if (!pattern_finite(u, P.wdtype)) pp[u] = make_float2(__int_as_float(0x7FC00000), __int_as_float(0x7FC00000));
  }
  cluster.sync();
}

// ============================================================================ launchers
int table_cluster_size(int nt) {
  if (nt <= 18) return 8;
  if (nt <= 37) return 4;
  if (nt <= 74) return 2;
  return 1;
}

#define EDKM_TABLE_LAUNCH(NAME, KERNEL)                                                          \
  cudaError_t NAME(const TableArgs& P, cudaStream_t s) {                                           \
    if (P.nt == 0) return cudaSuccess;                                                             \
    void (*fn)(const TableArgs);                                                                   \
    switch (P.k) {                                                                                 \
      case 2: fn = KERNEL<2>; break;                                                               \
      case 4: fn = KERNEL<4>; break;                                                               \
      case 8: fn = KERNEL<8>; break;                                                               \
      case 16: fn = KERNEL<16>; break;                                                             \
      default: return cudaErrorInvalidValue;                                                       \
    }                                                                                              \
    cudaLaunchConfig_t cfg = {};                                                                   \
    cfg.gridDim = dim3((unsigned)(P.nt * P.cl));                                                   \
    cfg.blockDim = dim3(kTThreads);                                                                \
    cfg.stream = s;                                                                                \
    cudaLaunchAttribute attr[1];                                                                   \
    attr[0].id = cudaLaunchAttributeClusterDimension;                                              \
    attr[0].val.clusterDim.x = (unsigned)P.cl;                                                     \
    attr[0].val.clusterDim.y = 1;                                                                  \
    attr[0].val.clusterDim.z = 1;                                                                  \
    cfg.attrs = attr;                                                                              \
    cfg.numAttrs = 1;                                                                              \
    return cudaLaunchKernelEx(&cfg, fn, P);                                                        \
  }

EDKM_TABLE_LAUNCH(launch_tf, tf_kernel)
EDKM_TABLE_LAUNCH(launch_tgamma, tgamma_kernel)
EDKM_TABLE_LAUNCH(launch_tb, tb_kernel)

}  // namespace edkm
