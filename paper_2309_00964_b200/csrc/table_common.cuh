// table_common.cuh -- row-balanced partitions of the table phase (S4 "Table phase").
//
// The cl CTAs of a tensor's cluster split its populated finite patterns ("rows") into cl
// pattern ranges [pb[r], pb[r+1]) holding ~U/cl rows each (16-pattern granularity), so the work
// per CTA is balanced whatever the value distribution (a split of the pattern space into equal
// ranges leaves most CTAs empty: N(0, 0.02^2) weights occupy a few percent of it).  Rows of
// partition r are stored at rows[pb[r] ...] (a range holds at most as many rows as patterns).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "launch.h"


namespace edkm {

// Every CTA of the cluster calls it (all threads); on return s_pb[0..cl] holds identical bounds
// in every CTA.  Also writes page_cnt[256] (weights per signed page, every present pattern).
// s_pg: shared int[256]; s_pref: shared int[257]; s_pb: shared int[kMaxCluster + 1].
template <int NT>
__device__ void table_partitions(const int32_t* cnt, int wdtype, int64_t* page_cnt, int cl, int crank,
                                 cooperative_groups::cluster_group& cluster, int* s_pg, int* s_pref, int* s_pb) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 1. rows and weights of the pages this CTA owns (page pg owned by CTA pg % cl), a warp per page
  for (int pg = crank + cl * warp; pg < 256; pg += cl * NW) {
    const int u0 = pg * 256 + lane * 8;
    const int4 a = __ldg(reinterpret_cast<const int4*>(cnt + u0));
    const int4 b = __ldg(reinterpret_cast<const int4*>(cnt + u0 + 4));
    const int c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    int rws = 0;
    long long w = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      rws += (pattern_finite(u0 + e, wdtype) && c[e] > 0) ? 1 : 0;
      w += c[e];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      rws += __shfl_xor_sync(0xffffffffu, rws, o);
      w += __shfl_xor_sync(0xffffffffu, w, o);
    }
    if (lane == 0) {
      s_pg[pg] = rws;
      page_cnt[pg] = w;
    }
  }
  cluster.sync();
  // 2. every page's row count from its owner (DSMEM), exclusive prefix s_pref[0..256]
  for (int pg = tid; pg < 256; pg += NT) {
    const int owner = pg % cl;
    s_pref[pg + 1] = owner == crank ? s_pg[pg] : cluster.map_shared_rank(s_pg, owner)[pg];
  }
  __syncthreads();
  if (warp == 0) {
    int v[8], sum = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[e] = s_pref[1 + lane * 8 + e];
      sum += v[e];
    }
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    int run = inc - sum;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      run += v[e];
      s_pref[1 + lane * 8 + e] = run;
    }
    if (lane == 0) s_pref[0] = 0;
  }
  __syncthreads();
  // 3. bound r = the smallest 16-aligned pattern b with rows_before(b) >= ceil(r U / cl); a warp per bound
  const int U = s_pref[256];
  for (int r = 1 + warp; r < cl; r += NW) {
    const int target = (int)(((long long)r * U + cl - 1) / cl);
    int bnd = 0;
    if (target > 0) {
      int lo = 0, hi = 255;  // smallest page P with s_pref[P + 1] >= target
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_pref[mid + 1] >= target) hi = mid; else lo = mid + 1;
      }
      const int P = lo;
      const int u0 = P * 256 + lane * 8;
      const int4 a = __ldg(reinterpret_cast<const int4*>(cnt + u0));
      const int4 b = __ldg(reinterpret_cast<const int4*>(cnt + u0 + 4));
      const int c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      int rws = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) rws += (pattern_finite(u0 + e, wdtype) && c[e] > 0) ? 1 : 0;
      int inc = rws;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      // odd lane l ends 16-pattern group (l+1)/2: the first one reaching the target
      const unsigned ok = __ballot_sync(0xffffffffu, (lane & 1) && s_pref[P] + inc >= target);
      const int l = __ffs(ok) - 1;  // exists: s_pref[P + 1] >= target
      bnd = P * 256 + 16 * ((l + 1) >> 1);
    }
    if (lane == 0) s_pb[r] = bnd;
  }
  if (tid == 0) {
    s_pb[0] = 0;
    s_pb[cl] = kPatterns;
  }
  __syncthreads();
}

// End of TF: once every CTA of the cluster has written its page masses (call after a cluster
// barrier), CTA 0's first warp chooses the magnitude-page windows of the per-weight kernels for
// this tensor and stores them in its TensorState (B1/B2, and F2 with fp32 output), so no
// per-weight kernel searches for them per segment.
__device__ __forceinline__ void table_windows(const int64_t* page_cnt, TensorState* st, int crank) {
  const int warp = threadIdx.x >> 5;
  if (crank != 0 || warp > 1) return;
  int pb, np;  // warp 0: the B1/B2 window, warp 1: the F2 fp32 window (in parallel)
  choose_window(page_cnt, warp == 0 ? kWinPagesB : kWinPagesF2, pb, np);
  if ((threadIdx.x & 31) == 0) {
    st->win[2 * warp] = (uint8_t)pb;
    st->win[2 * warp + 1] = (uint8_t)np;
  }
}

}  // namespace edkm
