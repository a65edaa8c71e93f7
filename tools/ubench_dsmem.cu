// Microbenchmark: lane-private shared-memory counters updated locally vs through distributed shared
// memory (red.shared::cluster.add.u32 to a random CTA of the cluster).  The question for a fp16 F1
// (DESIGN S9): can a 4-CTA cluster hold 4x the lane-private window, each element's counter living
// on the CTA that owns its page, at close to the local atomic rate?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_dsmem tools/ubench_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

constexpr int kRows = 1792;  // 7 pages x 256 rows, 32 lanes: 224 KiB
__global__ void __launch_bounds__(1024, 1) k_dsmem(int iters, int remote_pct, unsigned* out) {
  extern __shared__ uint32_t h[];
  cg::cluster_group cl = cg::this_cluster();
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kRows * 32; i += blockDim.x) h[i] = 0;
  cl.sync();
  const unsigned ncl = cl.num_blocks(), me = cl.block_rank();
  uint32_t x = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u + 12345u;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(h) + lane * 4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      x = x * 1664525u + 1013904223u;
      const uint32_t row = (x >> 8) % kRows;
      const uint32_t a = base + row * 128;
      unsigned tgt = me;
      if (ncl > 1 && ((x >> 24) % 100) < (unsigned)remote_pct) tgt = (me + 1 + (x & 7) % (ncl - 1)) % ncl;
      if (tgt == me) {
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a) : "memory");
      } else {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(tgt));
        asm volatile("red.shared::cluster.add.u32 [%0], 1;" ::"r"(ra) : "memory");
      }
    }
  }
  cl.sync();
  if (threadIdx.x == 0) atomicAdd(out, h[0]);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  cudaMalloc(&out, 4);
  const size_t smem = kRows * 32 * 4;
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int iters = 2000;
  for (int csize : {1, 2, 4}) {
    for (int pct : {0, 50, 75}) {
      if (csize == 1 && pct) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms / csize * csize);
      cfg.blockDim = dim3(1024);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = csize;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaLaunchKernelEx(&cfg, k_dsmem, 10, pct, out);
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, k_dsmem, iters, pct, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double elems = (double)cfg.gridDim.x * 1024 * iters * 16;
      printf("cluster %d remote %2d%%: %.3f ms  %.1f G elem/s  (%.2f elem/clk/SM at 1.965 GHz) %s\n", csize, pct, ms,
             elems / ms / 1e6, elems / (ms * 1e-3) / cfg.gridDim.x / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
