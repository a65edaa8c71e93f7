// How many clusters of a table-kernel shape fit on the GPU at once (cudaOccupancyMaxActiveClusters)
// and how many CTAs that is, per cluster size: the table phase's wave quantisation (DESIGN S9).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_clusters tools/probe_clusters.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MB>
__global__ void __launch_bounds__(256, MB) k_shape(float* out) {
  extern __shared__ float sm[];
  __shared__ float st[3000];  // ~12 KB static, like CSet + BSet + reduction buffers
  st[threadIdx.x] = sm[threadIdx.x];
  __syncthreads();
  if (out) out[threadIdx.x] = st[255 - threadIdx.x];
}

template <int MB>
void probe(const char* name, size_t dyn) {
  cudaFuncSetAttribute((const void*)k_shape<MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  cudaFuncSetAttribute((const void*)k_shape<MB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl = 1; cl <= 8; ++cl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * 64);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = dyn;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (const void*)k_shape<MB>, &cfg);
    printf("%s dyn %zu KiB cl %d: %d clusters = %d CTAs %s\n", name, dyn / 1024, cl, n, n * cl,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  probe<2>("TB<16> 2/SM", 6400 * 16);
  probe<3>("TF<16> 3/SM", 6400 * 8);
  probe<4>("k<=8  4/SM", 6400 * 8);
  return 0;
}
