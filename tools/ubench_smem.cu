// Microbenchmarks that size the per-weight passes before they are written:
// HBM streaming read, shared-memory atomics on 16-bit bit patterns (F1/B1
// shape) and shared-memory table gathers (F2/B2 shape), on bf16 N(0, 0.02^2)
// patterns. Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench_smem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void gen_bf16(uint16_t* w, size_t n, float sigma, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t a = hash32((uint32_t)i * 2u + seed), b = hash32((uint32_t)i * 2u + 1u + seed * 7u);
    float u1 = (a + 1.0f) * 2.3283064e-10f, u2 = b * 2.3283064e-10f;
    float z = sqrtf(-2.f * logf(u1)) * cospif(2.f * u2) * sigma;
    __nv_bfloat16 h = __float2bfloat16_rn(z);
    w[i] = *reinterpret_cast<uint16_t*>(&h);
  }
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ void ldg_stream8(const uint4* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(p));
}
__global__ void k_read8(const uint4* w, size_t n32, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n32; i += stride) {
    uint4 a, b; ldg_stream8(w + 2 * i, a, b);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
// copy with 256-bit loads/stores, U vectors in flight per thread
template <int U>
__global__ void k_copy8(const uint4* w, size_t n32, uint4* out) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n32; i += U * stride) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ldg_stream8(w + 2 * (i + u * stride), a[u], b[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(out + 2 * (i + u * stride)),
                   "r"(a[u].x), "r"(a[u].y), "r"(a[u].z), "r"(a[u].w), "r"(b[u].x), "r"(b[u].y), "r"(b[u].z), "r"(b[u].w) : "memory");
  }
}
__global__ void k_read(const uint4* w, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + stride < n16; i += 2 * stride) {
    uint4 a = ldg_stream(w + i), b = ldg_stream(w + i + stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
  }
  for (; i < n16; i += stride) { uint4 a = ldg_stream(w + i); acc ^= a.x ^ a.y ^ a.z ^ a.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

// MODE 0: packed u16 counters with return (overflow check); 1: packed, no return (red);
// 2: u32 counters over u & 0x7FFF (no packing); 3: f32 add into 16K buckets (u & 0x3FFF)
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_hist(const uint4* w, size_t n16, uint32_t* gout) {
  extern __shared__ uint32_t h[];
  const int nw = (MODE == 3) ? 16384 : ((MODE >= 10 || MODE == 5) ? 57344 : 32768);
  for (int i = threadIdx.x; i < nw; i += blockDim.x) h[i] = 0;
  __syncthreads();
  size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t spill = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
    uint4 v = ldg_stream(w + i);
    uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t u = (wd[q] >> (16 * hh)) & 0xFFFFu;
        if (MODE == 0) {
          uint32_t sh = (u & 1u) * 16u;
          uint32_t old = atomicAdd(&h[u >> 1], 1u << sh);
          if (((old >> sh) & 0xFFFFu) == 0x7FFFu) { atomicSub(&h[u >> 1], 0x8000u << sh); spill += 0x8000u; }
        } else if (MODE == 1) {
          uint32_t sh = (u & 1u) * 16u;
          asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&h[u >> 1])), "r"(1u << sh));
        } else if (MODE == 4) {
          uint32_t a = (uint32_t)__cvta_generic_to_shared(&h[u >> 1]);
          if (u & 1u) asm volatile("red.shared.add.u32 [%0], 65536;" :: "r"(a));
          else asm volatile("red.shared.add.u32 [%0], 1;" :: "r"(a));
        } else if (MODE == 5) {  // u32 atom with return, result consumed cheaply
          uint32_t old;
          asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"((uint32_t)__cvta_generic_to_shared(&h[u % 57344u])));
          spill ^= old;
        } else if (MODE >= 10) {  // C = MODE-10 copies interleaved: word = idx*C + lane%C, idx in [0, 224K/4/C)
          constexpr int C = MODE - 10;
          const uint32_t idx = u % (57344u / C);
          asm volatile("red.shared.add.u32 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&h[idx * C + (threadIdx.x & (C - 1))])));
        } else if (MODE == 2) {
          asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&h[u & 0x7FFFu])), "r"(1u));
        } else {
          float g = __uint_as_float(u << 16);
          atomicAdd(reinterpret_cast<float*>(&h[u & 0x3FFFu]), g);
        }
      }
    }
  }
  __syncthreads();
  uint32_t s = spill;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) s += h[i];
  if (s == 0x12345678u) gout[0] = s;
}

// L2 atomics: fraction 1/F of elements (u % F == 0) go to red.global on a 256 KB counter array, rest to SMEM
template <int F>
__global__ void __launch_bounds__(1024, 1) k_hist_l2(const uint4* w, size_t n16, uint32_t* gcnt, uint32_t* gout) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < 57344; i += blockDim.x) h[i] = 0;
  __syncthreads();
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
    uint4 v = ldg_stream(w + i);
    uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t u = (wd[q] >> (16 * hh)) & 0xFFFFu;
        if (F == 1 || (u % F) == 0) asm volatile("red.global.add.u32 [%0], 1;" :: "l"(gcnt + u));
        else asm volatile("red.shared.add.u32 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&h[u % 57344u])));
      }
    }
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < 57344; i += blockDim.x) s += h[i];
  if (s == 0x12345678u) gout[0] = s;
}

// lane-private replicas: 32 copies of packed u16 counters for NP magnitude pages x 2 signs, copy l
// entirely in bank l (word = (slot >> 1) * 32 + lane), so a warp's 32 atomics never share a bank.
// Patterns outside the window go to a shared u32 array (conflicting banks; ~0.5% of N(0,0.02^2)).
// Timing only: the u16 counters are not flushed (the real kernel flushes every 2M elements).
template <int NP, int V8>
__global__ void __launch_bounds__(1024, 1) k_hist_lane(const uint4* w, size_t n16, uint32_t* gout, int pbase) {
  extern __shared__ uint32_t h[];
  constexpr int kWords = NP * 256 * 32;  // 2*NP*256 slots / 2 per word * 32 copies
  constexpr int kLow = (232448 / 4 - kWords) & ~255;
  uint32_t* lowc = h + kWords;
  for (int i = threadIdx.x; i < kWords + kLow; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(h) + lane * 4u;
  const uint32_t pb = (uint32_t)pbase * 256u, np256 = NP * 256u;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16 / (V8 ? 2 : 1); i += stride) {
    uint32_t wd[8];
    if (V8) {
      uint4 a, b; ldg_stream8(w + 2 * i, a, b);
      wd[0] = a.x; wd[1] = a.y; wd[2] = a.z; wd[3] = a.w; wd[4] = b.x; wd[5] = b.y; wd[6] = b.z; wd[7] = b.w;
    } else {
      uint4 v = ldg_stream(w + i);
      wd[0] = v.x; wd[1] = v.y; wd[2] = v.z; wd[3] = v.w;
    }
#pragma unroll
    for (int q = 0; q < (V8 ? 8 : 4); ++q) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t u = (wd[q] >> (16 * hh)) & 0xFFFFu;
        const uint32_t rel = (u & 0x7FFFu) - pb;
        if (rel < np256) {
          const uint32_t slot = (u >> 15) * np256 + rel;
          asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(base + (slot >> 1) * 128u), "r"(1u << ((slot & 1u) * 16u)));
        } else {
          asm volatile("red.shared.add.u32 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&lowc[u % (uint32_t)kLow])));
        }
      }
    }
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < kWords + kLow; i += blockDim.x) s += h[i];
  if (s == 0x12345678u) gout[0] = s;
}

// gather: out[i] = table[u_i] with a 128 KB bf16 table in SMEM
__global__ void __launch_bounds__(1024, 1) k_gather(const uint4* w, size_t n16, uint4* out, const uint16_t* gtable) {
  extern __shared__ uint16_t t[];
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) t[i] = gtable[i];
  __syncthreads();
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
    uint4 v = ldg_stream(w + i);
    uint32_t wd[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = (uint32_t)t[wd[q] & 0xFFFF] | ((uint32_t)t[wd[q] >> 16] << 16);
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(out + i), "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]));
  }
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("%s SMs=%d clock=%d MHz smem/blk optin=%zu\n", p.name, p.multiProcessorCount, clk_khz / 1000, p.sharedMemPerBlockOptin);
  const size_t n = (size_t)1 << 31;  // 2^31 bf16 = 4 GiB
  uint16_t *w; uint32_t* o; uint4* out; uint16_t* tab;
  CK(cudaMalloc(&w, n * 2)); CK(cudaMalloc(&o, 64)); CK(cudaMalloc(&out, n * 2)); CK(cudaMalloc(&tab, 65536 * 2));
  CK(cudaMemset(tab, 0, 65536 * 2));
  gen_bf16<<<4096, 256>>>(w, n, 0.02f, 1234u); CK(cudaDeviceSynchronize());
  int sms = p.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, double bytes) {
    for (int r = 0; r < 2; ++r) launch();
    cudaEventRecord(e0); const int R = 5; for (int r = 0; r < R; ++r) launch(); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= R;
    cudaError_t e = cudaGetLastError();
    printf("%-28s %8.3f ms  %8.1f GB/s  %7.1f Gw/s  %s\n", name, ms, bytes / ms / 1e6, n / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  size_t n16 = n / 8;
  run("read_stream 148x1024", [&] { k_read<<<sms, 1024>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("read_stream 148*4x512", [&] { k_read<<<sms * 4, 512>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("read_v8 148*4x512", [&] { k_read8<<<sms * 4, 512>>>((const uint4*)w, n16 / 2, o); }, n * 2.0);
  run("read_v8 148*8x256", [&] { k_read8<<<sms * 8, 256>>>((const uint4*)w, n16 / 2, o); }, n * 2.0);
  run("copy v8 148x1024 U2", [&] { k_copy8<2><<<sms, 1024>>>((const uint4*)w, n16 / 2, out); }, n * 4.0);
  run("copy v8 148x1024 U1", [&] { k_copy8<1><<<sms, 1024>>>((const uint4*)w, n16 / 2, out); }, n * 4.0);
  run("copy v8 148*2x1024 U2", [&] { k_copy8<2><<<sms * 2, 1024>>>((const uint4*)w, n16 / 2, out); }, n * 4.0);
  run("copy v8 148*4x512 U4", [&] { k_copy8<4><<<sms * 4, 512>>>((const uint4*)w, n16 / 2, out); }, n * 4.0);
  run("copy v8 148*8x256 U2", [&] { k_copy8<2><<<sms * 8, 256>>>((const uint4*)w, n16 / 2, out); }, n * 4.0);
  cudaFuncSetAttribute(k_hist<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k_hist<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k_hist<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k_hist<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k_hist<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  run("hist packed u16 atom+ret", [&] { k_hist<0><<<sms, 1024, 131072>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("hist packed u16 red", [&] { k_hist<1><<<sms, 1024, 131072>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("hist packed 2x const red", [&] { k_hist<4><<<sms, 1024, 131072>>>((const uint4*)w, n16, o); }, n * 2.0);
  for (int m : {11, 12, 14, 18}) {}
  cudaFuncSetAttribute(k_hist<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
  cudaFuncSetAttribute(k_hist<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
  cudaFuncSetAttribute(k_hist<14>, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
  cudaFuncSetAttribute(k_hist<18>, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
  run("hist 1 copy  (57344 bins)", [&] { k_hist<11><<<sms, 1024, 229376>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("hist 2 copies interleaved", [&] { k_hist<12><<<sms, 1024, 229376>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("hist 4 copies interleaved", [&] { k_hist<14><<<sms, 1024, 229376>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("hist 8 copies interleaved", [&] { k_hist<18><<<sms, 1024, 229376>>>((const uint4*)w, n16, o); }, n * 2.0);
  uint32_t* gcnt; CK(cudaMalloc(&gcnt, 65536 * 4 * 4));
  cudaFuncSetAttribute(k_hist_l2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
  cudaFuncSetAttribute(k_hist_l2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
  cudaFuncSetAttribute(k_hist_l2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
  cudaFuncSetAttribute(k_hist_l2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
  run("hist all L2 red", [&] { k_hist_l2<1><<<sms, 1024, 229376>>>((const uint4*)w, n16, gcnt, o); }, n * 2.0);
  run("hist 1/2 L2 red", [&] { k_hist_l2<2><<<sms, 1024, 229376>>>((const uint4*)w, n16, gcnt, o); }, n * 2.0);
  run("hist 1/4 L2 red", [&] { k_hist_l2<4><<<sms, 1024, 229376>>>((const uint4*)w, n16, gcnt, o); }, n * 2.0);
  run("hist 1/8 L2 red", [&] { k_hist_l2<8><<<sms, 1024, 229376>>>((const uint4*)w, n16, gcnt, o); }, n * 2.0);
  cudaFuncSetAttribute(k_hist<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
  run("hist u32 atom+ret (xor)", [&] { k_hist<5><<<sms, 1024, 229376>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("hist u32 32K red", [&] { k_hist<2><<<sms, 1024, 131072>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("bucket f32 16K atom", [&] { k_hist<3><<<sms, 1024, 65536>>>((const uint4*)w, n16, o); }, n * 2.0);
  run("bucket f32 16K atom 3x/SM", [&] { k_hist<3><<<sms * 3, 1024 / 2, 65536>>>((const uint4*)w, n16, o); }, n * 2.0);
  cudaFuncSetAttribute(k_hist_lane<6, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaFuncSetAttribute(k_hist_lane<6, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaFuncSetAttribute(k_hist_lane<7, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  run("hist lane-private 6pg v4", [&] { k_hist_lane<6, 0><<<sms, 1024, 232448>>>((const uint4*)w, n16, o, 57); }, n * 2.0);
  run("hist lane-private 6pg v8", [&] { k_hist_lane<6, 1><<<sms, 1024, 232448>>>((const uint4*)w, n16, o, 57); }, n * 2.0);
  run("hist lane-private 7pg v8", [&] { k_hist_lane<7, 1><<<sms, 1024, 232448>>>((const uint4*)w, n16, o, 56); }, n * 2.0);
  run("gather bf16 128K smem", [&] { k_gather<<<sms, 1024, 131072>>>((const uint4*)w, n16, out, tab); }, n * 4.0);
  return 0;
}
