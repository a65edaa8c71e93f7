// Microbenchmark: per-SM throughput of the table phase's arithmetic units on this B200 -- MUFU
// ex2.approx.ftz.f32 (one per attention entry), rcp.approx, FFMA (fp32) and DFMA (fp64) -- the
// measured peaks of bench.py's `table_roofline` (DESIGN S8).  Each thread runs 8 independent
// dependency chains; 148 x 4 CTAs of 512 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mufu tools/ubench_mufu.cu
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void __launch_bounds__(512) k_op(int iters, float* out) {
  float x[8];
  double d[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    x[c] = 1e-3f * (threadIdx.x + c);
    d[c] = 1e-3 * (threadIdx.x + c);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
      if (OP == 1) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
      if (OP == 2) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFE, 0f33800000;" : "+f"(x[c]));
      if (OP == 3) asm volatile("fma.rn.f64 %0, %0, 0d3FEFFFFFFFFFFFFE, 0d3CB0000000000000;" : "+d"(d[c]));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c] + (float)d[c];
  if (s == 1234.5f) out[0] = s;
}

template <int OP>
static double rate(int sms, int clk_khz, float* out) {
  const int iters = 20000, ctas = sms * 4, threads = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_op<OP><<<ctas, threads>>>(iters / 10, out);
  cudaEventRecord(e0);
  k_op<OP><<<ctas, threads>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)ctas * threads * iters * 8;
  const double per_clk_sm = ops / sms / (ms * 1e-3 * clk_khz * 1e3);
  printf("  %-26s %8.3f ms  %7.2f ops/clk/SM  %8.1f Gops/s\n",
         OP == 0 ? "ex2.approx.ftz.f32" : OP == 1 ? "rcp.approx.ftz.f32" : OP == 2 ? "fma.rn.f32" : "fma.rn.f64", ms,
         per_clk_sm, ops / (ms * 1e6));
  return ops / (ms * 1e-3);
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4);
  printf("B200 SMs=%d clock(attr)=%d MHz (per-clock figures at that clock)\n", sms, clk / 1000);
  const double ex2 = rate<0>(sms, clk, out);
  rate<1>(sms, clk, out);
  rate<2>(sms, clk, out);
  const double f64 = rate<3>(sms, clk, out);
  printf("{\"ex2_per_s\": %.4e, \"dfma_per_s\": %.4e}\n", ex2, f64);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
