// fp64 peak microbenchmark for the roofline denominators of the fp64
// kernels (Cauchy contraction, pass-2 Z accumulation, eigen engine):
//   DFMA   : independent fma.rn.f64 chains, FMA = 2 flop
//   DMMA   : mma.sync.aligned.m8n8k4.row.col.f64 (256 FMA = 512 flop / warp-instr)
//   RCP    : the Newton reciprocal the kernels use (rcp.approx.ftz.f64 + 2 steps)
//   DIV    : IEEE a / b (div.rn.f64)
// Each kernel runs a one-wave persistent grid (all SMs x resident CTAs) for
// a fixed number of iterations; best of 5 launches, CUDA events.  Prints one
// JSON line.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

constexpr int CH = 8;   // independent chains per thread

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double acc[CH][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ double frcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  double e = fma(-q, r, 1.0);
  r = fma(r, e, r);
  e = fma(-q, r, 1.0);
  return fma(r, e, r);
}

__global__ void k_rcp(double* out, int iters) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = 1.5 + threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = frcp(x[c]) + 1.25;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_div(double* out, int iters) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = 1.5 + threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = 1.0 / x[c] + 1.25;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

template <class F>
float best_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 64));
  const int T = 256, B = sms * 8;   // 64 warps per SM
  const int it = 20000;
  const double threads = (double)T * B;
  float ms_fma = best_ms([&] { k_dfma<<<B, T>>>(out, it, 0.999999, 1e-7); });
  float ms_mma = best_ms([&] { k_dmma<<<B, T>>>(out, it / 4); });
  float ms_rcp = best_ms([&] { k_rcp<<<B, T>>>(out, it / 8); });
  float ms_div = best_ms([&] { k_div<<<B, T>>>(out, it / 8); });
  CK(cudaGetLastError());
  const double fma_tf = threads * it * CH * 2.0 / (ms_fma * 1e-3) / 1e12;
  const double mma_tf = (threads / 32.0) * (it / 4) * CH * 512.0 / (ms_mma * 1e-3) / 1e12;
  const double rcp_g = threads * (it / 8) * CH / (ms_rcp * 1e-3) / 1e9;
  const double div_g = threads * (it / 8) * CH / (ms_div * 1e-3) / 1e9;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_mhz_attr\": %.0f, "
         "\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"rcp_newton_gops\": %.1f, "
         "\"div_rn_gops\": %.1f, \"method\": \"one-wave grid %d x %d threads, %d independent chains "
         "per thread, best of 5 launches, CUDA events\"}\n",
         p.name, sms, clk / 1e3, fma_tf, mma_tf, rcp_g, div_g, B, T, CH);
  return 0;
}
