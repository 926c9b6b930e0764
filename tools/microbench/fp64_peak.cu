// FP64 pipe microbenchmark for sm_100a: DMMA (mma.sync m8n8k4 f64) and DFMA issue rates.
// Establishes the measured FP64 denominator that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CHAINS][2];
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CHAINS];
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) c[j] = j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) c[j] = fma(a, c[j], b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) s += c[j];
  if (s == 12345.0) out[0] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d smem/block optin %zu regs/SM %d clock(kHz) %d\n", p.name, p.multiProcessorCount,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, p.clockRate);
  double* out; cudaMalloc(&out, 8);
  int sms = p.multiProcessorCount;
  const int iters = 20000;
  for (int warps : {1, 2, 4, 8, 16, 32}) {
    int threads = 32 * warps;
    float ms = time_it([&] { dmma_loop<8><<<sms, threads>>>(out, iters); });
    double flops = (double)sms * warps * iters * 8 * 512.0;
    printf("DMMA m8n8k4 chains=8 warps/SM=%2d : %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  {
    float ms = time_it([&] { dmma_loop<1><<<sms, 32>>>(out, iters); });
    double cyc = (double)ms * 1e-3 * p.clockRate * 1e3 / iters;
    printf("DMMA dependent-chain latency ~ %.1f cycles (at nominal clock)\n", cyc);
  }
  for (int warps : {4, 8, 16, 32}) {
    int threads = 32 * warps;
    float ms = time_it([&] { dfma_loop<8><<<sms, threads>>>(out, iters); });
    double flops = (double)sms * threads * iters * 8 * 2.0;
    printf("DFMA chains=8 warps/SM=%2d : %.2f TFLOP/s\n", warps, flops / ms / 1e9);
  }
  return 0;
}
