// INT8 tensor-pipe peak on this B200: one CTA per SM issues back-to-back tcgen05.mma.cta_group::1.kind::i8
// 128 x 256 x 32 instructions on operands resident in shared memory (no TMA, no epilogue), accumulating
// in TMEM; MACs / event time.  Operands: random bytes (the power-relevant case) or zeros.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/microbench/i8_peak.cu -o tools/microbench/i8_peak
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void __launch_bounds__(128, 1) peak_kernel(int iters, int zero, unsigned long long* sink, int commit_every) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  uint8_t* A = base;              // 128 x 128 B
  uint8_t* B = base + 16384;      // 256 x 128 B
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) {
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    reinterpret_cast<uint32_t*>(A)[i] = zero ? 0u : x;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
  if (commit_every == -2) {   // the same with one lane doing the wait, fence, issue and commit
    if (threadIdx.x == 0) {
      const uint64_t da = desc(su32(A)), db = desc(su32(B));
      for (int it = 0; it < iters; ++it) {
        asm volatile("{\n.reg .pred p;\nW3:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1;\n@!p bra W3;\n}\n" ::"r"(su32(&bar2)));
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t acc = (it | k) != 0;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
  } else if (commit_every < 0) {   // the GEMM's MMA-warp loop with the data always ready: the whole warp waits on a
                            // completed barrier, fences, one lane issues the stage's 4 MMAs and a commit
    if (threadIdx.x < 32) {
      const uint64_t da = desc(su32(A)), db = desc(su32(B));
      for (int it = 0; it < iters; ++it) {
        asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1;\n@!p bra W2;\n}\n" ::"r"(su32(&bar2)));
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (threadIdx.x == 0) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t acc = (it | k) != 0;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem), "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)));
        }
        __syncwarp();
      }
      if (threadIdx.x == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
  } else if (threadIdx.x == 0) {
    const uint64_t da = desc(su32(A)), db = desc(su32(B));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t acc = (it | k) != 0;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
      }
      if (commit_every && (it % commit_every) == 0)   // the GEMM's per-stage commit (to a barrier nobody waits on)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  __syncwarp();
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((threadIdx.x & 96) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  if (v == 0x12345678u) atomicAdd(sink, 1ull);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int smem = 49152 + 1024;
  cudaFuncSetAttribute(peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int ce = 0; ce < 5; ++ce)
  for (int zero = 0; zero < 2; ++zero) {
    for (int rep = 0; rep < 2; ++rep) {
      const int iters = 150000;
      const int commit_every = ce == 0 ? 0 : (ce == 1 ? 1 : (ce == 2 ? 2 : (ce == 3 ? -1 : -2)));
      if (rep == 0) printf("commit every %d stage(s) of 4 MMAs (0: none):\n", commit_every);
      cudaEventRecord(e0);
      peak_kernel<<<sms, 128, smem>>>(iters, zero, sink, commit_every);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double macs = (double)sms * iters * 4 * 128.0 * 256.0 * 32.0;
      printf("int8 tcgen05.mma 128x256x32, %s operands, %d SMs: %.2f ms  %.1f TOPS (%.0f MAC/clk/SM at the %d MHz max)\n",
             zero ? "zero" : "random", sms, ms, 2 * macs / ms / 1e9, macs / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
