// Standalone check + timing of the INT8 tcgen05 GEMM (csrc/igemm.cu): exactness against a CPU
// int64 reference on ragged shapes (both epilogues, the upper / triangular flags), then the
// throughput of big square and K.U-shaped products.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2508_18468_b200/csrc \
//        tools/microbench/igemm_bench.cu -o /tmp/igemm_bench -lcuda
#include "../../paper_2508_18468_b200/csrc/igemm.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
namespace traj { std::atomic<long long> g_kernel_launches{0}; }
using namespace traj;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

static int check(long long M, long long N, long long K, int batch, int out, int flags, int ks = 1) {
  const long long lda = (K + 15) / 16 * 16, ldc = (N + 15) / 16 * 16;
  std::vector<int8_t> A(batch * M * lda), B(batch * N * lda);
  std::mt19937 rng(1234 + M + N + K);
  for (auto& x : A) x = (int8_t)(rng() & 255);
  for (auto& x : B) x = (int8_t)(rng() & 255);
  if (flags & IG_TRI_B)   // B[n][k] = 0 for k > n
    for (int z = 0; z < batch; ++z) for (long long n = 0; n < N; ++n) for (long long k = n + 1; k < K; ++k) B[(z * N + n) * lda + k] = 0;
  int mods[2] = {251, 256};
  int8_t *dA, *dB; void* dC; int* dm;
  const size_t esz = out == IG_OUT_I32 ? 4 : 1;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dC, ks * batch * M * ldc * esz)); CK(cudaMalloc(&dm, 8));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dm, mods, 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0x5a, ks * batch * M * ldc * esz));
  IgemmArgs g; g.M = M; g.N = N; g.K = K; g.batch = batch; g.A = dA; g.lda = lda; g.strideA = M * lda;
  g.B = dB; g.ldb = lda; g.strideB = N * lda; g.C = dC; g.ldc = ldc; g.strideC = M * ldc; g.out = out; g.moduli = dm; g.nmod = 2; g.flags = flags;
  g.ksplit = ks;
  std::string err;
  int s = igemm(0, g, &err);
  if (s) { printf("igemm failed %d %s\n", s, err.c_str()); return 1; }
  CK(cudaDeviceSynchronize());
  std::vector<uint8_t> Cs(ks * batch * M * ldc * esz), C(batch * M * ldc * esz);
  CK(cudaMemcpy(Cs.data(), dC, Cs.size(), cudaMemcpyDeviceToHost));
  for (int z = 0; z < batch; ++z)   // sum the split-K chunks (mod m for the modular epilogue)
    for (long long e = 0; e < M * ldc; ++e) {
      long long acc = 0;
      for (int c = 0; c < ks; ++c) {
        const long long off = ((long long)z * ks + c) * M * ldc + e;
        acc += out == IG_OUT_I32 ? (long long)reinterpret_cast<int*>(Cs.data())[off] : (long long)Cs[off];
      }
      if (out == IG_OUT_I32) reinterpret_cast<int*>(C.data())[z * M * ldc + e] = (int)acc;
      else C[z * M * ldc + e] = (uint8_t)(acc % mods[z % 2]);
    }
  long long bad = 0, checked = 0;
  for (int z = 0; z < batch; ++z) for (long long m = 0; m < M; ++m) for (long long n = 0; n < N; ++n) {
    if ((flags & IG_UPPER) && (n / 256 + 1) * 256 - 1 < (m / 128) * 128) continue;
    long long acc = 0;
    for (long long k = 0; k < K; ++k) acc += (long long)A[(z * M + m) * lda + k] * B[(z * N + n) * lda + k];
    long long got;
    if (out == IG_OUT_I32) got = reinterpret_cast<int*>(C.data())[(z * M + m) * ldc + n];
    else { got = C[(z * M + m) * ldc + n]; int md = mods[z % 2]; acc = ((acc % md) + md) % md; }
    ++checked;
    if (got != acc) { if (bad < 5) printf("  mismatch z=%d m=%lld n=%lld got %lld want %lld\n", z, m, n, got, acc); ++bad; }
  }
  printf("check M=%lld N=%lld K=%lld batch=%d out=%d flags=%d: %lld/%lld bad\n", M, N, K, batch, out, flags, bad, checked);
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dm);
  return bad != 0;
}

static void timeit(long long M, long long N, long long K, int batch, int out) {
  const long long lda = K, ldc = N;
  int8_t *dA, *dB; void* dC; int* dm;
  int mods[2] = {251, 256};
  CK(cudaMalloc(&dA, batch * M * lda)); CK(cudaMalloc(&dB, batch * N * lda));
  CK(cudaMalloc(&dC, batch * M * ldc * (out == IG_OUT_I32 ? 4 : 1))); CK(cudaMalloc(&dm, 8));
  CK(cudaMemcpy(dm, mods, 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(dA, 3, batch * M * lda)); CK(cudaMemset(dB, 5, batch * N * lda));
  IgemmArgs g; g.M = M; g.N = N; g.K = K; g.batch = batch; g.A = dA; g.lda = lda; g.strideA = M * lda;
  g.B = dB; g.ldb = lda; g.strideB = N * lda; g.C = dC; g.ldc = ldc; g.strideC = M * ldc; g.out = out; g.moduli = dm; g.nmod = 2;
  std::string err;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) igemm(0, g, &err);
  CK(cudaDeviceSynchronize());
  const int reps = 5;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) igemm(0, g, &err);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  const double ops = 2.0 * M * N * K * batch;
  printf("time M=%lld N=%lld K=%lld batch=%d out=%d: %.3f ms  %.1f TOPS\n", M, N, K, batch, out, ms, ops / ms / 1e9);
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dm);
}

static void timeit_rand(long long M, long long N, long long K, int batch) {
  int8_t *dA, *dB; void* dC; int* dm;
  int mods[2] = {251, 256};
  CK(cudaMalloc(&dA, batch * M * K)); CK(cudaMalloc(&dB, batch * N * K));
  const int ks = getenv("KSPLIT") ? atoi(getenv("KSPLIT")) : 1;
  CK(cudaMalloc(&dC, batch * M * N * ks)); CK(cudaMalloc(&dm, 8));
  CK(cudaMemcpy(dm, mods, 8, cudaMemcpyHostToDevice));
  {
    std::vector<int8_t> h(1 << 26);
    std::mt19937 rng(5);
    for (auto& x : h) x = (int8_t)(rng() & 255);
    const bool banded = getenv("BANDED_A") != nullptr;   // A like K's residues: nonzero only near the diagonal
    if (banded) {
      std::vector<int8_t> a1(M * K, 0);
      for (long long m = 0; m < M; ++m)
        for (long long k = std::max(0LL, m - 24); k < std::min(K, m + 25); ++k) a1[m * K + k] = (int8_t)(rng() & 255);
      for (int z = 0; z < batch; ++z) CK(cudaMemcpy(dA + z * M * K, a1.data(), M * K, cudaMemcpyHostToDevice));
    } else
    for (long long o = 0; o < batch * M * K; o += h.size())
      CK(cudaMemcpy(dA + o, h.data(), std::min<long long>(h.size(), batch * M * K - o), cudaMemcpyHostToDevice));
    for (long long o = 0; o < batch * N * K; o += h.size())
      CK(cudaMemcpy(dB + o, h.data(), std::min<long long>(h.size(), batch * N * K - o), cudaMemcpyHostToDevice));
  }
  IgemmArgs g; g.M = M; g.N = N; g.K = K; g.batch = batch; g.A = dA; g.lda = K; g.strideA = M * K;
  g.B = dB; g.ldb = K; g.strideB = N * K; g.C = dC; g.ldc = N; g.strideC = M * N; g.out = IG_OUT_MOD; g.moduli = dm; g.nmod = 2;
  g.ksplit = ks;
  std::string err;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  igemm(0, g, &err);
  CK(cudaDeviceSynchronize());
  const int reps = 3;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) igemm(0, g, &err);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  printf("%s K.U shape M=%lld N=%lld K=%lld batch=%d gm=%s ksplit=%d: %.3f ms  %.1f TOPS\n",
         getenv("BANDED_A") ? "banded-A" : "random", M, N, K, batch,
         getenv("TRAJ_IGEMM_GM") ? getenv("TRAJ_IGEMM_GM") : "16", ks, ms, 2.0 * M * N * K * batch / ms / 1e9);
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dm);
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "ku") {   // the c3 K U launch shape: 48 products, random data
    timeit_rand(16384, 8192, 16384, 48);
    return 0;
  }
  if (argc > 5 && std::string(argv[1]) == "shape") {   // shape M N K batch (random operands, modular epilogue)
    timeit_rand(atoll(argv[2]), atoll(argv[3]), atoll(argv[4]), atoi(argv[5]));
    return 0;
  }
  int bad = 0;
  bad |= check(300, 520, 1000, 2, IG_OUT_I32, 0);
  bad |= check(128, 256, 128, 1, IG_OUT_I32, 0);
  bad |= check(300, 520, 1000, 2, IG_OUT_MOD, 0);
  bad |= check(700, 700, 700, 1, IG_OUT_I32, IG_UPPER);
  bad |= check(400, 700, 700, 1, IG_OUT_I32, IG_TRI_B);
  bad |= check(300, 520, 1000, 2, IG_OUT_I32, 0, 3);
  bad |= check(300, 520, 1000, 2, IG_OUT_MOD, 0, 4);
  bad |= check(400, 700, 700, 1, IG_OUT_I32, IG_TRI_B, 2);
  if (bad) { printf("CHECK FAILED\n"); return 1; }
  timeit(8192, 8192, 8192, 1, IG_OUT_I32);
  timeit(8192, 8192, 8192, 4, IG_OUT_MOD);
  timeit(16384, 8192, 16384, 6, IG_OUT_MOD);
  return 0;
}
