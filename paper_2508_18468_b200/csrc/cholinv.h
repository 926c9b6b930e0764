// Internal interface of the batched Cholesky + triangular inverse (cholinv.cu).
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

size_t chol_scratch_bytes(long long n, long long batch);

// Distribution of the large recursion levels over the P ranks of a row-sharded trajectory (SURVEY
// §8(e): the replicated N x N factorisation bounds the sharded speed-up).  At every level with
// n >= min_n the four GEMMs are split into P row slices (128-row aligned; equal triangle area for
// the Hermitian update): rank r computes slice r, then share_rows() makes every slice visible on
// every rank.  rank < 0: a single-process emulation that computes every slice itself (share_rows
// is not called).  Only batch == 1.
struct CholDist {
  int P = 1, rank = 0;
  long long min_n = 2048;
  void* user = nullptr;
  // the block of ncols columns at base (row-major, leading dimension ld): rows [bounds[i],
  // bounds[i+1]) were computed by rank i
  int (*share_rows)(void* user, cplx* base, long long ld, long long ncols, const long long* bounds, int P,
                    cudaStream_t st, std::string* err) = nullptr;
};

// Called (on the host, in launch order) whenever a left-edge block X[0:h, 0:h] of the recursion has
// been queued on the stream (h increasing: 64, 128, ..., the top split): columns [0, h) of X are
// final from that point of the stream on.
struct CholHook {
  void (*left_ready)(void* user, long long h) = nullptr;
  void* user = nullptr;
};

// Optional workspace that runs the four products of every recursion level with n >= min_n as exact
// modular products on the INT8 tensor cores (ozaki.h): RA >= 4 s batch n^2/2 (rounded), RB >= 3 s batch
// n^2/2, RC >= 3 s batch n^2/2 bytes (upper bounds for the top level), eA / eB >= batch n ints each (row
// stride n), part >= 8 batch n doubles.
struct CholOzaki {
  int s = 16;
  long long min_n = 4096;
  int8_t* RA = nullptr;
  int8_t* RB = nullptr;
  uint8_t* RC = nullptr;
  int* eA = nullptr;
  int* eB = nullptr;
  long long sE = 0;        // exponent stride per batch entry (>= n)
  double* part = nullptr;
};

// G_b = R^dag R (upper triangle of G_b read; strict lower triangle used as scratch),
// X_b = R^-1 (upper; strict lower set to zero).  failed[b] = 1 on a non-positive or
// non-finite pivot.  gate (device, may be null): every kernel of the factorisation does nothing
// unless *gate != 0 -- the CholeskyQR2 fallback decided on the device, without a host round trip.
// With a gate X is not touched when gated off, and must already be zero below its diagonal.
int chol_inverse(cudaStream_t st, long long n, cplx* G, long long ldg, long long sG, cplx* X, long long ldx,
                 long long sX, long long batch, void* scratch, int32_t* failed, std::string* err,
                 const CholDist* dist = nullptr, const CholHook* hook = nullptr, const int32_t* gate = nullptr, const CholOzaki* oz = nullptr);

// CholeskyQR2's second-pass fallback as one CUDA graph: a decide node (any trajectory's max|G2 - I|,
// the bit pattern in dev[t], above thr) sets the condition of an IF node whose body is the captured
// chol_inverse(n) of these buffers.  One graph launch per step instead of the factorisation's
// ~640 gated kernel launches; the body runs only when needed.  build() returns non-zero when the
// runtime cannot build it (the caller keeps the gated launches).
struct CholFallbackGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int build(long long n, cplx* G, long long ldg, long long sG, cplx* X, long long ldx, long long sX, long long batch,
            void* scratch, int32_t* failed, const unsigned long long* dev, double thr, unsigned long long* fallbacks,
            std::string* err, const CholOzaki* oz = nullptr);
  int launch(cudaStream_t st, std::string* err);
  void destroy();
};

}  // namespace traj
