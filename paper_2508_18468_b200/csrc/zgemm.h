// Internal interface of the DMMA complex GEMM (zgemm.cu).
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

enum {
  TRAJ_TRI_A_UPPER_F = 1,
  TRAJ_TRI_A_LOWER_F = 2,
  TRAJ_TRI_B_UPPER_F = 4,
  TRAJ_TRI_B_LOWER_F = 8,
  TRAJ_C_UPPER_F = 16
};

// Bounds read on the device when the kernel runs, so that a launch sized on the host by a capacity
// needs no host round trip for a data-dependent size (the projective click counts) or decision (the
// CholeskyQR2 fallback).  Every pointer may be null.
//   gate: the launch does nothing unless *gate != 0;
//   m, n: rows / columns of C needed: output tiles starting at or past them exit (the rest of a
//         straddling tile is written with values the caller must not use);
//   k:    the reduction extent: k-blocks starting at or past k are skipped -- the operands must hold
//         zeros in the rest of the last block (zero-padded rows / columns), so the sum is exact.
//   per_batch: n[b], k[b] for batch entry b (else n[0], k[0] for every entry).
struct DevBounds {
  const int32_t* gate = nullptr;
  const int32_t* m = nullptr;
  const int32_t* n = nullptr;
  const int32_t* k = nullptr;
  int per_batch = 1;
};

// C_b = alpha op(A_b) op(B_b) + beta C_b.  Returns 0, or a traj_status with *err set.
// m_off, n_off: the global row / column of this call's C(0, 0) when it computes a slice of a larger
// product; only the triangle (TRI_*) and upper-tile (C_UPPER) tests use them.
int zgemm(cudaStream_t st, int opA, int opB, long long M, long long N, long long K, double alpha_re,
          double alpha_im, const cplx* A, long long lda, long long strideA, const cplx* B, long long ldb,
          long long strideB, double beta, cplx* C, long long ldc, long long strideC, long long batch, int flags,
          std::string* err, long long m_off = 0, long long n_off = 0, const DevBounds* db = nullptr);

// 0: 4M (two real MMAs over an interleaved k axis); 1: 3M (Gauss, three real MMAs; the default).
// Initialised from the environment (TRAJ_ZGEMM_3M=0 selects 4M); process-wide.
int zgemm_algorithm();
void set_zgemm_algorithm(int algo);

}  // namespace traj
