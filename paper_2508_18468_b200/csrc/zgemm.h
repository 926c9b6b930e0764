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

// C_b = alpha op(A_b) op(B_b) + beta C_b.  Returns 0, or a traj_status with *err set.
// m_off, n_off: the global row / column of this call's C(0, 0) when it computes a slice of a larger
// product; only the triangle (TRI_*) and upper-tile (C_UPPER) tests use them.
int zgemm(cudaStream_t st, int opA, int opB, long long M, long long N, long long K, double alpha_re,
          double alpha_im, const cplx* A, long long lda, long long strideA, const cplx* B, long long ldb,
          long long strideB, double beta, cplx* C, long long ldc, long long strideC, long long batch, int flags,
          std::string* err, long long m_off = 0, long long n_off = 0);

// 0: 4M (two real MMAs over an interleaved k axis); 1: 3M (Gauss, three real MMAs; the default).
// Initialised from the environment (TRAJ_ZGEMM_3M=0 selects 4M); process-wide.
int zgemm_algorithm();
void set_zgemm_algorithm(int algo);

}  // namespace traj
