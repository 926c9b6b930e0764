// Internal interface of the real FP64 DMMA GEMM (dgemm.cu): the building block of the planar 3M
// complex product.
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

// C_z = alpha A_z B_z + beta C_z (row-major, no transposes), z < batch (stride 0: shared operand).
// Needs K > 0, even lda and ldc, ldb a multiple of 16 with round_up(N, 16) <= ldb (whole 16-column
// chunks of B are read; the extra columns feed discarded outputs), 16-byte aligned pointers.
int dgemm_nn(cudaStream_t st, long long M, long long N, long long K, double alpha, const double* A, long long lda,
             long long strideA, const double* B, long long ldb, long long strideB, double beta, double* C,
             long long ldc, long long strideC, long long batch, std::string* err);

}  // namespace traj
