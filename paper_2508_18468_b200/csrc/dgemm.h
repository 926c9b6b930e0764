// Internal interface of the real FP64 DMMA GEMM (dgemm.cu): the building block of the planar 3M
// complex product.
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

enum { DG_TRI_B_UPPER = 4, DG_C_UPPER = 16 };   // the values of zgemm.h's TRAJ_TRI_B_UPPER_F / TRAJ_C_UPPER_F

// C_z = alpha op(A_z) B_z + beta C_z, row-major real matrices, z < batch (stride 0: shared operand);
// op(A) = A (opA = 0, A stored [M][K]) or A^T (opA = 1, A stored [K][M]).  flags: DG_TRI_B_UPPER
// (B upper triangular: k-blocks past the diagonal skipped), DG_C_UPPER (only C's upper triangle is
// written); m_off / n_off: global row / column of C(0, 0) for those tests.  Needs K > 0, even lda
// and ldc, ldb a multiple of 16 with round_up(N, 16) <= ldb (and for opA = 1 the same of lda and M:
// whole 16-column chunks are read; the extra columns feed discarded outputs), 16-byte alignment.
int dgemm(cudaStream_t st, int opA, long long M, long long N, long long K, double alpha, const double* A,
          long long lda, long long strideA, const double* B, long long ldb, long long strideB, double beta, double* C,
          long long ldc, long long strideC, long long batch, int flags, std::string* err, long long m_off = 0,
          long long n_off = 0, int a_div = 1);   // a_div: batch entries per A entry (A_z = A entry z / a_div)

inline int dgemm_nn(cudaStream_t st, long long M, long long N, long long K, double alpha, const double* A,
                    long long lda, long long strideA, const double* B, long long ldb, long long strideB, double beta,
                    double* C, long long ldc, long long strideC, long long batch, std::string* err) {
  return dgemm(st, 0, M, N, K, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC, batch, 0, err);
}

}  // namespace traj
