// Internal interface of the batched Cholesky + triangular inverse (cholinv.cu).
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

size_t chol_scratch_bytes(long long n, long long batch);

// G_b = R^dag R (upper triangle of G_b read; strict lower triangle used as scratch),
// X_b = R^-1 (upper; strict lower set to zero).  failed[b] = 1 on a non-positive or
// non-finite pivot.
int chol_inverse(cudaStream_t st, long long n, cplx* G, long long ldg, long long sG, cplx* X, long long ldx,
                 long long sX, long long batch, void* scratch, int32_t* failed, std::string* err);

}  // namespace traj
