// Internal interface of the orthonormality probe (probe.cu): a randomized certificate that the
// low-rank (Loewdin) projective step kept U^dag U = I, so the CholeskyQR refinement pass runs
// only when the accumulated rounding drift exceeds a tolerance (NEXT-1 option).
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

constexpr int PROBE_M = 4;        // probe vectors per trajectory
constexpr int PROBE_RS_MAX = 32;  // row splits of the U^dag Y pass

// scratch: X [T][N][PROBE_M], Y [T][L][PROBE_M], partial [T][PROBE_RS_MAX][N][PROBE_M] (complex),
// est [T] (double).
size_t probe_x_bytes(long long N, int T);
size_t probe_y_bytes(long long L, int T);
size_t probe_partial_bytes(long long N, int T);

// est[t] = sqrt( (1/m) sum_j || U_t^dag (U_t x_j) - x_j ||^2 ), an estimate of ||U_t^dag U_t - I||_F
// (Hutchinson: E[x x^dag] = I).  x_kj = (+-1 +- i)/sqrt(2) from Philox (k, step, traj_base + t, 3).
// U: T row-major L x N blocks (leading dimension ld, batch stride sU).  Device result est[T].
int probe_orthonormality(cudaStream_t st, const cplx* U, long long ld, long long sU, int L, int N, int T,
                         long long step, long long traj_base, uint64_t seed, cplx* X, cplx* Y, cplx* partial,
                         double* est, std::string* err);

}  // namespace traj
