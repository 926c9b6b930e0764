// Internal interface of the paper-literal RK4 QSD propagation (qsd_rk4.cu, NEXT-2).
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

// out = P4(X) U with X = -i dt J H~ + diag(d), d = dW + (2 n - 1) gamma dt (n: device [T][L] at
// time t); Wtmp: a scratch buffer shaped like U; d: device [T][L] scratch.
int qsd_rk4_propagate(cudaStream_t st, const cplx* U, cplx* Wtmp, cplx* out, long long ld, long long sU, int Lx,
                      int Ly, int N, int T, const double* n, double* d, long long step, long long traj_base,
                      uint64_t seed, const double* gamma_dev, double J, double dt, std::string* err);

}  // namespace traj
