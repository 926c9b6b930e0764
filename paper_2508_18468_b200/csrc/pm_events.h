// Internal interface of the event-driven projective protocol (pm_events.cu, NEXT-4).
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

// Axis taps: neighbour offsets lo .. lo+n-1 (mod the extent) with coefficients c[0..n).
// yhat = r_j / |r_j| with r_j row j of K(tau) U; coef = [alpha, beta, occ, p]; ++*occ_count if occupied
int event_prep(cudaStream_t st, const cplx* U, long long ld, int N, int Lx, int Ly, int j, const cplx* cx, int xlo,
               int xn, const cplx* cy, int ylo, int yn, double pc, cplx* yhat, double* coef, int32_t* occ_count,
               std::string* err);
// out = K(tau) U + x yhat, x = alpha (K(tau) U yhat^dag) + beta e_j (coef == nullptr: propagation only)
int event_update(cudaStream_t st, const cplx* U, cplx* out, long long ld, int N, int Lx, int Ly, const cplx* cx,
                 int xlo, int xn, const cplx* cy, int ylo, int yn, const cplx* yhat, const double* coef, int j,
                 std::string* err);

}  // namespace traj
