// CholeskyQR pass 1 on the structure G = I - V^dag V (structchol.h).
//
// Column blocks c of width b, sequential over c (Schur complement of the leading blocks):
//   Y = M V_c,  C_c = I - V_c^dag Y = R_c^dag R_c,  X_c = R_c^-1,  W_c = V_c X_c,  Z_c = M W_c,
//   M <- M + Z_c Z_c^dag                                  (= M + Y C_c^-1 Y^dag)
// so that R_cc = R_c and R_{c,d} = -Z_c^dag V_d (d > c).  The solve dst = src R^-1 then runs over
// the column blocks with the accumulator A = sum_{d < c} dst_d Z_d^dag:
//   dst_c = src_c X_c + A W_c,   A <- A + dst_c Z_c^dag.
// Rows of V past k0 are zero and every reduction over them is bounded by k0 on the device (zgemm.h
// DevBounds), so launches are sized by the host's capacity kc and the step stays asynchronous.
#include <algorithm>

#include "cholinv.h"
#include "monitor.h"
#include "structchol.h"
#include "zgemm.h"

namespace traj {

#define SC_TRY(x)         \
  do {                    \
    int s_ = (x);         \
    if (s_) return s_;    \
  } while (0)

namespace {

// block c of the structured factor (see struct_chol_factor)
int factor_block(cudaStream_t st, StructChol& s, const cplx* V, long long ldV, long long sV, const int32_t* k_dev,
                 int32_t* failed, std::string* err, int c) {
  const int b = s.b, N = s.N, kc = s.kc, T = s.T;
  DevBounds bk;
  bk.k = k_dev;
  bk.m = k_dev;
  DevBounds bm;
  bm.m = k_dev;
  DevBounds bmn;
  bmn.m = k_dev;
  bmn.n = k_dev;
  const int nblk = (int)ceil_div(N, b);
    const int c0 = c * b, bc = std::min(b, N - c0);
    const cplx* Vc = V + c0;
    cplx* Xc = s.Xb + (long long)c0 * b;
    // Y = M V_c (kc x bc);  C = I - V_c^dag Y (upper);  X_c = chol_inv(C)
    SC_TRY(zgemm(st, 0, 0, kc, bc, kc, 1.0, 0.0, s.M, s.ldM, s.sM, Vc, ldV, sV, 0.0, s.Y, b, s.sY, T, 0, err, 0, 0,
                 &bk));
    SC_TRY(set_identity(st, s.C, b, s.sC, bc, T, err));
    DevBounds bkk;  // the b x b C: reduction over k0 only
    bkk.k = k_dev;
    SC_TRY(zgemm(st, 1, 0, bc, bc, kc, -1.0, 0.0, Vc, ldV, sV, s.Y, b, s.sY, 1.0, s.C, b, s.sC, T, TRAJ_C_UPPER_F, err,
                 0, 0, &bkk));
    SC_TRY(chol_inverse(st, bc, s.C, b, s.sC, Xc, b, s.sXb, T, s.chol_scratch, failed, err));
    // W_c = V_c X_c,  Z_c = M W_c  (the block's columns of W, Z)
    SC_TRY(zgemm(st, 0, 0, kc, bc, bc, 1.0, 0.0, Vc, ldV, sV, Xc, b, s.sXb, 0.0, s.W + c0, s.ldWZ, s.sWZ, T,
                 TRAJ_TRI_B_UPPER_F, err, 0, 0, &bm));
    SC_TRY(zgemm(st, 0, 0, kc, bc, kc, 1.0, 0.0, s.M, s.ldM, s.sM, s.W + c0, s.ldWZ, s.sWZ, 0.0, s.Z + c0, s.ldWZ,
                 s.sWZ, T, 0, err, 0, 0, &bk));
    // M += Z_c Z_c^dag
    if (c + 1 < nblk)
      SC_TRY(zgemm(st, 0, 1, kc, kc, bc, 1.0, 0.0, s.Z + c0, s.ldWZ, s.sWZ, s.Z + c0, s.ldWZ, s.sWZ, 1.0, s.M, s.ldM,
                   s.sM, T, 0, err, 0, 0, &bmn));
    return 0;
}

int factor_init(cudaStream_t st, StructChol& s, std::string* err) {
  // M = I
  if (cudaMemsetAsync(s.M, 0, (size_t)((s.T - 1) * s.sM + (long long)s.kc * s.ldM) * 16, st) != cudaSuccess) {
    if (err) *err = "struct_chol: memset";
    return 4;
  }
  return axpby_identity(st, s.M, s.ldM, s.sM, s.kc, s.T, 1.0, 1.0, err);
}

}  // namespace

int struct_chol_factor(cudaStream_t st, StructChol& s, const cplx* V, long long ldV, long long sV,
                       const int32_t* k_dev, int32_t* failed, std::string* err) {
  SC_TRY(factor_init(st, s, err));
  const int nblk = (int)ceil_div(s.N, s.b);
  for (int c = 0; c < nblk; ++c) SC_TRY(factor_block(st, s, V, ldV, sV, k_dev, failed, err, c));
  return 0;
}

int struct_chol_apply(cudaStream_t st, const StructChol& s, int Lr, const cplx* src, cplx* dst, long long ldU,
                      long long sU, cplx* A, long long ldA, long long sA, const int32_t* k_dev, std::string* err) {
  const int b = s.b, N = s.N, kc = s.kc, T = s.T;
  DevBounds bk, bn;  // reductions over / outputs of the k0 columns of A
  bk.k = k_dev;
  bn.n = k_dev;
  // dst = src blockdiag(X_c): the full blocks as one batched launch per trajectory, then the tail
  const int nblk = (int)ceil_div(N, b), nfull = N / b;
  for (int t = 0; t < T; ++t) {
    if (nfull > 0)
      SC_TRY(zgemm(st, 0, 0, Lr, b, b, 1.0, 0.0, src + t * sU, ldU, b, s.Xb + t * s.sXb, b, (long long)b * b, 0.0,
                   dst + t * sU, ldU, b, nfull, TRAJ_TRI_B_UPPER_F, err));
    if (nfull < nblk) {
      const int c0 = nfull * b, bc = N - c0;
      SC_TRY(zgemm(st, 0, 0, Lr, bc, bc, 1.0, 0.0, src + t * sU + c0, ldU, 0, s.Xb + t * s.sXb + (long long)c0 * b, b,
                   0, 0.0, dst + t * sU + c0, ldU, 0, 1, TRAJ_TRI_B_UPPER_F, err));
    }
  }
  // the sequential part: dst_c += A W_c,  A (+)= dst_c Z_c^dag
  for (int c = 0; c < nblk; ++c) {
    const int c0 = c * b, bc = std::min(b, N - c0);
    if (c > 0)
      SC_TRY(zgemm(st, 0, 0, Lr, bc, kc, 1.0, 0.0, A, ldA, sA, s.W + c0, s.ldWZ, s.sWZ, 1.0, dst + c0, ldU, sU, T, 0,
                   err, 0, 0, &bk));
    if (c + 1 < nblk)
      SC_TRY(zgemm(st, 0, 1, Lr, kc, bc, 1.0, 0.0, dst + c0, ldU, sU, s.Z + c0, s.ldWZ, s.sWZ, c > 0 ? 1.0 : 0.0, A,
                   ldA, sA, T, 0, err, 0, 0, &bn));
  }
  return 0;
}

int struct_chol_factor_events(cudaStream_t st, StructChol& s, const cplx* V, long long ldV, long long sV,
                              const int32_t* k_dev, int32_t* failed, cudaEvent_t* ev, std::string* err) {
  SC_TRY(factor_init(st, s, err));
  const int nblk = (int)ceil_div(s.N, s.b);
  for (int c = 0; c < nblk; ++c) {
    SC_TRY(factor_block(st, s, V, ldV, sV, k_dev, failed, err, c));
    if (cudaEventRecord(ev[c], st) != cudaSuccess) {
      if (err) *err = "struct_chol_factor_events: event record";
      return 4;
    }
  }
  return 0;
}

int struct_chol_pipelined(cudaStream_t st, cudaStream_t aux, cudaEvent_t* ev, int nev, StructChol& s, const cplx* V,
                          long long ldV, long long sV, const int32_t* k_dev, int32_t* failed, int Lr, const cplx* src,
                          cplx* dst, long long ldU, long long sU, cplx* A, long long ldA, long long sA,
                          std::string* err) {
  const int b = s.b, N = s.N, kc = s.kc, T = s.T;
  const int nblk = (int)ceil_div(N, b);
  if (nblk > nev) {
    if (err) *err = "struct_chol_pipelined: too few events";
    return 1;
  }
  // the factor chain on aux, an event after each block
  SC_TRY(factor_init(aux, s, err));
  for (int c = 0; c < nblk; ++c) {
    SC_TRY(factor_block(aux, s, V, ldV, sV, k_dev, failed, err, c));
    if (cudaEventRecord(ev[c], aux) != cudaSuccess) {
      if (err) *err = "struct_chol_pipelined: event record";
      return 4;
    }
  }
  // the solve on st, block c after factor block c
  DevBounds bk, bn;
  bk.k = k_dev;
  bn.n = k_dev;
  for (int c = 0; c < nblk; ++c) {
    const int c0 = c * b, bc = std::min(b, N - c0);
    if (cudaStreamWaitEvent(st, ev[c], 0) != cudaSuccess) {
      if (err) *err = "struct_chol_pipelined: event wait";
      return 4;
    }
    // dst_c = src_c X_c (+ A W_c), A (+)= dst_c Z_c^dag
    SC_TRY(zgemm(st, 0, 0, Lr, bc, bc, 1.0, 0.0, src + c0, ldU, sU, s.Xb + (long long)c0 * b, b, s.sXb, 0.0, dst + c0,
                 ldU, sU, T, TRAJ_TRI_B_UPPER_F, err));
    if (c > 0)
      SC_TRY(zgemm(st, 0, 0, Lr, bc, kc, 1.0, 0.0, A, ldA, sA, s.W + c0, s.ldWZ, s.sWZ, 1.0, dst + c0, ldU, sU, T, 0,
                   err, 0, 0, &bk));
    if (c + 1 < nblk)
      SC_TRY(zgemm(st, 0, 1, Lr, kc, bc, 1.0, 0.0, dst + c0, ldU, sU, s.Z + c0, s.ldWZ, s.sWZ, c > 0 ? 1.0 : 0.0, A,
                   ldA, sA, T, 0, err, 0, 0, &bn));
  }
  return 0;
}

}  // namespace traj
