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

// S_c = I - sum_{d<c} H_d on the k0 x k0 block (identity elsewhere), upper triangle, for c < nblk:
// one thread per (i, j), the prefix over c sequential in registers (H_d = V_d V_d^dag in H, d < nblk - 1)
__global__ void struct_prefix_kernel(const cplx* __restrict__ H, cplx* __restrict__ S, long long ld, long long sS,
                                     int kc, int nblk, const int32_t* __restrict__ k_dev) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= kc || j >= kc || i > j) return;
  const int k0 = k_dev ? *k_dev : kc;
  const bool in = i < k0 && j < k0;
  const double d = i == j ? 1.0 : 0.0;
  double re = 0.0, im = 0.0;
  const long long o = (long long)i * ld + j;
  for (int c = 0; c < nblk; ++c) {
    S[c * sS + o] = make_double2(in ? d - re : d, in ? -im : 0.0);
    if (c + 1 < nblk) {
      const cplx h = H[c * sS + o];
      re += h.x;
      im += h.y;
    }
  }
}

// E_d <- sum_{d' <= d} E_d' for d < n, on the Lr x k0 block of each (the columns past k0 are never read)
__global__ void struct_prefix_rows_kernel(cplx* __restrict__ E, long long ld, long long sE, int Lr, int kc, int n,
                                          const int32_t* __restrict__ k_dev) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const long long i = blockIdx.y;
  const int k0 = k_dev ? *k_dev : kc;
  if (j >= k0 || i >= Lr) return;
  cplx* p = E + i * ld + j;
  double re = 0.0, im = 0.0;
  for (int d = 0; d < n; ++d) {
    const cplx e = p[d * sE];
    re += e.x;
    im += e.y;
    p[d * sE] = make_double2(re, im);
  }
}

// failed[0] = 1 if any of the n flags is set
__global__ void struct_or_flags_kernel(int32_t* failed, const int32_t* __restrict__ f, int n) {
  int any = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) any |= f[i];
  any = __syncthreads_or(any);
  if (threadIdx.x == 0 && any && failed) *failed = 1;
}

}  // namespace

int struct_chol_factor(cudaStream_t st, StructChol& s, const cplx* V, long long ldV, long long sV,
                       const int32_t* k_dev, int32_t* failed, std::string* err) {
  if (s.Sb) return struct_chol_factor_batched(st, s, V, ldV, sV, k_dev, failed, err);
  SC_TRY(factor_init(st, s, err));
  const int nblk = (int)ceil_div(s.N, s.b);
  for (int c = 0; c < nblk; ++c) SC_TRY(factor_block(st, s, V, ldV, sV, k_dev, failed, err, c));
  return 0;
}

int struct_chol_factor_batched(cudaStream_t st, StructChol& s, const cplx* V, long long ldV, long long sV,
                               const int32_t* k_dev, int32_t* failed, std::string* err) {
  const int b = s.b, N = s.N, kc = s.kc, T = s.T;
  const int nblk = (int)ceil_div(N, b), nfull = N / b;
  const int ct = N - nfull * b;   // the ragged last block's width (0: none)
  const long long bb = (long long)b * b, sQ = (long long)kc * b;
  s.Vsrc = V;
  s.ldVsrc = ldV;
  s.sVsrc = sV;
  for (int t = 0; t < T; ++t) {
    const cplx* Vt = V + t * sV;
    cplx* Xt = s.Xb + t * s.sXb;
    cplx* Wt = s.W + t * s.sWZ;
    cplx* Zt = s.Z + t * s.sWZ;
    DevBounds bmn, bk, bm;   // this trajectory's k0 for every batch entry (the blocks)
    bmn.m = bmn.n = k_dev + t;
    bmn.per_batch = 0;
    bk.k = k_dev + t;
    bk.per_batch = 0;
    bm.m = k_dev + t;
    bm.per_batch = 0;
    // H_d = V_d V_d^dag (upper tiles of the k0 x k0 block), d < nblk - 1 (all full blocks)
    if (nblk > 1)
      SC_TRY(zgemm(st, 0, 1, kc, kc, b, 1.0, 0.0, Vt, ldV, b, Vt, ldV, b, 0.0, s.XMb, s.ldS, s.sS, nblk - 1,
                   TRAJ_C_UPPER_F, err, 0, 0, &bmn));
    {
      const dim3 blk(32, 8), grd((unsigned)ceil_div(kc, 32), (unsigned)ceil_div(kc, 8));
      struct_prefix_kernel<<<grd, blk, 0, st>>>(s.XMb, s.Sb, s.ldS, s.sS, kc, nblk, k_dev + t);
    }
    if (cudaMemsetAsync(s.bfail, 0, (size_t)2 * nblk * 4, st) != cudaSuccess) {
      if (err) *err = "struct_chol_factor_batched: memset";
      return 4;
    }
    // X_S,c = R_S,c^-1 (S_0 = I gives X_S,0 = I)
    SC_TRY(chol_inverse(st, kc, s.Sb, s.ldS, s.sS, s.XMb, s.ldS, s.sS, nblk, s.bscratch, s.bfail, err));
    // Q_c = X_S,c^dag V_c (lower-triangular op(A); rows past k0 come out zero)
    if (nfull > 0)
      SC_TRY(zgemm(st, 1, 0, kc, b, kc, 1.0, 0.0, s.XMb, s.ldS, s.sS, Vt, ldV, b, 0.0, s.Qb, b, sQ, nfull,
                   TRAJ_TRI_A_LOWER_F, err, 0, 0, &bk));
    if (ct)
      SC_TRY(zgemm(st, 1, 0, kc, ct, kc, 1.0, 0.0, s.XMb + nfull * s.sS, s.ldS, 0, Vt + (long long)nfull * b, ldV, 0,
                   0.0, s.Qb + nfull * sQ, b, 0, 1, TRAJ_TRI_A_LOWER_F, err, 0, 0, &bk));
    // C_c = I - Q_c^dag Q_c (upper), X_c = R_c^-1 into the blocks of Xb
    SC_TRY(set_identity(st, s.Cb, b, bb, b, nblk, err));
    if (nfull > 0) {
      SC_TRY(zgemm(st, 1, 0, b, b, kc, -1.0, 0.0, s.Qb, b, sQ, s.Qb, b, sQ, 1.0, s.Cb, b, bb, nfull, TRAJ_C_UPPER_F,
                   err, 0, 0, &bk));
      SC_TRY(chol_inverse(st, b, s.Cb, b, bb, Xt, b, bb, nfull, s.bscratch, s.bfail + nblk, err));
    }
    if (ct) {
      SC_TRY(zgemm(st, 1, 0, ct, ct, kc, -1.0, 0.0, s.Qb + nfull * sQ, b, 0, s.Qb + nfull * sQ, b, 0, 1.0,
                   s.Cb + nfull * bb, b, 0, 1, TRAJ_C_UPPER_F, err, 0, 0, &bk));
      SC_TRY(chol_inverse(st, ct, s.Cb + nfull * bb, b, 0, Xt + nfull * bb, b, 0, 1, s.bscratch,
                          s.bfail + nblk + nfull, err));
    }
    // W_c = V_c X_c (rows < k0), T1_c = Q_c X_c (into Sb), Z_c = X_S,c T1_c
    auto block_products = [&](int c_first, int count, int w) -> int {
      const long long c0 = (long long)c_first * b;
      const long long sx = count > 1 ? bb : 0, sv = count > 1 ? b : 0, sq = count > 1 ? sQ : 0,
                      ss = count > 1 ? s.sS : 0;
      SC_TRY(zgemm(st, 0, 0, kc, w, w, 1.0, 0.0, Vt + c0, ldV, sv, Xt + c_first * bb, b, sx, 0.0, Wt + c0, s.ldWZ, sv,
                   count, TRAJ_TRI_B_UPPER_F, err, 0, 0, &bm));
      SC_TRY(zgemm(st, 0, 0, kc, w, w, 1.0, 0.0, s.Qb + c_first * sQ, b, sq, Xt + c_first * bb, b, sx, 0.0,
                   s.Sb + c_first * s.sS, b, ss, count, TRAJ_TRI_B_UPPER_F, err));
      SC_TRY(zgemm(st, 0, 0, kc, w, kc, 1.0, 0.0, s.XMb + c_first * s.sS, s.ldS, ss, s.Sb + c_first * s.sS, b, ss,
                   0.0, Zt + c0, s.ldWZ, sv, count, TRAJ_TRI_A_UPPER_F, err, 0, 0, &bk));
      return 0;
    };
    if (nfull > 0) SC_TRY(block_products(0, nfull, b));
    if (ct) SC_TRY(block_products(nfull, 1, ct));
    struct_or_flags_kernel<<<1, 256, 0, st>>>(failed ? failed + t : nullptr, s.bfail, 2 * nblk);
    if (cudaGetLastError() != cudaSuccess) {
      if (err) *err = "struct_chol_factor_batched: launch";
      return 4;
    }
  }
  return 0;
}

// dst = src R^-1 without the chain over blocks (structchol.h Eb).  The chain's accumulator obeys
// A_{c+1} = A_c F_c + src_c X_c Z_c^dag with F_c = I + W_c Z_c^dag = M_c^-1 M_{c+1}, so
// A_c = sum_{d<c} src_d X_d Z_d^dag S_{d+1} M_c, and X_d Z_d^dag S_{d+1} = X_d W_d^dag (I - M_d V_d V_d^dag)
// = X_d (X_d^dag V_d^dag - (X_d^dag - R_d) V_d^dag) = X_d R_d V_d^dag = V_d^dag (C_d = R_d^dag R_d =
// I - V_d^dag M_d V_d).  Hence A_c = P_c M_c with P_c = sum_{d<c} src_d V_d^dag, and A_c W_c = P_c Z_c.
int struct_chol_apply_batched(cudaStream_t st, const StructChol& s, int Lr, const cplx* src, cplx* dst,
                              long long ldU, long long sU, const int32_t* k_dev, std::string* err) {
  const int b = s.b, N = s.N, kc = s.kc, T = s.T;
  const int nblk = (int)ceil_div(N, b), nfull = N / b;
  for (int t = 0; t < T; ++t) {
    const cplx* st_src = src + t * sU;
    cplx* st_dst = dst + t * sU;
    const cplx* Vt = s.Vsrc + t * s.sVsrc;
    const cplx* Xt = s.Xb + t * s.sXb;
    const cplx* Zt = s.Z + t * s.sWZ;
    DevBounds bn, bk;
    bn.n = k_dev + t;
    bn.per_batch = 0;
    bk.k = k_dev + t;
    bk.per_batch = 0;
    // dst_c = src_c X_c for every block (the full ones batched, then the tail)
    if (nfull > 0)
      SC_TRY(zgemm(st, 0, 0, Lr, b, b, 1.0, 0.0, st_src, ldU, b, Xt, b, (long long)b * b, 0.0, st_dst, ldU, b, nfull,
                   TRAJ_TRI_B_UPPER_F, err));
    if (nfull < nblk) {
      const int c0 = nfull * b, bc = N - c0;
      SC_TRY(zgemm(st, 0, 0, Lr, bc, bc, 1.0, 0.0, st_src + c0, ldU, 0, Xt + (long long)c0 * b, b, 0, 0.0,
                   st_dst + c0, ldU, 0, 1, TRAJ_TRI_B_UPPER_F, err));
    }
    if (nblk < 2) continue;
    // E_d = src_d V_d^dag (d < nblk - 1: full blocks), then P_{d+1} = E_0 + ... + E_d in place
    SC_TRY(zgemm(st, 0, 1, Lr, kc, b, 1.0, 0.0, st_src, ldU, b, Vt, s.ldVsrc, b, 0.0, s.Eb, s.ldE, s.sE, nblk - 1, 0,
                 err, 0, 0, &bn));
    {
      const dim3 grd((unsigned)ceil_div(kc, 128), (unsigned)Lr);
      struct_prefix_rows_kernel<<<grd, 128, 0, st>>>(s.Eb, s.ldE, s.sE, Lr, kc, nblk - 1, k_dev + t);
      if (cudaGetLastError() != cudaSuccess) {
        if (err) *err = "struct_chol_apply_batched: launch";
        return 4;
      }
    }
    // dst_c += P_c Z_c, c >= 1 (reduction over the k0 columns of P_c)
    const int nf1 = nfull - 1;   // full blocks among c >= 1
    if (nf1 > 0)
      SC_TRY(zgemm(st, 0, 0, Lr, b, kc, 1.0, 0.0, s.Eb, s.ldE, s.sE, Zt + b, s.ldWZ, b, 1.0, st_dst + b, ldU, b, nf1,
                   0, err, 0, 0, &bk));
    if (nfull < nblk) {
      const int c = nfull, c0 = c * b, bc = N - c0;
      SC_TRY(zgemm(st, 0, 0, Lr, bc, kc, 1.0, 0.0, s.Eb + (c - 1) * s.sE, s.ldE, 0, Zt + c0, s.ldWZ, 0, 1.0,
                   st_dst + c0, ldU, 0, 1, 0, err, 0, 0, &bk));
    }
  }
  return 0;
}

int struct_chol_apply(cudaStream_t st, const StructChol& s, int Lr, const cplx* src, cplx* dst, long long ldU,
                      long long sU, cplx* A, long long ldA, long long sA, const int32_t* k_dev, std::string* err) {
  const int b = s.b, N = s.N, kc = s.kc, T = s.T;
  if (s.Eb) return struct_chol_apply_batched(st, s, Lr, src, dst, ldU, sU, k_dev, err);
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
  const int nblk = (int)ceil_div(s.N, s.b);
  if (s.Sb) SC_TRY(struct_chol_factor_batched(st, s, V, ldV, sV, k_dev, failed, err));
  else SC_TRY(factor_init(st, s, err));
  for (int c = 0; c < nblk; ++c) {
    if (!s.Sb) SC_TRY(factor_block(st, s, V, ldV, sV, k_dev, failed, err, c));
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
  if (s.Sb) SC_TRY(struct_chol_factor_batched(aux, s, V, ldV, sV, k_dev, failed, err));
  else SC_TRY(factor_init(aux, s, err));
  for (int c = 0; c < nblk; ++c) {
    if (!s.Sb) SC_TRY(factor_block(aux, s, V, ldV, sV, k_dev, failed, err, c));
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

// The solve dst = src R^-1 with its products on the INT8 modular path: the block-diagonal part
// dst_c = src_c X_c from one row split of src (each block's k-range is a byte offset into the
// residues), then per block c
//   dst_c += A W_c   (A = sum_{d<c} dst_d Z_d^dag, Lr x k0; W_c past row k0 taken as zero)
//   A (+)= dst_c Z_c^dag  (columns past k0 skipped)
// with k0 bounding the INT8 launches on the device.
int struct_chol_apply_oz(cudaStream_t st, const StructChol& s, const OzWork& w, int Lr, const cplx* src, cplx* dst,
                         long long ldU, long long sU, cplx* A, long long ldA, long long sA, const int32_t* k0,
                         const cudaEvent_t* ev, std::string* err) {
  const int b = s.b, N = s.N, kc = s.kc, T = s.T, sq = w.s;
  const int nblk = (int)ceil_div(N, b);
  // the product scratch in two halves: outputs, and the per-block residues of A / dst_c (src's row
  // residues stay in RU for every block's block-diagonal product)
  const size_t half = (size_t)oz_residue_bytes(3, sq, T, Lr, std::max(kc, b));
  // interleaved (block c's solve right after its factor block) when the scratch holds both halves;
  // otherwise all block-diagonal products first, then the sequential part with its residues in RU
  const bool inter = 2 * half + 256 <= w.RC_bytes;
  uint8_t* RCo = w.RC;
  int8_t* R2 = inter ? reinterpret_cast<int8_t*>(w.RC + (half + 255) / 256 * 256) : w.RU;
  auto prod = [&](int M, int Nn, int K, const int8_t* RA, long long lda, const int* eA, const int8_t* RB,
                  const int* eB, cplx* C, long long ldc, long long sC, const cplx* base, int flags, const int32_t* kdev,
                  const int32_t* ndev) {
    OzProduct p;
    p.M = M;
    p.N = Nn;
    p.K = K;
    p.T = T;
    p.s = sq;
    p.RA = RA;
    p.a_traj = 1;
    p.lda_override = lda;
    p.eA = eA;
    p.sEA = w.sEU;
    p.RB = RB;
    p.eB = eB;
    p.sEB = w.sEX;
    p.RC = RCo;
    p.C = C;
    p.ldc = ldc;
    p.sC = sC;
    p.base = base;
    p.flags = flags;
    p.kdev = kdev;
    p.ndev = ndev;
    return oz_product(st, p, err);
  };
  // src's row residues once; block c's k-range starts c0 bytes into each row
  SC_TRY(oz_split_rows(st, src, ldU, sU, Lr, N, T, 0, sq, w.RU, w.eU, w.sEU, err));
  auto diag = [&](int c) {   // dst_c = src_c X_c
    const int c0 = c * b, bc = std::min(b, N - c0);
    if (ev && cudaStreamWaitEvent(st, ev[c], 0) != cudaSuccess) {   // factor block c done (pipelined)
      if (err) *err = "struct_chol_apply_oz: event wait";
      return 4;
    }
    SC_TRY(oz_split_cols(st, s.Xb + (long long)c0 * b, b, s.sXb, bc, bc, T, 3, sq, w.RX, w.eX, w.sEX, w.part, err));
    SC_TRY(prod(Lr, bc, bc, w.RU + c0, oz_ld(N), w.eU, w.RX, w.eX, dst + c0, ldU, sU, nullptr, OZ_TRI_B, nullptr,
                nullptr));
    return 0;
  };
  if (!inter)
    for (int c = 0; c < nblk; ++c) SC_TRY(diag(c));
  for (int c = 0; c < nblk; ++c) {
    const int c0 = c * b, bc = std::min(b, N - c0);
    if (inter) SC_TRY(diag(c));
    if (c > 0) {   // dst_c += A W_c: A's rows (k < k0), W_c's columns (rows past k0 zero)
      SC_TRY(oz_split_rows(st, A, ldA, sA, Lr, kc, T, 0, sq, R2, w.eU2, w.sEU, err, nullptr, k0));
      SC_TRY(oz_split_cols(st, s.W + c0, s.ldWZ, s.sWZ, kc, bc, T, 3, sq, w.RX, w.eX, w.sEX, w.part, err, 0, nullptr,
                           nullptr, k0));
      SC_TRY(prod(Lr, bc, kc, R2, 0, w.eU2, w.RX, w.eX, dst + c0, ldU, sU, dst + c0, 0, k0, nullptr));
    }
    if (c + 1 < nblk) {   // A (+)= dst_c Z_c^dag: dst_c's rows, Z_c's rows conjugated (rows past k0 zero)
      SC_TRY(oz_split_rows(st, dst + c0, ldU, sU, Lr, bc, T, 0, sq, R2, w.eU2, w.sEU, err));
      SC_TRY(oz_split_rows(st, s.Z + c0, s.ldWZ, s.sWZ, kc, bc, T, 1, sq, w.RX, w.eX, w.sEX, err, nullptr, nullptr, 3,
                           k0));
      SC_TRY(prod(Lr, kc, bc, R2, 0, w.eU2, w.RX, w.eX, A, ldA, sA, c > 0 ? A : nullptr, 0, nullptr, k0));
    }
  }
  return 0;
}

}  // namespace traj
