// CholeskyQR pass 1 on the structure of its Gram (structchol.cu).
//
// After a projective step the Gram of U' (rows S0 of an orthonormal U zeroed) is G = I - V^dag V,
// V the k0 zeroed rows (k0 << N).  Every Schur complement of G is then I - V^dag M V with a k0 x k0
// matrix M, so the N x N Cholesky factor R (G = R^dag R) and the solve U' R^-1 need O(N k0^2) and
// O(L N k0 + L N b) flops instead of O(N^3) and O(L N^2) -- the same R and the same U' R^-1, up to
// rounding, as the dense CholeskyQR pass.
#pragma once
#include <string>
#include "common.cuh"
#include "ozaki.h"

namespace traj {

struct StructChol {
  int b = 128;                          // column block
  int N = 0, kc = 0, T = 1;             // columns, capacity of the k0 rows, batch
  cplx* M = nullptr;                    // [T][kc][ldM]  the Schur-complement matrix
  long long ldM = 0, sM = 0;
  cplx* Y = nullptr;                    // [T][kc][b]    M V_c
  long long sY = 0;
  cplx* C = nullptr;                    // [T][b][b]     I - V_c^dag M V_c
  long long sC = 0;
  cplx* Xb = nullptr;                   // [T][ceil(N/b) b][b]  R_c^-1 of every block
  long long sXb = 0;
  cplx *W = nullptr, *Z = nullptr;      // [T][kc][ldWZ] W = V_c R_c^-1, Z = M W by column blocks
  long long ldWZ = 0, sWZ = 0;
  void* chol_scratch = nullptr;         // chol_scratch_bytes(b, T)
  // the batched factor (struct_chol_factor_batched; null Sb: the sequential chain).  Per trajectory,
  // for every block c of the nblk = ceil(N / b) column blocks at once:
  cplx* Sb = nullptr;                   // [nblk][kc][ldS]  S_c = I - sum_{d<c} V_d V_d^dag, then Q_c X_c ([kc][b])
  cplx* XMb = nullptr;                  // [nblk][kc][ldS]  the block Grams V_d V_d^dag, then R_S,c^-1
  long long ldS = 0, sS = 0;            // ldS >= kc, sS >= kc max(ldS, b)
  cplx* Qb = nullptr;                   // [nblk][kc][b]    Q_c = R_S,c^-dag V_c
  cplx* Cb = nullptr;                   // [nblk][b][b]     I - Q_c^dag Q_c
  void* bscratch = nullptr;             // max(chol_scratch_bytes(kc, nblk), chol_scratch_bytes(b, nblk))
  int32_t* bfail = nullptr;             // [2 nblk] the batched factorisations' pivot flags
  // the batched solve (struct_chol_apply when Eb is set): the accumulator of the chain,
  // A_c = sum_{d<c} dst_d Z_d^dag, equals P_c M_c with P_c = sum_{d<c} src_d V_d^dag (push-through
  // identity, structchol.cu), so dst_c = src_c X_c + P_c Z_c with every P_c a prefix sum of the blocks'
  // src_d V_d^dag -- no product waits for another block's dst
  cplx* Eb = nullptr;                   // [nblk - 1][Lr][ldE]  src_d V_d^dag, then the prefix sums P_{d+1}
  long long ldE = 0, sE = 0;
  const cplx* Vsrc = nullptr;           // V as passed to the factor (recorded by struct_chol_factor_batched)
  long long ldVsrc = 0, sVsrc = 0;
};

// From V ([T][kc rows][ldV], rows past k_dev[t] zero): the blocks' R_c^-1, W and Z.  failed[t] is set
// on a non-positive pivot (as the dense factorisation would).
int struct_chol_factor(cudaStream_t st, StructChol& s, const cplx* V, long long ldV, long long sV,
                       const int32_t* k_dev, int32_t* failed, std::string* err);

// The same blocks without the sequential chain over c (used by every entry point when s.Sb is set).
// The chain's M before block c is M_c = (I - sum_{d<c} V_d V_d^dag)^-1 (each step of the chain is the
// Woodbury update of this inverse), so with S_c = I - sum_{d<c} V_d V_d^dag = R_S^dag R_S, X_S = R_S^-1
// (M_c = X_S X_S^dag) and Q_c = X_S^dag V_c:
//   C_c = I - V_c^dag M_c V_c = I - Q_c^dag Q_c,  X_c = chol_inv(C_c),  W_c = V_c X_c,  Z_c = M_c W_c = X_S (Q_c X_c)
// -- every block is independent: one batched launch per product over the nblk blocks (plus the
// ragged last block), two batched factorisations, instead of ~8 dependent launches per block.
int struct_chol_factor_batched(cudaStream_t st, StructChol& s, const cplx* V, long long ldV, long long sV,
                               const int32_t* k_dev, int32_t* failed, std::string* err);

// dst = src R^-1 for Lr rows of U ([T][Lr][ldU], batch stride sU); A: [T][Lr][ldA] scratch (the
// L x k0 accumulator), ldA >= kc.
int struct_chol_apply(cudaStream_t st, const StructChol& s, int Lr, const cplx* src, cplx* dst, long long ldU,
                      long long sU, cplx* A, long long ldA, long long sA, const int32_t* k_dev, std::string* err);

// The factor and the solve pipelined over two streams: block c's factor (a chain of small launches) is
// issued on aux, and the solve of block c on st waits only for it (events ev[0..nblk), created by the
// caller), so the latency-bound factor chain runs under the solve's L-row GEMMs.  V is read on aux:
// the caller orders aux after V's producer; st is joined with aux on return.  Same results as
// struct_chol_factor followed by struct_chol_apply.
// struct_chol_factor with an event recorded on st after each block c (ev[c], created by the caller)
int struct_chol_factor_events(cudaStream_t st, StructChol& s, const cplx* V, long long ldV, long long sV,
                              const int32_t* k_dev, int32_t* failed, cudaEvent_t* ev, std::string* err);

int struct_chol_pipelined(cudaStream_t st, cudaStream_t aux, cudaEvent_t* ev, int nev, StructChol& s, const cplx* V,
                          long long ldV, long long sV, const int32_t* k_dev, int32_t* failed, int Lr, const cplx* src,
                          cplx* dst, long long ldU, long long sU, cplx* A, long long ldA, long long sA,
                          std::string* err);

// struct_chol_apply with its products on the INT8 modular path (ozaki.h; many zeroed rows, c5: k0 ~
// 1830): dst_c = src_c X_c from one row split of src, then per block c dst_c += A W_c and
// A (+)= dst_c Z_c^dag (A: Lr x k0, accumulated), k_dev bounding the launches on the device.  ev
// (optional): block c's solve waits for ev[c] (the factor on another stream, struct_chol_factor_events).
int struct_chol_apply_oz(cudaStream_t st, const StructChol& s, const OzWork& w, int Lr, const cplx* src, cplx* dst,
                         long long ldU, long long sU, cplx* A, long long ldA, long long sA, const int32_t* k_dev,
                         const cudaEvent_t* ev, std::string* err);

}  // namespace traj
