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
};

// From V ([T][kc rows][ldV], rows past k_dev[t] zero): the blocks' R_c^-1, W and Z.  failed[t] is set
// on a non-positive pivot (as the dense factorisation would).
int struct_chol_factor(cudaStream_t st, StructChol& s, const cplx* V, long long ldV, long long sV,
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
