// Internal interface of the INT8 tensor-core GEMM (igemm.cu): tcgen05.mma kind::i8 with TMEM
// accumulators, TMA-fed 128B-swizzled K-major tiles, persistent CTAs.  It is the building block of
// the exact modular (Ozaki-II / CRT) complex-FP64 products in ozaki.cu.
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

enum IgemmOut {
  IG_OUT_I32 = 0,   // C_z[m][n] = sum_k A_z[m][k] B_z[n][k] as int32 (exact: |A|,|B| <= 128, K < 2^17)
  IG_OUT_MOD = 1,   // C_z[m][n] = that sum mod moduli[z % nmod] in [0, m) as uint8
  IG_OUT_MOD_ACC = 2,   // C_z[m][n] = (C_z[m][n] + that sum) mod m: products of k-chunks summed in residues
};

enum IgemmFlags {
  IG_UPPER = 1,     // only tiles that meet the upper triangle (n >= m, global indices) are computed/written
  IG_TRI_B = 2,     // B_z is the transpose of an upper-triangular K x N matrix: B[n][k] = 0 for k > n (k-blocks skipped)
};

struct IgemmArgs {
  long long M = 0, N = 0, K = 0;   // C is M x N, contraction length K
  long long batch = 1;
  const int8_t* A = nullptr;       // [batch_A][M][lda] (K-major rows), batch_A = batch / a_div
  long long lda = 0, strideA = 0;
  int a_div = 1;                    // A_z = A entry z / a_div
  const int8_t* B = nullptr;       // [batch][N][ldb] (K-major rows)
  long long ldb = 0, strideB = 0;
  int b_div = 1;                    // B_z = B entry z / b_div
  void* C = nullptr;               // int32 or uint8 [batch][M][ldc]
  long long ldc = 0, strideC = 0;
  int out = IG_OUT_I32;
  const int* moduli = nullptr;     // device, nmod entries (IG_OUT_MOD)
  int nmod = 1;
  int flags = 0;
  // modular-product batch map (oz_s > 0, ozaki.cu): batch = 3 oz_s oz_T entries z = (p oz_s + q) oz_T + t
  // for product p < 3, modulus q < oz_s, trajectory t; A_z = A entry (oz_pa[p] oz_s + q) Ta + t (Ta =
  // oz_T when oz_a_traj, else 1 and t dropped), B_z likewise; the epilogue's modulus is moduli[q].
  // a_div / b_div / nmod are ignored; oz_na / oz_nb = the number of matrices in the A / B buffers.
  int oz_s = 0, oz_T = 1;
  int oz_np = 3;                    // products per modulus (batch = oz_np oz_s oz_T)
  int oz_pa[3] = {0, 1, 2}, oz_pb[3] = {0, 1, 2};
  int oz_a_traj = 0, oz_b_traj = 1;
  long long oz_na = 0, oz_nb = 0;
  const int32_t* gate = nullptr;   // device flag: when set and *gate == 0 the launch does nothing
  // device bounds per trajectory t (modular map) or per batch entry (plain): the contraction runs over
  // k < kdev[t] only (whole 128-k blocks; the operands must hold zeros in [kdev, round_up(kdev, 128))),
  // and 256-column tiles at n >= ndev[t] are skipped (their outputs are not written)
  const int32_t* kdev = nullptr;
  const int32_t* ndev = nullptr;
  // split-K: the contraction is cut into ksplit chunks of whole 128-k blocks (the chunk outermost in
  // the tile order, so a wave of CTAs shares a K-slab ksplit times narrower through L2); chunk c of
  // batch entry z is written to output matrix z * ksplit + c (the caller sums them: mod m for the
  // modular epilogue)
  int ksplit = 1;
};

// Needs lda, ldb multiples of 16 bytes, 16-byte aligned A/B, ldc a multiple of 16 elements and C
// 16-byte aligned.  Returns 0, 1 (bad argument) or 4 (CUDA error), with *err set.
int igemm(cudaStream_t st, const IgemmArgs& a, std::string* err);

}  // namespace traj
