// Batched Cholesky factorisation with the triangular inverse: G = R^dag R, X = R^-1.
//
// CholeskyQR2 (the per-step QR of P:209) needs only X = R^-1 to apply
// U <- U X as one large triangular GEMM.  The recursion on the 2x2 block split
//     G = [[A, B], [B^dag, C]]:
//   (R_A, X_A) = chol_inv(A)
//   R_B^dag    = B^dag X_A                   (GEMM, B-operand upper triangular)
//   C'         = C - R_B^dag R_B             (Hermitian rank-h update, upper tiles only)
//   (R_C, X_C) = chol_inv(C')
//   X_B        = -X_A (R_B X_C)              (two triangular GEMMs)
// puts (8/3) n^3 of the (4/3 + 4/3) n^3 POTRF + TRTRI flops on the DMMA GEMM; only
// the 64 x 64 diagonal leaves run in a small shared-memory kernel.  R_B^dag is kept in
// G's (unused) strict lower triangle, so the only scratch is the h x (n-h) product.
#include <math.h>
#include "common.cuh"
#include "zgemm.h"
#include "cholinv.h"

namespace traj {

namespace {

constexpr int NB = 64;            // leaf size


// One CTA (1024 threads) per batch entry: n <= 64 diagonal block.  Reads the upper
// triangle of G, writes X = R^-1 (upper) and zeros below the diagonal.  Each thread owns a
// 2 x 2 block of the (identity-padded, full Hermitian) working matrix A and of W in registers.
// Step j of the right-looking elimination (G = L L^dag, L = R^dag): the owners publish row j
// of A and W and column j of A through shared memory; every thread then applies
//   l_i = A_ij / r_jj (= conj R_ji),  A_ik -= l_i A_jk / r_jj (i, k > j),  W_ik -= l_i W_jk / r_jj (i > j),
// W ends as L^-1 (rows scaled by 1/r_jj at their step), so X = R^-1 = W^dag.
template <int TW>   // TW x TW threads, each owning a 2 x 2 block (n <= 2 TW)
__global__ void __launch_bounds__(TW * TW) chol_leaf_kernel(int n, cplx* G, long long ldg, long long sG, cplx* X,
                                                            long long ldx, long long sX, int32_t* failed) {
  __shared__ double2 rowA[NB], rowW[NB], colA[NB];
  __shared__ int bad;
  const int b = blockIdx.x, tid = threadIdx.x;
  const cplx* g = G + b * sG;
  cplx* x = X + b * sX;
  const int i0 = 2 * (tid / TW), k0 = 2 * (tid % TW);
  double2 A[2][2], W[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int i = i0 + a, k = k0 + c;
      double2 v = make_double2(i == k ? 1.0 : 0.0, 0.0);
      if (i < n && k < n) {
        if (i <= k) v = g[(long long)i * ldg + k];
        else {
          const double2 u = g[(long long)k * ldg + i];
          v = make_double2(u.x, -u.y);
        }
      }
      A[a][c] = v;
      W[a][c] = make_double2(i == k ? 1.0 : 0.0, 0.0);
    }
  if (tid == 0) bad = 0;
  for (int j = 0; j < n; ++j) {     // padded identity rows/columns need no elimination
    if ((j >> 1) == (i0 >> 1)) {
      const int a = j & 1;
      rowA[k0] = A[a][0];
      rowA[k0 + 1] = A[a][1];
      rowW[k0] = W[a][0];
      rowW[k0 + 1] = W[a][1];
    }
    if ((j >> 1) == (k0 >> 1)) {
      const int c = j & 1;
      colA[i0] = A[0][c];
      colA[i0 + 1] = A[1][c];
    }
    __syncthreads();
    const double d = rowA[j].x;
    if (tid == 0 && j < n && (!(d > 0.0) || !isfinite(d))) bad = 1;
    const double ip = 1.0 / d;            // l_i * A_jk / r_jj = (A_ij / r)(A_jk / r) = A_ij A_jk / d
    const double ir = 1.0 / sqrt(d);
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int i = i0 + a;
      if (i == j) {
#pragma unroll
        for (int c = 0; c < 2; ++c) W[a][c] = make_double2(W[a][c].x * ir, W[a][c].y * ir);
      } else if (i > j) {
        const double2 l = colA[i];        // A_ij
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int k = k0 + c;
          if (k > j) {
            const double2 r = rowA[k];    // A_jk
            A[a][c].x -= (l.x * r.x - l.y * r.y) * ip;
            A[a][c].y -= (l.x * r.y + l.y * r.x) * ip;
          }
          const double2 w = rowW[k];      // W_jk (unscaled): l/r * W_jk/r
          W[a][c].x -= (l.x * w.x - l.y * w.y) * ip;
          W[a][c].y -= (l.x * w.y + l.y * w.x) * ip;
        }
      }
    }
    __syncthreads();
  }
  // X = W^dag: X_ki = conj(W_ik) for k <= i; zeros below the diagonal
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int i = i0 + a, k = k0 + c;    // element W_ik  ->  X_ki
      if (i < n && k < n) x[(long long)k * ldx + i] = k <= i ? make_double2(W[a][c].x, -W[a][c].y) : make_double2(0.0, 0.0);
    }
  if (tid == 0 && bad && failed) failed[b] = 1;
}

int split(long long n) { return (int)(NB * ceil_div(ceil_div(n, NB), 2)); }

struct Ctx {
  cudaStream_t st;
  cplx* G;
  long long ldg, sG;
  cplx* X;
  long long ldx, sX;
  long long batch;
  cplx* tmp;
  long long ldt, sT;
  int32_t* failed;
  std::string* err;
};

int rec(Ctx& c, long long o, long long n) {
  if (n <= NB) {
    auto leaf = n <= 16 ? chol_leaf_kernel<8> : (n <= 32 ? chol_leaf_kernel<16> : chol_leaf_kernel<32>);
    const int tw = n <= 16 ? 8 : (n <= 32 ? 16 : 32);
    leaf<<<(unsigned)c.batch, tw * tw, 0, c.st>>>((int)n, c.G + o * c.ldg + o, c.ldg, c.sG,
                                                                      c.X + o * c.ldx + o, c.ldx, c.sX, c.failed);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      if (c.err) *c.err = std::string("chol leaf: ") + cudaGetErrorString(e);
      return 4;
    }
    return 0;
  }
  const long long h = split(n), r = n - h;
  cplx* B_blk = c.G + o * c.ldg + (o + h);       // B = G[o:o+h, o+h:o+n]; A = G[o:o+h, o:o+h]
  cplx* L_blk = c.G + (o + h) * c.ldg + o;       // G[o+h:o+n, o:o+h] <- R_B^dag (scratch)
  cplx* C_blk = c.G + (o + h) * c.ldg + (o + h);
  cplx* XA = c.X + o * c.ldx + o;
  cplx* XB = c.X + o * c.ldx + (o + h);
  cplx* XC = c.X + (o + h) * c.ldx + (o + h);
  int s;
  if ((s = rec(c, o, h))) return s;
  // R_B^dag = B^dag X_A : (r x h) = op_C(B: h x r) * X_A (h x h, upper)
  if ((s = zgemm(c.st, 1, 0, r, h, h, 1.0, 0.0, B_blk, c.ldg, c.sG, XA, c.ldx, c.sX, 0.0, L_blk, c.ldg, c.sG, c.batch,
                 TRAJ_TRI_B_UPPER_F, c.err)))
    return s;
  // C -= R_B^dag R_B (upper tiles)
  if ((s = zgemm(c.st, 0, 1, r, r, h, -1.0, 0.0, L_blk, c.ldg, c.sG, L_blk, c.ldg, c.sG, 1.0, C_blk, c.ldg, c.sG,
                 c.batch, TRAJ_C_UPPER_F, c.err)))
    return s;
  if ((s = rec(c, o + h, r))) return s;
  // tmp = R_B X_C : (h x r) = op_C(L_blk: r x h) * X_C (r x r, upper)
  if ((s = zgemm(c.st, 1, 0, h, r, r, 1.0, 0.0, L_blk, c.ldg, c.sG, XC, c.ldx, c.sX, 0.0, c.tmp, c.ldt, c.sT, c.batch,
                 TRAJ_TRI_B_UPPER_F, c.err)))
    return s;
  // X_B = -X_A tmp
  if ((s = zgemm(c.st, 0, 0, h, r, h, -1.0, 0.0, XA, c.ldx, c.sX, c.tmp, c.ldt, c.sT, 0.0, XB, c.ldx, c.sX, c.batch,
                 TRAJ_TRI_A_UPPER_F, c.err)))
    return s;
  return 0;
}

}  // namespace

size_t chol_scratch_bytes(long long n, long long batch) {
  if (n <= NB) return 256;
  const long long h = split(n);
  return (size_t)(batch * h * round_up(n, 8) * 16);
}

int chol_inverse(cudaStream_t st, long long n, cplx* G, long long ldg, long long sG, cplx* X, long long ldx,
                 long long sX, long long batch, void* scratch, int32_t* failed, std::string* err) {
  if (n <= 0 || batch <= 0) return 0;
  if (batch > 65535) {
    if (err) *err = "chol_inverse: batch too large";
    return 1;
  }
  Ctx c;
  c.st = st;
  c.G = G;
  c.ldg = ldg;
  c.sG = sG;
  c.X = X;
  c.ldx = ldx;
  c.sX = sX;
  c.batch = batch;
  c.tmp = reinterpret_cast<cplx*>(scratch);
  c.ldt = round_up(n, 8);
  c.sT = n <= NB ? 0 : split(n) * c.ldt;
  c.failed = failed;
  c.err = err;
  if (n > NB) {
    // the strict lower triangle of X must read as zeros (triangular GEMM tiles cross it)
    cudaError_t e = cudaSuccess;
    if (batch == 1 || sX == n * ldx) {
      e = cudaMemset2DAsync(X, (size_t)ldx * 16, 0, (size_t)n * 16, (size_t)(n * batch), st);
    } else {
      for (long long b = 0; b < batch && e == cudaSuccess; ++b)
        e = cudaMemset2DAsync(X + b * sX, (size_t)ldx * 16, 0, (size_t)n * 16, (size_t)n, st);
    }
    if (e != cudaSuccess) {
      if (err) *err = std::string("chol_inverse memset: ") + cudaGetErrorString(e);
      return 4;
    }
  }
  return rec(c, 0, n);
}

}  // namespace traj
