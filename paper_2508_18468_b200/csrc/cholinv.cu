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
constexpr int LD = NB + 1;        // padded smem row (complex)
constexpr int LEAF_THREADS = 256;

__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// One CTA per batch entry: n <= 64 diagonal block.  Reads the upper triangle of G,
// writes X = R^-1 (upper) and zeros below the diagonal.  Right-looking elimination with
// G = L L^dag (L = R^dag): step j scales row j of the working matrix A (its final row of
// R) and row j of W, then eliminates rows i > j in A (upper part) and applies the same
// row operation to W; W ends as L^-1, so X = R^-1 = W^dag.  Two barriers per column.
__global__ void __launch_bounds__(LEAF_THREADS) chol_leaf_kernel(int n, cplx* G, long long ldg, long long sG, cplx* X,
                                                                  long long ldx, long long sX, int32_t* failed) {
  extern __shared__ double2 sm[];
  double2* R = sm;               // [NB][LD]  working matrix -> R (upper)
  double2* Ws = sm + NB * LD;    // [NB][LD]  -> L^-1 (lower)
  __shared__ int bad;
  const int b = blockIdx.x, tid = threadIdx.x;
  const cplx* g = G + b * sG;
  cplx* x = X + b * sX;
  if (tid == 0) bad = 0;
  for (int idx = tid; idx < n * n; idx += LEAF_THREADS) {
    const int i = idx / n, j = idx % n;
    if (i <= j) R[i * LD + j] = g[(long long)i * ldg + j];
    Ws[i * LD + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    // (1) pivot and scaling of row j (every thread reads the pivot itself: no extra barrier)
    const double d = R[j * LD + j].x;
    const double r = sqrt(d);
    const double ip = 1.0 / r;
    if (tid == 0 && (!(d > 0.0) || !isfinite(d))) bad = 1;
    __syncthreads();     // all threads have read R[j][j] before it is overwritten
    for (int k = j + tid; k < n; k += LEAF_THREADS) {
      const double2 v = R[j * LD + k];
      R[j * LD + k] = k == j ? make_double2(r, 0.0) : make_double2(v.x * ip, v.y * ip);
    }
    for (int k = tid; k <= j; k += LEAF_THREADS) {
      const double2 v = Ws[j * LD + k];
      Ws[j * LD + k] = make_double2(v.x * ip, v.y * ip);
    }
    __syncthreads();
    // (2) eliminate rows i > j: l_ij = conj(R_ji)
    const int m = n - j - 1;
    const int wA = m * m, wW = m * (j + 1);
    for (int idx = tid; idx < wA + wW; idx += LEAF_THREADS) {
      if (idx < wA) {
        const int i = j + 1 + idx / m, k = j + 1 + idx % m;
        if (i <= k) {
          const double2 p = cmulc(R[j * LD + i], R[j * LD + k]);
          R[i * LD + k].x -= p.x;
          R[i * LD + k].y -= p.y;
        }
      } else {
        const int q = idx - wA;
        const int i = j + 1 + q / (j + 1), k = q % (j + 1);
        const double2 p = cmulc(R[j * LD + i], Ws[j * LD + k]);
        Ws[i * LD + k].x -= p.x;
        Ws[i * LD + k].y -= p.y;
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < n * n; idx += LEAF_THREADS) {
    const int i = idx / n, j = idx % n;     // X_ij = conj(W_ji), upper
    const double2 w = Ws[j * LD + i];
    x[(long long)i * ldx + j] = i <= j ? make_double2(w.x, -w.y) : make_double2(0.0, 0.0);
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
    static bool attr = false;
    const int smem = 2 * NB * LD * sizeof(double2);
    if (!attr) {
      cudaFuncSetAttribute(chol_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    chol_leaf_kernel<<<(unsigned)c.batch, LEAF_THREADS, smem, c.st>>>((int)n, c.G + o * c.ldg + o, c.ldg, c.sG,
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
