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
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "zgemm.h"
#include "cholinv.h"
#include "comm_plan.h"

namespace traj {

namespace {

constexpr int NB = 64;            // leaf size


// One CTA per batch entry: n <= 64 diagonal block.  Reads the upper triangle of G, writes
// X = R^-1 (upper) and zeros below the diagonal.  Each of the TW x TW threads owns a BS x BS
// block of the (identity-padded) working matrix A (upper triangle kept) and of W in registers.
// Step j of the right-looking elimination (G = L L^dag, L = R^dag): the owners of row j publish
// row j of A and W and the pivot scalars 1/d, 1/sqrt(d) (double-buffered, so one barrier per
// step; only the diagonal owner evaluates the rsqrt); A is Hermitian, so the column entry A_ij
// is conj(A_ji) and needs no second broadcast.  Every thread then applies
//   A_ik -= A_ij A_jk / d  (j < i <= k),   W_ik -= A_ij W_jk / d  (i > j, k <= j),   d = A_jj,
// and the owners of row j scale it by 1/sqrt(d).  W ends as L^-1, so X = R^-1 = W^dag.
template <int TW, int BS>
__global__ void __launch_bounds__(TW * TW) chol_leaf_kernel(int n, cplx* G, long long ldg, long long sG, cplx* X,
                                                            long long ldx, long long sX, int32_t* failed,
                                                            const int32_t* gate) {
  if (gate && *gate == 0) return;
  __shared__ double2 rowA[2][TW * BS], rowW[2][TW * BS], piv[2];
  __shared__ int bad;
  const int b = blockIdx.x, tid = threadIdx.x;
  const cplx* g = G + b * sG;
  cplx* x = X + b * sX;
  const int i0 = BS * (tid / TW), k0 = BS * (tid % TW);
  double2 A[BS][BS], W[BS][BS];
#pragma unroll
  for (int a = 0; a < BS; ++a)
#pragma unroll
    for (int c = 0; c < BS; ++c) {
      const int i = i0 + a, k = k0 + c;
      double2 v = make_double2(i == k ? 1.0 : 0.0, 0.0);
      if (i <= k && k < n) v = g[(long long)i * ldg + k];
      A[a][c] = v;
      W[a][c] = make_double2(i == k ? 1.0 : 0.0, 0.0);
    }
  if (tid == 0) bad = 0;
  for (int j = 0; j < n; ++j) {     // padded identity rows/columns need no elimination
    const int buf = j & 1;
    if (j >= i0 && j < i0 + BS) {
#pragma unroll
      for (int a = 0; a < BS; ++a)
        if (i0 + a == j) {
#pragma unroll
          for (int c = 0; c < BS; ++c) {
            rowA[buf][k0 + c] = A[a][c];
            rowW[buf][k0 + c] = W[a][c];
            if (k0 + c == j) {              // the diagonal owner publishes the pivot scalars
              const double d = A[a][c].x;
              if (!(d > 0.0) || !isfinite(d)) bad = 1;
              const double ir = rsqrt(d);
              piv[buf] = make_double2(ir * ir, ir);
            }
          }
        }
    }
    __syncthreads();
    const double ip = piv[buf].x;           // 1 / d
    const double ir = piv[buf].y;           // 1 / sqrt(d)
    if (i0 + BS - 1 < j) continue;          // rows all eliminated
#pragma unroll
    for (int a = 0; a < BS; ++a) {
      const int i = i0 + a;
      if (i == j) {
#pragma unroll
        for (int c = 0; c < BS; ++c) W[a][c] = make_double2(W[a][c].x * ir, W[a][c].y * ir);
      } else if (i > j) {
        const double2 u = rowA[buf][i];     // A_ji;  A_ij = conj(u)
        const double lx = u.x * ip, ly = -u.y * ip;
#pragma unroll
        for (int c = 0; c < BS; ++c) {
          const int k = k0 + c;
          if (k > j) {
            if (k >= i) {
              const double2 r = rowA[buf][k];   // A_jk
              A[a][c].x -= lx * r.x - ly * r.y;
              A[a][c].y -= lx * r.y + ly * r.x;
            }
          } else {
            const double2 w = rowW[buf][k];     // W_jk (unscaled)
            W[a][c].x -= lx * w.x - ly * w.y;
            W[a][c].y -= lx * w.y + ly * w.x;
          }
        }
      }
    }
  }
  // X = W^dag: X_ki = conj(W_ik) for k <= i; zeros below the diagonal
#pragma unroll
  for (int a = 0; a < BS; ++a)
#pragma unroll
    for (int c = 0; c < BS; ++c) {
      const int i = i0 + a, k = k0 + c;    // element W_ik  ->  X_ki
      if (i < n && k < n) x[(long long)k * ldx + i] = k <= i ? make_double2(W[a][c].x, -W[a][c].y) : make_double2(0.0, 0.0);
    }
  __syncthreads();
  if (tid == 0 && bad && failed) failed[b] = 1;
}

// The same leaf by Gaussian elimination of [G | I] in shared memory (the fused small step's
// scheme, small_step.cu): 16 warps, rows on warps and columns on lanes, two pivots per barrier --
// row a + 1 after pivot a is formed on the fly (m = conj(G_a,a+1) / p_a, p_a+1 = G_a+1,a+1 -
// |G_a,a+1|^2 / p_a) and each row i > a + 1 takes row_i -= c_a row_a + c_b row_a+1 with
// c_b = conj(G_a+1,i - m G_a,i) / p_a+1, c_a = conj(G_a,i) / p_a - c_b m; W's row a + 1 becomes
// W_a+1 - m W_a one phase later.  W ends as L^-1 of G = L D L^dag on unscaled rows and
// X = R^-1 = W^dag D^-1/2.  A non-positive pivot flags the batch entry and fills X with NaN.
constexpr int EW = 16;            // warps of the elimination leaf
constexpr int ELD = NB + 1;

__device__ __forceinline__ void pending_w_row(double2* Ws, const double2* Gs, const double* piv, int prev, int lane) {
  const double2 g = Gs[prev * ELD + prev + 1];
  const double ip = 1.0 / piv[prev];
  const double mx = g.x * ip, my = -g.y * ip;
  for (int k = lane; k <= prev; k += 32) {
    const double2 w = Ws[prev * ELD + k];
    Ws[(prev + 1) * ELD + k].x -= mx * w.x - my * w.y;
    Ws[(prev + 1) * ELD + k].y -= mx * w.y + my * w.x;
  }
}

__global__ void __launch_bounds__(EW * 32) chol_leaf_elim_kernel(int n, const cplx* G, long long ldg, long long sG,
                                                                 cplx* X, long long ldx, long long sX, int32_t* failed,
                                                                 const int32_t* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) double2 lsm[];
  double2* Gs = lsm;                 // [NB][ELD] upper triangle, eliminated in place
  double2* Ws = lsm + NB * ELD;      // [NB][ELD] W = L^-1 (lower)
  __shared__ double piv[NB];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const cplx* g = G + b * sG;
  cplx* x = X + b * sX;
  for (int i = warp; i < n; i += EW)
    for (int k = lane; k < n; k += 32) {
      if (k >= i) Gs[i * ELD + k] = g[(long long)i * ldg + k];
      Ws[i * ELD + k] = make_double2(i == k ? 1.0 : 0.0, 0.0);
    }
  __syncthreads();
  bool bad = false;
  int prev = -1;
  for (int j = 0; j < n; j += 2) {
    const bool pair = j + 1 < n;
    const double pa = Gs[j * ELD + j].x;
    if (!(pa > 0.0) || !isfinite(pa)) {   // the same value in every thread: uniform exit
      bad = true;
      break;
    }
    const double ia = 1.0 / pa;
    double2 mm = make_double2(0.0, 0.0);
    double ib = 0.0;
    if (pair) {
      const double2 gab = Gs[j * ELD + j + 1];
      mm = make_double2(gab.x * ia, -gab.y * ia);
      const double pb = Gs[(j + 1) * ELD + j + 1].x - (gab.x * gab.x + gab.y * gab.y) * ia;
      if (!(pb > 0.0) || !isfinite(pb)) {
        bad = true;
        break;
      }
      ib = 1.0 / pb;
      if (tid == 0) piv[j + 1] = pb;
    }
    if (tid == 0) piv[j] = pa;
    if (prev >= 0 && warp == EW - 1) pending_w_row(Ws, Gs, piv, prev, lane);
    const int bb = pair ? j + 1 : j;
    for (int i = bb + 1 + warp; i < n; i += EW) {
      const double2 gai = Gs[j * ELD + i];
      const double lax = gai.x * ia, lay = -gai.y * ia;
      double cax = lax, cay = lay, cbx = 0.0, cby = 0.0;
      if (pair) {
        const double2 gbi = Gs[(j + 1) * ELD + i];
        const double px = gbi.x - (mm.x * gai.x - mm.y * gai.y), py = gbi.y - (mm.x * gai.y + mm.y * gai.x);
        cbx = px * ib;
        cby = -py * ib;
        cax = lax - (cbx * mm.x - cby * mm.y);
        cay = lay - (cbx * mm.y + cby * mm.x);
      }
      for (int k = i + lane; k < n; k += 32) {
        const double2 ra = Gs[j * ELD + k];
        double2 v = Gs[i * ELD + k];
        v.x -= cax * ra.x - cay * ra.y;
        v.y -= cax * ra.y + cay * ra.x;
        if (pair) {
          const double2 rb = Gs[(j + 1) * ELD + k];
          v.x -= cbx * rb.x - cby * rb.y;
          v.y -= cbx * rb.y + cby * rb.x;
        }
        Gs[i * ELD + k] = v;
      }
      for (int k = lane; k <= bb; k += 32) {
        const double2 wa = Ws[j * ELD + k];
        double2 v = Ws[i * ELD + k];
        v.x -= cax * wa.x - cay * wa.y;
        v.y -= cax * wa.y + cay * wa.x;
        if (pair) {
          const double2 wb = Ws[(j + 1) * ELD + k];
          v.x -= cbx * wb.x - cby * wb.y;
          v.y -= cbx * wb.y + cby * wb.x;
        }
        Ws[i * ELD + k] = v;
      }
    }
    prev = pair ? j : -1;
    __syncthreads();
  }
  if (!bad && prev >= 0) {
    if (warp == EW - 1) pending_w_row(Ws, Gs, piv, prev, lane);
    __syncthreads();
  }
  // X_ki = conj(W_ik) / sqrt(p_i) for k <= i, zero below the diagonal
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  for (int k = warp; k < n; k += EW)
    for (int i = lane; i < n; i += 32) {
      double2 v = make_double2(0.0, 0.0);
      if (bad) {
        v = make_double2(nan, nan);
      } else if (k <= i) {
        const double ir = 1.0 / sqrt(piv[i]);
        const double2 w = Ws[i * ELD + k];
        v = make_double2(w.x * ir, -w.y * ir);
      }
      x[(long long)k * ldx + i] = v;
    }
  if (tid == 0 && bad && failed) failed[b] = 1;
}

constexpr int ELEAF_SMEM = 2 * NB * ELD * 16;

// The leaf by 16 x 16 blocks (default; TRAJ_CHOL_LEAF=elim / regs select the others).  A (the upper
// triangle of G, padded with the identity to 64 x 64) and X live in shared memory.  Right-looking over
// the four block columns: warp 0 factors the diagonal block (16 pivots, warp-synchronous) and inverts
// its factor; the block row R_kj = R_kk^-dag A_kj and the trailing update A_ij -= R_ki^dag R_kj are
// 16 x 16 x 16 products, one block per warp; then X = R^-1 by block back-substitution along the
// superdiagonals, X_ij = -R_ii^-1 sum_{i<k<=j} R_ik X_kj.  Four barriers per block column instead of
// one per pivot pair: the 64-pivot dependency chain stays inside one warp.
constexpr int BW = 4;                     // warps of the blocked leaf
constexpr int BLD = NB + 1;               // padded leading dimension (complex)
constexpr int BLEAF_SMEM = (2 * NB * BLD + BW * 16 * 17) * 16;

__device__ __forceinline__ double2 cfma_conj(double2 a, double2 b, double2 acc) {   // acc + conj(a) b
  acc.x += a.x * b.x + a.y * b.y;
  acc.y += a.x * b.y - a.y * b.x;
  return acc;
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {        // acc + a b
  acc.x += a.x * b.x - a.y * b.y;
  acc.y += a.x * b.y + a.y * b.x;
  return acc;
}

// out[r] (rows r0 + r, column c) = sum_k conj(A[k][r0 + r]) B[k][c] over k < 16 (16 x 16 blocks)
__device__ __forceinline__ void warp_ahb(const double2* A, int lda, const double2* B, int ldb, int r0, int c,
                                         double2 (&out)[8]) {
#pragma unroll
  for (int r = 0; r < 8; ++r) out[r] = make_double2(0.0, 0.0);
#pragma unroll 4
  for (int k = 0; k < 16; ++k) {
    const double2 b = B[k * ldb + c];
#pragma unroll
    for (int r = 0; r < 8; ++r) out[r] = cfma_conj(A[k * lda + r0 + r], b, out[r]);
  }
}

// out[r] = sum_k A[r0 + r][k] B[k][c]
__device__ __forceinline__ void warp_ab(const double2* A, int lda, const double2* B, int ldb, int r0, int c,
                                        double2 (&out)[8]) {
#pragma unroll
  for (int r = 0; r < 8; ++r) out[r] = make_double2(0.0, 0.0);
#pragma unroll 4
  for (int k = 0; k < 16; ++k) {
    const double2 b = B[k * ldb + c];
#pragma unroll
    for (int r = 0; r < 8; ++r) out[r] = cfma(A[(r0 + r) * lda + k], b, out[r]);
  }
}

__global__ void __launch_bounds__(BW * 32) chol_leaf_blk_kernel(int n, const cplx* G, long long ldg, long long sG,
                                                                cplx* X, long long ldx, long long sX, int32_t* failed,
                                                                const int32_t* gate) {
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) double2 bsm[];
  double2* As = bsm;                      // [64][BLD]: A, overwritten by R (upper)
  double2* Xs = bsm + NB * BLD;           // [64][BLD]: X = R^-1 (upper)
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2* Ts = bsm + 2 * NB * BLD + warp * 16 * 17;   // this warp's 16 x 16 scratch
  const cplx* g = G + b * sG;
  cplx* x = X + b * sX;
  const int nblk = (n + 15) >> 4;
  for (int idx = tid; idx < NB * NB; idx += BW * 32) {
    const int i = idx >> 6, k = idx & 63;
    double2 v = make_double2(i == k ? 1.0 : 0.0, 0.0);
    if (i < n && k < n && k >= i) v = g[(long long)i * ldg + k];
    As[i * BLD + k] = v;
    Xs[i * BLD + k] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  __shared__ int bad;
  if (tid == 0) bad = 0;
  const int c = lane & 15, r0 = (lane >> 4) * 8;
  for (int kb = 0; kb < nblk; ++kb) {
    const int o = kb * 16;
    double2* D = As + o * BLD + o;
    double2* Xd = Xs + o * BLD + o;
    if (warp == 0) {
      // unblocked Cholesky of the diagonal block: row p of R = row p of A / sqrt(d_p), then
      // A_ik -= conj(R_pi) R_pk for p < i <= k
      for (int p = 0; p < 16; ++p) {
        const double d = D[p * BLD + p].x;
        if (!(d > 0.0) || !isfinite(d)) {
          if (lane == 0) bad = 1;
        }
        const double ir = rsqrt(d);
        __syncwarp();
        if (lane >= p && lane < 16) {
          const double2 v = D[p * BLD + lane];
          D[p * BLD + lane] = make_double2(v.x * ir, v.y * ir);
        }
        __syncwarp();
        for (int e = lane; e < 256; e += 32) {
          const int i = e >> 4, k = e & 15;
          if (i > p && k >= i) {
            const double2 ri = D[p * BLD + i], rk = D[p * BLD + k];
            double2 v = D[i * BLD + k];
            v.x -= ri.x * rk.x + ri.y * rk.y;
            v.y -= ri.x * rk.y - ri.y * rk.x;
            D[i * BLD + k] = v;
          }
        }
        __syncwarp();
      }
      // X_dd = R_dd^-1 (upper): lane c < 16 solves column c by back substitution
      if (lane < 16) {
        double2 col[16];
#pragma unroll
        for (int i = 15; i >= 0; --i) {
          double2 acc = make_double2(i == c ? 1.0 : 0.0, 0.0);
#pragma unroll
          for (int k = i + 1; k < 16; ++k) {
            if (k <= c) {
              const double2 r = D[i * BLD + k];
              acc.x -= r.x * col[k].x - r.y * col[k].y;
              acc.y -= r.x * col[k].y + r.y * col[k].x;
            }
          }
          const double rii = D[i * BLD + i].x;
          col[i] = i <= c ? make_double2(acc.x / rii, acc.y / rii) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) Xd[i * BLD + c] = col[i];
      }
    }
    __syncthreads();
    // block row: R_kj = R_kk^-dag A_kj  (X_dd^dag A_kj)
    for (int j = kb + 1 + warp; j < nblk; j += BW) {
      double2 out[8];
      double2* Akj = As + o * BLD + j * 16;
      warp_ahb(Xd, BLD, Akj, BLD, r0, c, out);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 8; ++r) Akj[(r0 + r) * BLD + c] = out[r];
    }
    __syncthreads();
    // trailing update A_ij -= R_ki^dag R_kj, kb < i <= j
    {
      int t = 0;
      for (int i = kb + 1; i < nblk; ++i)
        for (int j = i; j < nblk; ++j, ++t) {
          if (t % BW != warp) continue;
          double2 out[8];
          warp_ahb(As + o * BLD + i * 16, BLD, As + o * BLD + j * 16, BLD, r0, c, out);
          double2* Aij = As + (i * 16) * BLD + j * 16;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            double2 v = Aij[(r0 + r) * BLD + c];
            v.x -= out[r].x;
            v.y -= out[r].y;
            Aij[(r0 + r) * BLD + c] = v;
          }
        }
    }
    __syncthreads();
  }
  // X_ij = -X_ii sum_{i<k<=j} R_ik X_kj along the superdiagonals d = j - i
  for (int d = 1; d < nblk; ++d) {
    for (int i = warp; i + d < nblk; i += BW) {
      const int j = i + d;
      double2 acc[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[r] = make_double2(0.0, 0.0);
      for (int k = i + 1; k <= j; ++k) {
        double2 out[8];
        warp_ab(As + (i * 16) * BLD + k * 16, BLD, Xs + (k * 16) * BLD + j * 16, BLD, r0, c, out);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          acc[r].x += out[r].x;
          acc[r].y += out[r].y;
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) Ts[(r0 + r) * 17 + c] = acc[r];
      __syncwarp();
      double2 out[8];
      warp_ab(Xs + (i * 16) * BLD + i * 16, BLD, Ts, 17, r0, c, out);
#pragma unroll
      for (int r = 0; r < 8; ++r) Xs[(i * 16 + r0 + r) * BLD + j * 16 + c] = make_double2(-out[r].x, -out[r].y);
      __syncwarp();
    }
    __syncthreads();
  }
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  for (int idx = tid; idx < n * n; idx += BW * 32) {
    const int i = idx / n, k = idx % n;
    x[(long long)i * ldx + k] = bad ? make_double2(nan, nan) : (k >= i ? Xs[i * BLD + k] : make_double2(0.0, 0.0));
  }
  if (tid == 0 && bad && failed) failed[b] = 1;
}

int split(long long n) { return (int)chol_split(n); }

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
  const CholDist* dist;
  const CholHook* hook;
  DevBounds db;            // gate: every launch of the factorisation runs only if *gate != 0
  long long n_top;
  int leaf;                // 0: blocked (default), 1: elimination (TRAJ_CHOL_LEAF=elim), 2: registers (=regs)
};

// row slice boundaries of M rows over P ranks (comm_plan.h row_slices: the schedule the ranks share)
std::vector<long long> slices(long long M, int P, bool tri) { return row_slices(M, P, tri); }

// C rows [0, M) of op(A) op(B) split over the ranks (see CholDist); A's rows (opA = 0) or columns
// (opA = 1) follow the slice
int dist_gemm(Ctx& c, bool tri_c, int opA, int opB, long long M, long long N, long long K, double alpha,
              const cplx* A, long long lda, const cplx* B, long long ldb, double beta, cplx* C, long long ldc,
              int flags) {
  const CholDist* d = c.dist;
  const std::vector<long long> b = slices(M, d->P, tri_c);
  for (int i = 0; i < d->P; ++i) {
    if (d->rank >= 0 && d->rank != i) continue;
    const long long m = b[i + 1] - b[i];
    if (m <= 0) continue;
    const cplx* Ai = opA == 0 ? A + b[i] * lda : A + b[i];
    int s = zgemm(c.st, opA, opB, m, N, K, alpha, 0.0, Ai, lda, 0, B, ldb, 0, beta, C + b[i] * ldc, ldc, 0, 1, flags,
                  c.err, b[i], 0, &c.db);
    if (s) return s;
  }
  if (d->rank < 0) return 0;
  return d->share_rows(d->user, C, ldc, N, b.data(), d->P, c.st, c.err);
}

int rec(Ctx& c, long long o, long long n) {
  if (n <= NB) {
    cudaError_t e = cudaSuccess;
    if (c.leaf == 0) {             // blocked leaf (default)
      e = ensure_smem(reinterpret_cast<const void*>(chol_leaf_blk_kernel), BLEAF_SMEM);
      if (e == cudaSuccess)
        chol_leaf_blk_kernel<<<(unsigned)c.batch, BW * 32, BLEAF_SMEM, c.st>>>(
            (int)n, c.G + o * c.ldg + o, c.ldg, c.sG, c.X + o * c.ldx + o, c.ldx, c.sX, c.failed, c.db.gate);
    } else if (n > 16 && c.leaf == 1) {   // elimination leaf (TRAJ_CHOL_LEAF=elim)
      e = ensure_smem(reinterpret_cast<const void*>(chol_leaf_elim_kernel), ELEAF_SMEM);
      if (e == cudaSuccess)
        chol_leaf_elim_kernel<<<(unsigned)c.batch, EW * 32, ELEAF_SMEM, c.st>>>(
            (int)n, c.G + o * c.ldg + o, c.ldg, c.sG, c.X + o * c.ldx + o, c.ldx, c.sX, c.failed, c.db.gate);
    } else {
      auto leaf = n <= 16 ? chol_leaf_kernel<8, 2> : (n <= 32 ? chol_leaf_kernel<16, 2> : chol_leaf_kernel<32, 2>);
      const int threads = n <= 16 ? 64 : (n <= 32 ? 256 : 1024);
      leaf<<<(unsigned)c.batch, threads, 0, c.st>>>((int)n, c.G + o * c.ldg + o, c.ldg, c.sG, c.X + o * c.ldx + o,
                                                    c.ldx, c.sX, c.failed, c.db.gate);
    }
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
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
  if (o == 0 && c.hook && c.hook->left_ready) c.hook->left_ready(c.hook->user, h);   // X[:, 0:h] final
  if (c.dist && c.dist->P > 1 && n >= c.dist->min_n && c.batch == 1) {
    // the same four products, each split into row slices over the ranks
    if ((s = dist_gemm(c, false, 1, 0, r, h, h, 1.0, B_blk, c.ldg, XA, c.ldx, 0.0, L_blk, c.ldg, TRAJ_TRI_B_UPPER_F)))
      return s;
    if ((s = dist_gemm(c, true, 0, 1, r, r, h, -1.0, L_blk, c.ldg, L_blk, c.ldg, 1.0, C_blk, c.ldg, TRAJ_C_UPPER_F)))
      return s;
    if ((s = rec(c, o + h, r))) return s;
    if ((s = dist_gemm(c, false, 1, 0, h, r, r, 1.0, L_blk, c.ldg, XC, c.ldx, 0.0, c.tmp, c.ldt, TRAJ_TRI_B_UPPER_F)))
      return s;
    if ((s = dist_gemm(c, false, 0, 0, h, r, h, -1.0, XA, c.ldx, c.tmp, c.ldt, 0.0, XB, c.ldx, TRAJ_TRI_A_UPPER_F)))
      return s;
    return 0;
  }
  // R_B^dag = B^dag X_A : (r x h) = op_C(B: h x r) * X_A (h x h, upper)
  if ((s = zgemm(c.st, 1, 0, r, h, h, 1.0, 0.0, B_blk, c.ldg, c.sG, XA, c.ldx, c.sX, 0.0, L_blk, c.ldg, c.sG, c.batch,
                 TRAJ_TRI_B_UPPER_F, c.err, 0, 0, &c.db)))
    return s;
  // C -= R_B^dag R_B (upper tiles)
  if ((s = zgemm(c.st, 0, 1, r, r, h, -1.0, 0.0, L_blk, c.ldg, c.sG, L_blk, c.ldg, c.sG, 1.0, C_blk, c.ldg, c.sG,
                 c.batch, TRAJ_C_UPPER_F, c.err, 0, 0, &c.db)))
    return s;
  if ((s = rec(c, o + h, r))) return s;
  // tmp = R_B X_C : (h x r) = op_C(L_blk: r x h) * X_C (r x r, upper)
  if ((s = zgemm(c.st, 1, 0, h, r, r, 1.0, 0.0, L_blk, c.ldg, c.sG, XC, c.ldx, c.sX, 0.0, c.tmp, c.ldt, c.sT, c.batch,
                 TRAJ_TRI_B_UPPER_F, c.err, 0, 0, &c.db)))
    return s;
  // X_B = -X_A tmp
  if ((s = zgemm(c.st, 0, 0, h, r, h, -1.0, 0.0, XA, c.ldx, c.sX, c.tmp, c.ldt, c.sT, 0.0, XB, c.ldx, c.sX, c.batch,
                 TRAJ_TRI_A_UPPER_F, c.err, 0, 0, &c.db)))
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
                 long long sX, long long batch, void* scratch, int32_t* failed, std::string* err,
                 const CholDist* dist, const CholHook* hook, const int32_t* gate) {
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
  c.dist = dist;
  c.hook = hook;
  c.db.gate = gate;
  c.n_top = n;
  {
    const char* lf = getenv("TRAJ_CHOL_LEAF");
    c.leaf = !lf ? 0 : (lf[0] == 'e' ? 1 : (lf[0] == 'r' ? 2 : 0));
  }
  if (n > NB && !gate) {
    // the strict lower triangle of X must read as zeros (triangular GEMM tiles cross it); with a
    // gate the caller's X (the first-order factor) already is, and must stay intact when gated off
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
