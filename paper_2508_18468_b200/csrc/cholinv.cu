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
#include "ozaki.h"
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
  int leaf;                // 1: elimination (default), 2: register-blocked (TRAJ_CHOL_LEAF=regs)
  const CholOzaki* oz;     // the large levels' products on the INT8 modular path (may be null)
};

// the four products of one recursion level as exact modular products (see rec below for their roles)
int rec_level_ozaki(Ctx& c, long long n, cplx* B_blk, cplx* L_blk, cplx* C_blk, cplx* XA, cplx* XB, cplx* XC,
                    bool before_c) {
  const CholOzaki& z = *c.oz;
  const long long h = split(n), r = n - h;
  const int T = (int)c.batch, sq = z.s;
  const int32_t* gate = c.db.gate;
  auto prod = [&](int M, int N, int K, int a_planes, int pa2, int b_planes, int pb2, const int8_t* RB, int flags,
                  cplx* C, long long ldc, long long sC, const cplx* base) {
    OzProduct p;
    p.M = M;
    p.N = N;
    p.K = K;
    p.T = T;
    p.s = sq;
    p.RA = z.RA;
    p.a_traj = 1;
    p.a_planes = a_planes;
    p.pa[2] = pa2;
    p.eA = z.eA;
    p.sEA = z.sE;
    p.RB = RB;
    p.b_planes = b_planes;
    p.pb[2] = pb2;
    p.eB = z.eB;
    p.sEB = z.sE;
    p.RC = z.RC;
    p.C = C;
    p.ldc = ldc;
    p.sC = sC;
    p.base = base;
    p.flags = flags;
    p.gate = gate;
    return oz_product(c.st, p, c.err);
  };
  int s;
  if (before_c) {
    // L = B^dag X_A (r x h): B's columns conjugated (planes re, im, re - im; P2 negated), X_A's columns
    if ((s = oz_split_cols(c.st, B_blk, c.ldg, c.sG, (int)h, (int)r, T, 4, sq, z.RA, z.eA, z.sE, z.part, c.err, 0,
                           gate)))
      return s;
    if ((s = oz_split_cols(c.st, XA, c.ldx, c.sX, (int)h, (int)h, T, 3, sq, z.RB, z.eB, z.sE, z.part, c.err, 0, gate)))
      return s;
    if ((s = prod((int)r, (int)h, (int)h, 4, 3, 3, 2, z.RB, OZ_NEG_P2 | OZ_TRI_B, L_blk, c.ldg, c.sG, nullptr)))
      return s;
    // C -= L L^dag (upper): one 4-plane row split of L serves both sides
    if ((s = oz_split_rows(c.st, L_blk, c.ldg, c.sG, (int)r, (int)h, T, 0, sq, z.RA, z.eA, z.sE, c.err, gate, nullptr,
                           4)))
      return s;
    {
      OzProduct p;
      p.M = (int)r;
      p.N = (int)r;
      p.K = (int)h;
      p.T = T;
      p.s = sq;
      p.RA = z.RA;
      p.a_traj = 1;
      p.a_planes = 4;
      p.eA = z.eA;
      p.sEA = z.sE;
      p.RB = z.RA;
      p.b_planes = 4;
      p.pb[2] = 3;
      p.eB = z.eA;
      p.sEB = z.sE;
      p.RC = z.RC;
      p.C = C_blk;
      p.ldc = c.ldg;
      p.sC = c.sG;
      p.base = C_blk;
      p.flags = OZ_NEG_P2 | OZ_UPPER | OZ_NEGATE;
      p.gate = gate;
      if ((s = oz_product(c.st, p, c.err))) return s;
    }
    return 0;
  }
  // tmp = L^dag X_C (h x r): L's columns conjugated, X_C's columns
  if ((s = oz_split_cols(c.st, L_blk, c.ldg, c.sG, (int)r, (int)h, T, 4, sq, z.RA, z.eA, z.sE, z.part, c.err, 0, gate)))
    return s;
  if ((s = oz_split_cols(c.st, XC, c.ldx, c.sX, (int)r, (int)r, T, 3, sq, z.RB, z.eB, z.sE, z.part, c.err, 0, gate)))
    return s;
  if ((s = prod((int)h, (int)r, (int)r, 4, 3, 3, 2, z.RB, OZ_NEG_P2 | OZ_TRI_B, c.tmp, c.ldt, c.sT, nullptr))) return s;
  // X_B = -X_A tmp: X_A's rows (its zero lower triangle included), tmp's columns
  if ((s = oz_split_rows(c.st, XA, c.ldx, c.sX, (int)h, (int)h, T, 0, sq, z.RA, z.eA, z.sE, c.err, gate)))
    return s;
  if ((s = oz_split_cols(c.st, c.tmp, c.ldt, c.sT, (int)h, (int)r, T, 3, sq, z.RB, z.eB, z.sE, z.part, c.err, 0, gate)))
    return s;
  return prod((int)h, (int)r, (int)h, 3, 2, 3, 2, z.RB, OZ_NEGATE, XB, c.ldx, c.sX, nullptr);
}

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
    if (n > 16 && c.leaf == 1) {   // elimination leaf (default; TRAJ_CHOL_LEAF=regs: the register-blocked one)
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
  if (c.oz && n >= c.oz->min_n) {   // the same four products on the INT8 modular path
    if ((s = rec_level_ozaki(c, n, B_blk, L_blk, C_blk, XA, XB, XC, true))) return s;
    if ((s = rec(c, o + h, r))) return s;
    return rec_level_ozaki(c, n, B_blk, L_blk, C_blk, XA, XB, XC, false);
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
                 const CholDist* dist, const CholHook* hook, const int32_t* gate, const CholOzaki* oz) {
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
  c.oz = (dist && dist->P > 1) ? nullptr : oz;
  c.db.gate = gate;
  c.n_top = n;
  {
    const char* lf = getenv("TRAJ_CHOL_LEAF");
    c.leaf = (lf && lf[0] == 'r') ? 2 : 1;
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

namespace {

__global__ void fallback_decide_kernel(const unsigned long long* dev, int T, double thr,
                                       cudaGraphConditionalHandle cond, unsigned long long* fallbacks) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned int full = 0;
  for (int t = 0; t < T; ++t)
    if (__longlong_as_double((long long)dev[t]) > thr) full = 1;   // a NaN does not force it
  if (full && fallbacks) fallbacks[0] += 1ull;
  cudaGraphSetConditional(cond, full);
}

}  // namespace

int CholFallbackGraph::build(long long n, cplx* G, long long ldg, long long sG, cplx* X, long long ldx, long long sX,
                             long long batch, void* scratch, int32_t* failed, const unsigned long long* dev, double thr,
                             unsigned long long* fallbacks, std::string* err, const CholOzaki* oz) {
  auto bad = [&](const char* what, cudaError_t e) {
    if (err) *err = std::string("fallback graph: ") + what + ": " + cudaGetErrorString(e);
    destroy();
    return 4;
  };
  cudaError_t e = cudaGraphCreate(&graph, 0);
  if (e != cudaSuccess) return bad("create", e);
  cudaGraphConditionalHandle cond;
  if ((e = cudaGraphConditionalHandleCreate(&cond, graph, 0, 0)) != cudaSuccess) return bad("handle", e);
  int T = (int)batch;
  void* args[] = {const_cast<unsigned long long**>(&dev), &T, &thr, &cond, &fallbacks};
  cudaKernelNodeParams kp = {};
  kp.func = reinterpret_cast<void*>(fallback_decide_kernel);
  kp.gridDim = dim3(1);
  kp.blockDim = dim3(32);
  kp.kernelParams = args;
  cudaGraphNode_t decide;
  if ((e = cudaGraphAddKernelNode(&decide, graph, nullptr, 0, &kp)) != cudaSuccess) return bad("decide node", e);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = cond;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t ifn;
  if ((e = cudaGraphAddNode(&ifn, graph, &decide, 1, &cp)) != cudaSuccess) return bad("if node", e);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStream_t cs;
  if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess) return bad("stream", e);
  if ((e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)) != cudaSuccess) {
    cudaStreamDestroy(cs);
    return bad("capture", e);
  }
  std::string cerr;
  const int r = chol_inverse(cs, n, G, ldg, sG, X, ldx, sX, batch, scratch, failed, &cerr, nullptr, nullptr, nullptr, oz);
  cudaGraph_t captured = body;
  e = cudaStreamEndCapture(cs, &captured);
  cudaStreamDestroy(cs);
  if (r) {
    if (err) *err = "fallback graph: " + cerr;
    destroy();
    return r;
  }
  if (e != cudaSuccess) return bad("end capture", e);
  if ((e = cudaGraphInstantiate(&exec, graph, 0)) != cudaSuccess) return bad("instantiate", e);
  return 0;
}

int CholFallbackGraph::launch(cudaStream_t st, std::string* err) {
  const cudaError_t e = cudaGraphLaunch(exec, st);
  count_launch();
  if (e != cudaSuccess) {
    if (err) *err = std::string("fallback graph launch: ") + cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

void CholFallbackGraph::destroy() {
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  exec = nullptr;
  graph = nullptr;
}

}  // namespace traj
