// NEXT-4: the paper-literal event-driven projective protocol.
//
// Between events the orbitals evolve with K(tau) = exp(-i H~ tau) for the random waiting time
// tau = -ln(eta)/(gamma N) (reading Q12); K(tau) is applied as a banded circulant stencil
// per lattice axis (Bessel coefficients, tail < 1e-18).  At an event at site j (uniform)
// with Born probability p = |r_j|^2 of the propagated row r_j:
//   occupied (P1 = n_j, Eq. A1):  U <- U - (U w - e_j) w^dag,             w = r_j^dag / |r_j|
//   empty    (P0 = 1 - n_j, A2):   row j zeroed, then the exact rank-1 re-orthonormalisation
//                                  U <- U' (I - u^dag u)^(-1/2), u = r_j
// Both are U <- U + x yhat with yhat = r_j / |r_j| and x = alpha (U yhat^dag) + beta e_j,
// (alpha, beta) = (-1, 1) or (c, -(1 + c) sqrt(p)), c = 1/sqrt(1-p) - 1.  One CTA prepares yhat
// and (alpha, beta); one fused pass per event then propagates each row by the stencil, forms
// v_i = <r_i, yhat> and writes r_i + (alpha v_i + beta delta_ij) yhat: O(L N) per event.
#include <math.h>

#include <algorithm>

#include <stdlib.h>
#include "common.cuh"
#include "pm_events.h"

namespace traj {

namespace {

// taps along an axis: neighbour offsets lo, lo+1, ..., lo+n-1 (mod the extent) with
// coefficients c[0..n): the band [-W, W] (lo = -W, n = 2W+1) or the whole circulant (lo = 0).
struct Taps {
  const cplx* c;
  int lo, n;
};

__device__ __forceinline__ double2 stencil(const cplx* U, long long ld, int Lx, int Ly, int i, int k, Taps tx,
                                           Taps ty) {
  const int x = i % Lx, y = i / Lx;
  double re = 0.0, im = 0.0;
  for (int q = 0; q < ty.n; ++q) {
    const int yy = ((y + ty.lo + q) % Ly + Ly) % Ly;
    const double2 b = ty.c[q];
    double sr = 0.0, si = 0.0;
    for (int r = 0; r < tx.n; ++r) {
      const int xx = ((x + tx.lo + r) % Lx + Lx) % Lx;
      const double2 a = tx.c[r];
      const double2 u = U[(long long)(yy * Lx + xx) * ld + k];
      sr += a.x * u.x - a.y * u.y;
      si += a.x * u.y + a.y * u.x;
    }
    re += b.x * sr - b.y * si;
    im += b.x * si + b.y * sr;
  }
  return make_double2(re, im);
}

__device__ __forceinline__ double block_sum256(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < 8; ++w) s += red[w];
  return s;
}

// coef: [alpha, beta, occupied, p]
__global__ void __launch_bounds__(256) event_prep_kernel(const cplx* U, long long ld, int N, int Lx, int Ly, int j,
                                                         Taps tx, Taps ty, double pc, cplx* yhat, double* coef,
                                                         int32_t* occ_count) {
  __shared__ double red[8];
  __shared__ double scale;
  double p = 0.0;
  for (int k = threadIdx.x; k < N; k += 256) {
    const double2 r = stencil(U, ld, Lx, Ly, j, k, tx, ty);
    yhat[k] = r;
    p += r.x * r.x + r.y * r.y;
  }
  p = block_sum256(p, red);
  if (threadIdx.x == 0) {
    const double pcl = fmin(fmax(p, 0.0), 1.0);
    bool occ = pc <= pcl;                       // occupied iff p_j >= p_c
    if (occ && pcl < 1e-12) occ = false;        // reading Q17
    else if (!occ && 1.0 - pcl < 1e-12) occ = true;
    double alpha = 0.0, beta = 0.0, s = 0.0;
    if (p > 1e-300) {
      s = 1.0 / sqrt(p);
      if (occ) {
        alpha = -1.0;
        beta = 1.0;
      } else {
        const double c = 1.0 / sqrt(fmax(1.0 - p, 1e-300)) - 1.0;
        alpha = c;
        beta = -(1.0 + c) * sqrt(p);
      }
    }
    coef[0] = alpha;
    coef[1] = beta;
    coef[2] = occ ? 1.0 : 0.0;
    coef[3] = p;
    if (occ) ++*occ_count;
    scale = s;
  }
  __syncthreads();
  const double s = scale;
  for (int k = threadIdx.x; k < N; k += 256) {
    const double2 r = yhat[k];
    yhat[k] = make_double2(r.x * s, r.y * s);
  }
}

// one CTA per row: out_i = r_i + (alpha <r_i, yhat> + beta delta_ij) yhat  (coef == nullptr: r_i).
// The tap rows of row i and their product coefficients are resolved once per CTA in shared
// memory; the second pass re-reads the freshly written row (L1/L2).
constexpr int MAXTAPS = 128;

__global__ void __launch_bounds__(256) event_update_kernel(const cplx* U, cplx* out, long long ld, int N, int Lx,
                                                           int Ly, Taps tx, Taps ty, const cplx* yhat,
                                                           const double* coef, int j) {
  __shared__ double red[8];
  __shared__ long long trow[MAXTAPS];
  __shared__ double2 tcoef[MAXTAPS];
  const int i = blockIdx.x;
  const int nt = tx.n * ty.n;
  cplx* o = out + (long long)i * ld;
  const bool fast = nt <= MAXTAPS;
  if (fast) {
    const int x = i % Lx, y = i / Lx;
    for (int q = threadIdx.x; q < nt; q += 256) {
      const int qy = q / tx.n, qx = q % tx.n;
      const int yy = ((y + ty.lo + qy) % Ly + Ly) % Ly, xx = ((x + tx.lo + qx) % Lx + Lx) % Lx;
      trow[q] = (long long)(yy * Lx + xx) * ld;
      const double2 a = tx.c[qx], b = ty.c[qy];
      tcoef[q] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
    }
    __syncthreads();
    double vr = 0.0, vi = 0.0;
    for (int k = threadIdx.x; k < N; k += 256) {
      double re = 0.0, im = 0.0;
      for (int q = 0; q < nt; ++q) {
        const double2 c = tcoef[q];
        const double2 u = U[trow[q] + k];
        re += c.x * u.x - c.y * u.y;
        im += c.x * u.y + c.y * u.x;
      }
      o[k] = make_double2(re, im);
      if (coef) {
        const double2 yk = yhat[k];
        vr += re * yk.x + im * yk.y;
        vi += im * yk.x - re * yk.y;
      }
    }
    if (!coef) return;
    vr = block_sum256(vr, red);
    vi = block_sum256(vi, red);
    const double xr = coef[0] * vr + (i == j ? coef[1] : 0.0), xi = coef[0] * vi;
    for (int k = threadIdx.x; k < N; k += 256) {
      const double2 yk = yhat[k];
      double2 r = o[k];
      r.x += xr * yk.x - xi * yk.y;
      r.y += xr * yk.y + xi * yk.x;
      o[k] = r;
    }
    return;
  }
  double vr = 0.0, vi = 0.0;
  for (int k = threadIdx.x; k < N; k += 256) {
    const double2 r = stencil(U, ld, Lx, Ly, i, k, tx, ty);
    o[k] = r;
    if (coef) {
      const double2 y = yhat[k];                 // v = sum_k r_k conj(y_k)
      vr += r.x * y.x + r.y * y.y;
      vi += r.y * y.x - r.x * y.y;
    }
  }
  if (!coef) return;
  vr = block_sum256(vr, red);
  vi = block_sum256(vi, red);
  const double alpha = coef[0], beta = coef[1];
  const double xr = alpha * vr + (i == j ? beta : 0.0), xi = alpha * vi;
  for (int k = threadIdx.x; k < N; k += 256) {
    const double2 y = yhat[k];
    double2 r = o[k];
    r.x += xr * y.x - xi * y.y;
    r.y += xr * y.y + xi * y.x;
    o[k] = r;
  }
}

}  // namespace

int event_prep(cudaStream_t st, const cplx* U, long long ld, int N, int Lx, int Ly, int j, const cplx* cx, int xlo,
               int xn, const cplx* cy, int ylo, int yn, double pc, cplx* yhat, double* coef, int32_t* occ_count,
               std::string* err) {
  event_prep_kernel<<<1, 256, 0, st>>>(U, ld, N, Lx, Ly, j, Taps{cx, xlo, xn}, Taps{cy, ylo, yn}, pc, yhat, coef,
                                       occ_count);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("event_prep: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

int event_update(cudaStream_t st, const cplx* U, cplx* out, long long ld, int N, int Lx, int Ly, const cplx* cx,
                 int xlo, int xn, const cplx* cy, int ylo, int yn, const cplx* yhat, const double* coef, int j,
                 std::string* err) {
  event_update_kernel<<<Lx * Ly, 256, 0, st>>>(U, out, ld, N, Lx, Ly, Taps{cx, xlo, xn}, Taps{cy, ylo, yn}, yhat,
                                               coef, j);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("event_update: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}



// ---------------------------------------------------------------------------------------------
// One-pass event updates.  With g = U yhat^dag (an L-vector) the rank-1 coefficient of every row
// is known before the pass: <r_i, yhat> = (K(tau) g)_i, r = K(tau) U.  The pass for event q then
// reads U once, writes r_i + (alpha (K g)_i + beta delta_ij) yhat once, and accumulates
// g' = out yhat'^dag for the NEXT event q+1, whose yhat' (row j' of K(tau') out) was prepared
// before the pass: the K(tau) commute, so row j' of K(tau') out = row j' of K(tau + tau') U plus
// (K(tau') x)_j' yhat with x_m = alpha (K(tau) g)_m + beta delta_mj -- one row stencil and a
// scalar.  yhat is kept unnormalised (r) with its scale s = 1/|r| in coef[4].
namespace {

struct DevTaps {
  const cplx* c;
  int lo, n;
};

__device__ __forceinline__ int nb_site(int m, int Lx, int Ly, int ox, int oy) {
  const int x = m % Lx, y = m / Lx;
  int xx = x + ox, yy = y + oy;
  xx %= Lx;
  if (xx < 0) xx += Lx;
  yy %= Ly;
  if (yy < 0) yy += Ly;
  return yy * Lx + xx;
}

// (K g)_m for the product taps (tx, ty), g an L-vector
__device__ __forceinline__ double2 stencil_vec(const double2* g, int Lx, int Ly, int m, DevTaps tx, DevTaps ty) {
  double re = 0.0, im = 0.0;
  for (int qy = 0; qy < ty.n; ++qy)
    for (int qx = 0; qx < tx.n; ++qx) {
      const double2 a = tx.c[qx], b = ty.c[qy];
      const double cr = a.x * b.x - a.y * b.y, ci = a.x * b.y + a.y * b.x;
      const double2 v = g[nb_site(m, Lx, Ly, tx.lo + qx, ty.lo + qy)];
      re += cr * v.x - ci * v.y;
      im += cr * v.y + ci * v.x;
    }
  return make_double2(re, im);
}

// r_k = (K(tau + tau') U)_{j', k} + X yprev_k sprev,  X = (K(tau') x)_{j'} with x_m = alpha (K(tau) g)_m + beta delta_{m,jprev}
// (prev event), i.e. X = alpha (K(tau + tau') g)_{j'} + beta K(tau')_{j', jprev}: the combined taps c on g and the
// one entry of the own taps o that reaches jprev (K(tau') K(tau) = K(tau + tau')), summed over the block's threads.
// part[b] = sum over this block's k of |r_k|^2.  Without a previous event: r = (K(tau') U)_{j'}.
constexpr int EVP_THREADS = 256;
__global__ void __launch_bounds__(EVP_THREADS) ev_prep_kernel(const cplx* U, long long ld, int N, int Lx, int Ly, int j,
                                                             DevTaps cx, DevTaps cy, DevTaps ox, DevTaps oy,
                                                             const double* coef_prev, const double2* g_prev,
                                                             const cplx* y_prev, int j_prev, cplx* y_out,
                                                             double* part) {
  __shared__ double red[EVP_THREADS / 32];
  __shared__ double redx[2][EVP_THREADS / 32];
  __shared__ double2 Xs;
  if (coef_prev) {
    const double alpha = coef_prev[0], beta = coef_prev[1];
    double xr = 0.0, xi = 0.0;
    for (int q = threadIdx.x; q < cx.n * cy.n; q += EVP_THREADS) {
      const int qy = q / cx.n, qx = q % cx.n;
      const double2 a = cx.c[qx], b = cy.c[qy];
      const double cr = a.x * b.x - a.y * b.y, ci = a.x * b.y + a.y * b.x;
      const double2 v = g_prev[nb_site(j, Lx, Ly, cx.lo + qx, cy.lo + qy)];
      xr += alpha * (cr * v.x - ci * v.y);
      xi += alpha * (cr * v.y + ci * v.x);
    }
    for (int q = threadIdx.x; q < ox.n * oy.n; q += EVP_THREADS) {
      const int qy = q / ox.n, qx = q % ox.n;
      if (nb_site(j, Lx, Ly, ox.lo + qx, oy.lo + qy) != j_prev) continue;
      const double2 a = ox.c[qx], b = oy.c[qy];
      xr += beta * (a.x * b.x - a.y * b.y);
      xi += beta * (a.x * b.y + a.y * b.x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      xr += __shfl_xor_sync(0xffffffffu, xr, o);
      xi += __shfl_xor_sync(0xffffffffu, xi, o);
    }
    if ((threadIdx.x & 31) == 0) {
      redx[0][threadIdx.x >> 5] = xr;
      redx[1][threadIdx.x >> 5] = xi;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 X = make_double2(0.0, 0.0);
    if (coef_prev) {
      for (int w = 0; w < EVP_THREADS / 32; ++w) {
        X.x += redx[0][w];
        X.y += redx[1][w];
      }
      X.x *= coef_prev[4];
      X.y *= coef_prev[4];
    }
    Xs = X;
  }
  __syncthreads();
  const double2 X = Xs;
  double p = 0.0;
  for (int k = blockIdx.x * EVP_THREADS + threadIdx.x; k < N; k += gridDim.x * EVP_THREADS) {
    double2 r = stencil(U, ld, Lx, Ly, j, k, Taps{cx.c, cx.lo, cx.n}, Taps{cy.c, cy.lo, cy.n});
    if (coef_prev) {
      const double2 y = y_prev[k];
      r.x += X.x * y.x - X.y * y.y;
      r.y += X.x * y.y + X.y * y.x;
    }
    y_out[k] = r;
    p += r.x * r.x + r.y * r.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = p;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < EVP_THREADS / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

// coef = [alpha, beta, occ, p, s]: the Born decision of P:174 on p = |r_j|^2 (readings Q13, Q17)
__global__ void ev_decide_kernel(const double* part, int nparts, double pc, double* coef, int32_t* occ_count) {
  if (threadIdx.x != 0) return;
  double p = 0.0;
  for (int b = 0; b < nparts; ++b) p += part[b];
  const double pcl = fmin(fmax(p, 0.0), 1.0);
  bool occ = pc <= pcl;
  if (occ && pcl < 1e-12) occ = false;
  else if (!occ && 1.0 - pcl < 1e-12) occ = true;
  double alpha = 0.0, beta = 0.0, s = 0.0;
  if (p > 1e-300) {
    s = 1.0 / sqrt(p);
    if (occ) {
      alpha = -1.0;
      beta = 1.0;
    } else {
      const double c = 1.0 / sqrt(fmax(1.0 - p, 1e-300)) - 1.0;
      alpha = c;
      beta = -(1.0 + c) * sqrt(p);
    }
  }
  coef[0] = alpha;
  coef[1] = beta;
  coef[2] = occ ? 1.0 : 0.0;
  coef[3] = p;
  coef[4] = s;
  if (occ) ++*occ_count;
}

// g_i = s sum_k U_ik conj(y_k): one warp per row
__global__ void __launch_bounds__(256) ev_gemv_kernel(const cplx* U, long long ld, int N, int L, const cplx* y,
                                                      const double* coef, double2* g) {
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= L) return;
  const cplx* u = U + (long long)i * ld;
  double re = 0.0, im = 0.0;
#pragma unroll 4
  for (int k = lane; k < N; k += 32) {
    const double2 a = u[k], b = y[k];
    re += a.x * b.x + a.y * b.y;
    im += a.y * b.x - a.x * b.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if (lane == 0) {
    const double s = coef[4];
    g[i] = make_double2(s * re, s * im);
  }
}

// taps by value for the 1d row-blocked pass: (re, im, -im) so no negation is formed per thread
template <int W>
struct EvTaps {
  double c[2 * W + 1][3];
};

// 1d ring: EV_R (8 for W <= 6, else 4: registers) consecutive rows per CTA, each input row loaded once per column into a register
// window.  out_i = sum_d c_d U_{i+d} + x_i yhat (x_i from g), gn_i = <out_i, yhat_next>.
// ALT: the taps of K(tau) on the bipartite ring alternate real / imaginary, c_d = (-i)^|d| J_|d|(2 J tau)
// (axis_taps builds them in exactly that form), so each tap is two FMAs instead of four.
template <int W, int EV_R, bool ALT>
__global__ void __launch_bounds__(256) ev_pass_1d_kernel(const cplx* __restrict__ U, cplx* __restrict__ out,
                                                         long long ld, int N, int L,
                                                         const __grid_constant__ EvTaps<W> taps,
                                                         const cplx* __restrict__ y, const double* __restrict__ coef,
                                                         const double2* __restrict__ g, int j,
                                                         const cplx* __restrict__ yn, const double* __restrict__ coefn,
                                                         double2* __restrict__ gn, int bstride, int pstride) {
  // ring blockIdx.y of a 2d lattice's axis: its site p is row blockIdx.y * bstride + p * pstride of U, g, gn
  // (x axis: bstride = Lx, pstride = 1; y axis: 1, Lx; the 1d ring: 0, 1)
  U += (long long)blockIdx.y * bstride * ld;
  out += (long long)blockIdx.y * bstride * ld;
  g += (long long)blockIdx.y * bstride;
  gn += (long long)blockIdx.y * bstride;
  j -= blockIdx.y * bstride;
  const long long ldp = ld * pstride;
  __shared__ double2 xs[EV_R];
  __shared__ double red[8][2 * EV_R];
  const int i0 = blockIdx.x * EV_R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < EV_R) {
    double2 x = make_double2(0.0, 0.0);
    const int i = i0 + threadIdx.x;
    if (coef && i < L) {
      double vr = 0.0, vi = 0.0;
      for (int d = 0; d < 2 * W + 1; ++d) {
        int p = i - W + d;
        p = p < 0 ? p + L : (p >= L ? p - L : p);
        const double2 v = g[(long long)p * pstride];
        vr += taps.c[d][0] * v.x - taps.c[d][1] * v.y;
        vi += taps.c[d][0] * v.y + taps.c[d][1] * v.x;
      }
      const double s = coef[4];
      x = make_double2(s * (coef[0] * vr + (i * pstride == j ? coef[1] : 0.0)), s * coef[0] * vi);
    }
    xs[threadIdx.x] = x;
  }
  __syncthreads();
  double2 x[EV_R];
#pragma unroll
  for (int r = 0; r < EV_R; ++r) x[r] = xs[r];
  const double sn = coefn ? coefn[4] : 0.0;
  double ar[EV_R], ai[EV_R];
#pragma unroll
  for (int r = 0; r < EV_R; ++r) ar[r] = ai[r] = 0.0;
  const bool wraps = i0 - W < 0 || i0 + EV_R + W > L;
#pragma unroll 1
  for (int k = threadIdx.x; k < N; k += 256) {
    double2 in[EV_R + 2 * W];
#pragma unroll
    for (int q = 0; q < EV_R + 2 * W; ++q) {
      int p = i0 - W + q;
      if (wraps) p = p < 0 ? p + L : (p >= L ? p - L : p);
      in[q] = U[p * ldp + k];
    }
    const double2 yk = coef ? y[k] : make_double2(0.0, 0.0);
    const double2 ynk = yn ? yn[k] : make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < EV_R; ++r) {
      double re = x[r].x * yk.x - x[r].y * yk.y, im = x[r].x * yk.y + x[r].y * yk.x;
#pragma unroll
      for (int d = 0; d < 2 * W + 1; ++d) {
        const double2 b = in[r + d];
        if (!ALT) {
          re = fma(taps.c[d][0], b.x, re);
          re = fma(taps.c[d][2], b.y, re);
          im = fma(taps.c[d][0], b.y, im);
          im = fma(taps.c[d][1], b.x, im);
        } else if (((d - W) & 1) == 0) {   // real tap
          re = fma(taps.c[d][0], b.x, re);
          im = fma(taps.c[d][0], b.y, im);
        } else {                           // imaginary tap i s: (re, im) += (-s b.y, s b.x)
          re = fma(taps.c[d][2], b.y, re);
          im = fma(taps.c[d][1], b.x, im);
        }
      }
      if (i0 + r < L) out[(i0 + r) * ldp + k] = make_double2(re, im);
      ar[r] += re * ynk.x + im * ynk.y;
      ai[r] += im * ynk.x - re * ynk.y;
    }
  }
  if (!yn) return;
#pragma unroll
  for (int r = 0; r < EV_R; ++r) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ar[r] += __shfl_xor_sync(0xffffffffu, ar[r], o);
      ai[r] += __shfl_xor_sync(0xffffffffu, ai[r], o);
    }
    if (lane == 0) {
      red[warp][2 * r] = ar[r];
      red[warp][2 * r + 1] = ai[r];
    }
  }
  __syncthreads();
  if (threadIdx.x < EV_R && i0 + threadIdx.x < L) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 8; ++w) {
      a += red[w][2 * threadIdx.x];
      b += red[w][2 * threadIdx.x + 1];
    }
    gn[(long long)(i0 + threadIdx.x) * pstride] = make_double2(sn * a, sn * b);
  }
}

// any lattice / any taps: one CTA per row with the resolved tap table in shared memory
constexpr int EVG_MAXTAPS = 1024;
__global__ void __launch_bounds__(256) ev_pass_generic_kernel(const cplx* __restrict__ U, cplx* __restrict__ out,
                                                              long long ld, int N, int Lx, int Ly, DevTaps tx,
                                                              DevTaps ty, const cplx* __restrict__ y,
                                                              const double* __restrict__ coef,
                                                              const double2* __restrict__ g, int j,
                                                              const cplx* __restrict__ yn,
                                                              const double* __restrict__ coefn,
                                                              double2* __restrict__ gn) {
  __shared__ int trow[EVG_MAXTAPS];
  __shared__ double2 tcoef[EVG_MAXTAPS];
  __shared__ double red[16];
  __shared__ double2 xs;
  const int i = blockIdx.x;
  const int nt = tx.n * ty.n;
  for (int q = threadIdx.x; q < nt; q += 256) {
    const int qy = q / tx.n, qx = q % tx.n;
    trow[q] = nb_site(i, Lx, Ly, tx.lo + qx, ty.lo + qy);
    const double2 a = tx.c[qx], b = ty.c[qy];
    tcoef[q] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 x = make_double2(0.0, 0.0);
    if (coef) {
      double vr = 0.0, vi = 0.0;
      for (int q = 0; q < nt; ++q) {
        const double2 c = tcoef[q], v = g[trow[q]];
        vr += c.x * v.x - c.y * v.y;
        vi += c.x * v.y + c.y * v.x;
      }
      const double s = coef[4];
      x = make_double2(s * (coef[0] * vr + (i == j ? coef[1] : 0.0)), s * coef[0] * vi);
    }
    xs = x;
  }
  __syncthreads();
  const double2 x = xs;
  const double sn = coefn ? coefn[4] : 0.0;
  double ar = 0.0, ai = 0.0;
  cplx* o = out + (long long)i * ld;
  for (int k = threadIdx.x; k < N; k += 256) {
    const double2 yk = coef ? y[k] : make_double2(0.0, 0.0);
    double re = x.x * yk.x - x.y * yk.y, im = x.x * yk.y + x.y * yk.x;
    for (int q = 0; q < nt; ++q) {
      const double2 c = tcoef[q];
      const double2 u = U[(long long)trow[q] * ld + k];
      re += c.x * u.x - c.y * u.y;
      im += c.x * u.y + c.y * u.x;
    }
    o[k] = make_double2(re, im);
    if (yn) {
      const double2 b = yn[k];
      ar += re * b.x + im * b.y;
      ai += im * b.x - re * b.y;
    }
  }
  if (!yn) return;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    ar += __shfl_xor_sync(0xffffffffu, ar, off);
    ai += __shfl_xor_sync(0xffffffffu, ai, off);
  }
  if ((threadIdx.x & 31) == 0) {
    red[2 * (threadIdx.x >> 5)] = ar;
    red[2 * (threadIdx.x >> 5) + 1] = ai;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 8; ++w) {
      a += red[2 * w];
      b += red[2 * w + 1];
    }
    gn[i] = make_double2(sn * a, sn * b);
  }
}

// Separable 2d pass: K(tau) = K_x(tau) (x) K_y(tau) on the square lattice, so the (2w+1)^2 product taps of a row
// become 2 (2w+1): tmp = (K_x (x) 1) U, then out = (1 (x) K_y) tmp + x yhat with x from g_x = (K_x (x) 1) g.
// Two reads and two writes of U instead of one each, against (2w+1)/2 times fewer row reads through L2.
__device__ cplx ev_unit_tap = {1.0, 0.0};

__global__ void __launch_bounds__(256) ev_vec_axis_kernel(const double2* __restrict__ g, double2* __restrict__ gx,
                                                          int Lx, int Ly, DevTaps tx) {
  const int m = blockIdx.x * 256 + threadIdx.x;
  if (m >= Lx * Ly) return;
  double re = 0.0, im = 0.0;
  for (int q = 0; q < tx.n; ++q) {
    const double2 c = tx.c[q], v = g[nb_site(m, Lx, Ly, tx.lo + q, 0)];
    re += c.x * v.x - c.y * v.y;
    im += c.x * v.y + c.y * v.x;
  }
  gx[m] = make_double2(re, im);
}

// TRAJ_EV_SEPARABLE=0: the 2d pass with the product taps in one kernel
bool ev_separable() {
  const char* e = getenv("TRAJ_EV_SEPARABLE");
  return !(e && e[0] == '0');
}

// TRAJ_EV_ALT_TAPS=0: always the general four-FMA taps
bool ev_alt_taps() {
  const char* e = getenv("TRAJ_EV_ALT_TAPS");
  return !(e && e[0] == '0');
}

template <int W>
cudaError_t launch_pass_1d(cudaStream_t st, const cplx* U, cplx* out, long long ld, int N, int L,
                           const cplx* taps_host, int w, const cplx* y, const double* coef, const double2* g, int j,
                           const cplx* yn, const double* coefn, double2* gn, int rings = 1, int bstride = 0,
                           int pstride = 1) {
  constexpr int R = W <= 6 ? 8 : 4;
  EvTaps<W> t;
  for (int d = 0; d < 2 * W + 1; ++d) t.c[d][0] = t.c[d][1] = t.c[d][2] = 0.0;
  bool alt = true;   // even offsets purely real, odd offsets purely imaginary (exactly)
  for (int d = 0; d < 2 * w + 1; ++d) {
    t.c[W - w + d][0] = taps_host[d].x;
    t.c[W - w + d][1] = taps_host[d].y;
    t.c[W - w + d][2] = -taps_host[d].y;
    alt = alt && (((d - w) & 1) == 0 ? taps_host[d].y == 0.0 : taps_host[d].x == 0.0);
  }
  const dim3 grid((unsigned)ceil_div(L, R), (unsigned)rings);
  if (alt && ev_alt_taps())
    ev_pass_1d_kernel<W, R, true><<<grid, 256, 0, st>>>(U, out, ld, N, L, t, y, coef, g, j, yn, coefn, gn, bstride,
                                                        pstride);
  else
    ev_pass_1d_kernel<W, R, false><<<grid, 256, 0, st>>>(U, out, ld, N, L, t, y, coef, g, j, yn, coefn, gn, bstride,
                                                         pstride);
  return cudaGetLastError();
}

}  // namespace

int ev_prep(cudaStream_t st, const cplx* U, long long ld, int N, int Lx, int Ly, int j, const cplx* cxc, int cxlo,
            int cxn, const cplx* cyc, int cylo, int cyn, const cplx* oxc, int oxlo, int oxn, const cplx* oyc, int oylo,
            int oyn, const double* coef_prev, const double2* g_prev, const cplx* y_prev, int j_prev, double pc,
            cplx* y_out, double* part, double* coef_out, int32_t* occ_count, std::string* err) {
  const int nb = (int)std::min<long long>(ceil_div(N, EVP_THREADS), 64);
  ev_prep_kernel<<<nb, EVP_THREADS, 0, st>>>(U, ld, N, Lx, Ly, j, DevTaps{cxc, cxlo, cxn}, DevTaps{cyc, cylo, cyn},
                                             DevTaps{oxc, oxlo, oxn}, DevTaps{oyc, oylo, oyn}, coef_prev, g_prev,
                                             y_prev, j_prev, y_out, part);
  ev_decide_kernel<<<1, 32, 0, st>>>(part, nb, pc, coef_out, occ_count);
  count_launch(2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("ev_prep: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

int ev_gemv(cudaStream_t st, const cplx* U, long long ld, int N, int L, const cplx* y, const double* coef, double2* g,
            std::string* err) {
  ev_gemv_kernel<<<(unsigned)ceil_div(L, 8), 256, 0, st>>>(U, ld, N, L, y, coef, g);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("ev_gemv: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

namespace {
// one axis of the pass on the row-blocked kernel (the band [-w, w], w <= 9, on rings of extent >= 2w + 17)
bool ring_ok(int lo, int n, int extent) { return lo == -(n - 1) / 2 && (n - 1) / 2 <= 9 && n + 16 <= extent; }

cudaError_t launch_ring(cudaStream_t st, const cplx* U, cplx* out, long long ld, int N, int L, const cplx* taps_host,
                        int w, const cplx* y, const double* coef, const double2* g, int j, const cplx* yn,
                        const double* coefn, double2* gn, int rings, int bstride, int pstride) {
  if (w <= 2) return launch_pass_1d<2>(st, U, out, ld, N, L, taps_host, w, y, coef, g, j, yn, coefn, gn, rings, bstride, pstride);
  if (w <= 4) return launch_pass_1d<4>(st, U, out, ld, N, L, taps_host, w, y, coef, g, j, yn, coefn, gn, rings, bstride, pstride);
  if (w <= 6) return launch_pass_1d<6>(st, U, out, ld, N, L, taps_host, w, y, coef, g, j, yn, coefn, gn, rings, bstride, pstride);
  return launch_pass_1d<9>(st, U, out, ld, N, L, taps_host, w, y, coef, g, j, yn, coefn, gn, rings, bstride, pstride);
}
}  // namespace

int ev_pass(cudaStream_t st, const cplx* U, cplx* out, long long ld, int N, int Lx, int Ly, const cplx* cx_dev,
            const cplx* cx_host, int xlo, int xn, const cplx* cy_dev, const cplx* cy_host, int ylo, int yn_taps,
            const cplx* y, const double* coef, const double2* g, int j, const cplx* yn, const double* coefn,
            double2* gn, cplx* tmp, double2* gx, std::string* err) {
  const int w = (xn - 1) / 2;
  cudaError_t e;
  if (Ly == 1 && cx_host && ring_ok(xlo, xn, Lx)) {
    e = launch_ring(st, U, out, ld, N, Lx, cx_host, w, y, coef, g, j, yn, coefn, gn, 1, 0, 1);
  } else if (Ly > 1 && xn > 1 && yn_taps > 1 && tmp && gx && xn <= EVG_MAXTAPS && yn_taps <= EVG_MAXTAPS &&
             ev_separable()) {
    const cplx* one = nullptr;
    e = cudaGetSymbolAddress((void**)&one, ev_unit_tap);
    if (e == cudaSuccess) {
      const DevTaps tx{cx_dev, xlo, xn}, ty{cy_dev, ylo, yn_taps}, id{one, 0, 1};
      // x axis: tmp = (K_x (x) 1) U on the Ly lattice lines (consecutive rows), g_x = (K_x (x) 1) g
      if (cx_host && ring_ok(xlo, xn, Lx))
        e = launch_ring(st, U, tmp, ld, N, Lx, cx_host, w, nullptr, nullptr, g, -1, nullptr, nullptr, gn, Ly, Lx, 1);
      else
        ev_pass_generic_kernel<<<Lx * Ly, 256, 0, st>>>(U, tmp, ld, N, Lx, Ly, tx, id, nullptr, nullptr, nullptr, -1,
                                                        nullptr, nullptr, nullptr);
      if (coef) ev_vec_axis_kernel<<<(unsigned)ceil_div(Lx * Ly, 256), 256, 0, st>>>(g, gx, Lx, Ly, tx);
      // y axis: out = (1 (x) K_y) tmp + x yhat on the Lx lattice columns (rows Lx apart), and the next event's g
      if (e == cudaSuccess && cy_host && ring_ok(ylo, yn_taps, Ly))
        e = launch_ring(st, tmp, out, ld, N, Ly, cy_host, (yn_taps - 1) / 2, y, coef, coef ? gx : g, j, yn, coefn, gn,
                        Lx, 1, Lx);
      else if (e == cudaSuccess)
        ev_pass_generic_kernel<<<Lx * Ly, 256, 0, st>>>(tmp, out, ld, N, Lx, Ly, id, ty, y, coef, coef ? gx : g, j, yn,
                                                        coefn, gn);
      count_launch(coef ? 2 : 1);
      if (e == cudaSuccess) e = cudaGetLastError();
    }
  } else {
    if (xn * yn_taps > EVG_MAXTAPS) {
      if (err) *err = "ev_pass: more than 1024 taps";
      return 1;
    }
    ev_pass_generic_kernel<<<Lx * Ly, 256, 0, st>>>(U, out, ld, N, Lx, Ly, DevTaps{cx_dev, xlo, xn},
                                                    DevTaps{cy_dev, ylo, yn_taps}, y, coef, g, j, yn, coefn, gn);
    e = cudaGetLastError();
  }
  count_launch();
  if (e != cudaSuccess && err) *err = std::string("ev_pass: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

}  // namespace traj
