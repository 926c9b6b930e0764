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

}  // namespace traj
