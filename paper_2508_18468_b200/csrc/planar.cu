// Planar 3M form of the dense propagator U <- K U (row a1; the north star's dense complex-FP64
// contraction).  With K = Kr + i Ki and U = Ur + i Ui:
//   P1 = Kr Ur,  P2 = Ki Ui,  P3 = (Kr + Ki)(Ur + Ui),   K U = (P1 - P2) + i (P3 - P1 - P2)
// -- the Gauss/3M identity of csrc/zgemm.cu's interleaved kernels, here as three independent real
// GEMMs on whole planes (dgemm.cu: one accumulator set per warp, 96% of the DMMA pipe).  K's planes
// (Kr, Ki, Kr + Ki) are built once; U is split into (Ur, Ui, Ur + Ui) before and the products are
// recombined after: two HBM passes, 40 L N bytes each way per trajectory.
#include "common.cuh"
#include "planar.h"

namespace traj {

namespace {

__device__ __forceinline__ double2 cmul2(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// K[i][j] = kx[(jx - ix) mod Lx] ky[(jy - iy) mod Ly]; planes (re, im, re + im)
__global__ void build_k_planar_kernel(double* Kp, long long ld, long long ps, int Lx, int Ly, const cplx* kx,
                                      const cplx* ky, long long row0, long long nrows) {
  const long long L = (long long)Lx * Ly;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < nrows * L;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long r = idx / L, j = idx % L, i = row0 + r;
    const int ix = (int)(i % Lx), iy = (int)(i / Lx), jx = (int)(j % Lx), jy = (int)(j / Lx);
    const int dx = ((jx - ix) % Lx + Lx) % Lx, dy = ((jy - iy) % Ly + Ly) % Ly;
    const double2 v = cmul2(kx[dx], ky[dy]);
    const long long o = r * ld + j;
    Kp[o] = v.x;
    Kp[ps + o] = v.y;
    Kp[2 * ps + o] = v.x + v.y;
  }
}

// planes[t][0..2][row][col] = (re, im, re + im) of U[t][row][col]; two columns per thread
__global__ void split_kernel(const cplx* __restrict__ U, long long ldu, long long sU, int L, int N,
                             double* __restrict__ Pl, long long ldp, long long ps, long long ts) {
  const int t = blockIdx.z;
  const int row = blockIdx.y;
  const cplx* u = U + t * sU + (long long)row * ldu;
  double* p = Pl + t * ts + (long long)row * ldp;
  for (int c = 2 * (blockIdx.x * blockDim.x + threadIdx.x); c < N; c += 2 * gridDim.x * blockDim.x) {
    const double2 a = u[c];
    const double2 b = c + 1 < N ? u[c + 1] : make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(p + c) = make_double2(a.x, b.x);
    *reinterpret_cast<double2*>(p + ps + c) = make_double2(a.y, b.y);
    *reinterpret_cast<double2*>(p + 2 * ps + c) = make_double2(a.x + a.y, b.x + b.y);
  }
}

// U[t][row][col] = (P1 - P2) + i (P3 - P1 - P2)
__global__ void combine_kernel(const double* __restrict__ Pl, long long ldp, long long ps, long long ts, int L, int N,
                               cplx* __restrict__ U, long long ldu, long long sU) {
  const int t = blockIdx.z;
  const int row = blockIdx.y;
  const double* p = Pl + t * ts + (long long)row * ldp;
  cplx* u = U + t * sU + (long long)row * ldu;
  for (int c = 2 * (blockIdx.x * blockDim.x + threadIdx.x); c < N; c += 2 * gridDim.x * blockDim.x) {
    const double2 p1 = *reinterpret_cast<const double2*>(p + c);
    const double2 p2 = *reinterpret_cast<const double2*>(p + ps + c);
    const double2 p3 = *reinterpret_cast<const double2*>(p + 2 * ps + c);
    u[c] = make_double2(p1.x - p2.x, p3.x - p1.x - p2.x);
    if (c + 1 < N) u[c + 1] = make_double2(p1.y - p2.y, p3.y - p1.y - p2.y);
  }
}

// planes (re, im, re - im, re, im, re + im) of U: the Gram's A operands (Ur, Ui, Ur - Ui; U^dag =
// Ur^T - i Ui^T) followed by its B operands (Ur, Ui, Ur + Ui), each triple a constant-stride batch
__global__ void split6_kernel(const cplx* __restrict__ U, long long ldu, long long sU, int L, int N,
                              double* __restrict__ Pl, long long ldp, long long ps, long long ts) {
  const int t = blockIdx.z;
  const int row = blockIdx.y;
  const cplx* u = U + t * sU + (long long)row * ldu;
  double* p = Pl + t * ts + (long long)row * ldp;
  for (int c = 2 * (blockIdx.x * blockDim.x + threadIdx.x); c < N; c += 2 * gridDim.x * blockDim.x) {
    const double2 a = u[c];
    const double2 b = c + 1 < N ? u[c + 1] : make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(p + c) = make_double2(a.x, b.x);
    *reinterpret_cast<double2*>(p + ps + c) = make_double2(a.y, b.y);
    *reinterpret_cast<double2*>(p + 2 * ps + c) = make_double2(a.x - a.y, b.x - b.y);
    *reinterpret_cast<double2*>(p + 3 * ps + c) = make_double2(a.x, b.x);
    *reinterpret_cast<double2*>(p + 4 * ps + c) = make_double2(a.y, b.y);
    *reinterpret_cast<double2*>(p + 5 * ps + c) = make_double2(a.x + a.y, b.x + b.y);
  }
}

// G = U^dag U from P1 = Ur^T Ur, Q2 = Ui^T Ui, P3 = (Ur - Ui)^T (Ur + Ui): Re = P1 + Q2,
// Im = P3 - P1 + Q2; upper triangle only
__global__ void combine_gram_kernel(const double* __restrict__ Pl, long long ldp, long long ps, long long ts, int n,
                                    cplx* __restrict__ G, long long ldg, long long sG) {
  const int t = blockIdx.z;
  const int row = blockIdx.y;
  const double* p = Pl + t * ts + (long long)row * ldp;
  cplx* g = G + t * sG + (long long)row * ldg;
  for (int c = row + blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const double p1 = p[c], q2 = p[ps + c], p3 = p[2 * ps + c];
    g[c] = make_double2(p1 + q2, p3 - p1 + q2);
  }
}

// buf[row][c - c0] (ld w) = the Gram entry (row, c) combined from the planes for row < c1, c in [c0, c1)
// with row <= c; zeros below the diagonal
__global__ void pack_gram_panel_kernel(const double* __restrict__ Pl, long long ldp, long long ps, int c0, int c1,
                                       cplx* __restrict__ buf, int w) {
  const int row = blockIdx.y;
  for (int c = c0 + blockIdx.x * blockDim.x + threadIdx.x; c < c1; c += gridDim.x * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (row <= c) {
      const double* p = Pl + (long long)row * ldp;
      const double p1 = p[c], q2 = p[ps + c], p3 = p[2 * ps + c];
      v = make_double2(p1 + q2, p3 - p1 + q2);
    }
    buf[(long long)row * w + (c - c0)] = v;
  }
}

}  // namespace

int pack_gram_panel(cudaStream_t st, const double* Pl, long long ldp, long long ps, int c0, int c1, cplx* buf, int w,
                    std::string* err) {
  if (c1 <= c0) return 0;
  dim3 grid((unsigned)ceil_div(c1 - c0, 256), c1);
  pack_gram_panel_kernel<<<grid, 256, 0, st>>>(Pl, ldp, ps, c0, c1, buf, w);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("pack_gram_panel: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

int split6_planes(cudaStream_t st, const cplx* U, long long ldu, long long sU, int L, int N, int T, double* Pl,
                  long long ldp, long long ps, long long ts, std::string* err) {
  dim3 grid((unsigned)std::min<long long>(ceil_div(N, 512), 16), L, T);
  split6_kernel<<<grid, 256, 0, st>>>(U, ldu, sU, L, N, Pl, ldp, ps, ts);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("split6_planes: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

int combine_gram(cudaStream_t st, const double* Pl, long long ldp, long long ps, long long ts, int n, int T, cplx* G,
                 long long ldg, long long sG, std::string* err) {
  dim3 grid((unsigned)std::min<long long>(ceil_div(n, 256), 32), n, T);
  combine_gram_kernel<<<grid, 256, 0, st>>>(Pl, ldp, ps, ts, n, G, ldg, sG);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("combine_gram: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

int build_k_planar(cudaStream_t st, double* Kp, long long ld, long long ps, int Lx, int Ly, const cplx* kx,
                   const cplx* ky, std::string* err, long long row0, long long nrows) {
  const long long L = (long long)Lx * Ly;
  if (nrows < 0) nrows = L;
  build_k_planar_kernel<<<(unsigned)std::min<long long>(ceil_div(nrows * L, 256), 148 * 64), 256, 0, st>>>(
      Kp, ld, ps, Lx, Ly, kx, ky, row0, nrows);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("build_k_planar: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

int split_planes(cudaStream_t st, const cplx* U, long long ldu, long long sU, int L, int N, int T, double* Pl,
                 long long ldp, long long ps, long long ts, std::string* err) {
  dim3 grid((unsigned)std::min<long long>(ceil_div(N, 512), 16), L, T);
  split_kernel<<<grid, 256, 0, st>>>(U, ldu, sU, L, N, Pl, ldp, ps, ts);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("split_planes: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

int combine_planes(cudaStream_t st, const double* Pl, long long ldp, long long ps, long long ts, int L, int N, int T,
                   cplx* U, long long ldu, long long sU, std::string* err) {
  dim3 grid((unsigned)std::min<long long>(ceil_div(N, 512), 16), L, T);
  combine_kernel<<<grid, 256, 0, st>>>(Pl, ldp, ps, ts, L, N, U, ldu, sU);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("combine_planes: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

}  // namespace traj
