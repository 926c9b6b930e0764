// NEXT-2: the paper-literal QSD integrator ("fourth-order
// Runge-Kutta ... with a time step dt = 0.05", then QR).
//
// Over one step the generator of Eq. (A3) is held fixed (dW and <n>_t at time t):
//     dU/dt = M U,   X = dt M = -i dt H~ + diag(d),   d_i = dW_i + (2 n_i - 1) gamma dt,
// with H~ the nearest-neighbour hopping applied as a stencil.  Classical RK4 on a
// linear autonomous system is exactly the degree-4 Taylor polynomial of exp(X), evaluated
// here in Horner form with four fused passes (W_4 = U + X U / 4, W_j = U + X W_{j+1} / j,
// U' = W_1), each reading W and U and writing W': HBM-bound, 48 L N bytes per pass.
#include <math.h>
#include "common.cuh"
#include "qsd_rk4.h"

namespace traj {

namespace {

// d[t][i] = sqrt(gamma dt) z_i + (2 n_i - 1) gamma dt, z from the Philox draw of (i, step, traj)
__global__ void qsd_diag_kernel(const double* n, int L, int T, long long step, long long traj_base, uint32_t k0,
                                uint32_t k1, const double* gamma, double dt, double* d) {
  const int t = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    const u32x4 x = philox4x32_10(u32x4{(uint32_t)i, (uint32_t)step, (uint32_t)(traj_base + t), 0u}, k0, k1);
    const double u0 = u53(x.x, x.y), u1 = u53(x.z, x.w);
    const double z = sqrt(-2.0 * log(1.0 - u0)) * cos(2.0 * M_PI * u1);
    const double gdt = gamma[t] * dt;
    d[(long long)t * L + i] = sqrt(gdt) * z + (2.0 * n[(long long)t * L + i] - 1.0) * gdt;
  }
}

// out = U + inv_j (X W), X W = -i dt J sum_nbr W_nbr + d_i W_i   (one thread per (row, col))
__global__ void horner_pass_kernel(const cplx* __restrict__ U, const cplx* __restrict__ W, cplx* __restrict__ out,
                                   long long ld, long long sU, int N, int Lx, int Ly, const double* __restrict__ d,
                                   double hop, double inv_j) {
  const int t = blockIdx.z;
  const int i = blockIdx.y;
  const int L = Lx * Ly;
  const int x = i % Lx, y = i / Lx;
  const int ip = y * Lx + (x + 1) % Lx, im = y * Lx + (x + Lx - 1) % Lx;
  const int jp = ((y + 1) % Ly) * Lx + x, jm = ((y + Ly - 1) % Ly) * Lx + x;
  const cplx* w = W + (long long)t * sU;
  const double di = d[(long long)t * L + i];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    double2 s = w[(long long)ip * ld + k];
    const double2 a = w[(long long)im * ld + k];
    s.x += a.x;
    s.y += a.y;
    if (Ly > 1) {
      const double2 b = w[(long long)jp * ld + k], c = w[(long long)jm * ld + k];
      s.x += b.x + c.x;
      s.y += b.y + c.y;
    }
    const double2 wi = w[(long long)i * ld + k];
    const double2 u = U[(long long)t * sU + (long long)i * ld + k];
    // -i hop s + d_i w_i
    const double xr = hop * s.y + di * wi.x;
    const double xi = -hop * s.x + di * wi.y;
    out[(long long)t * sU + (long long)i * ld + k] = make_double2(u.x + inv_j * xr, u.y + inv_j * xi);
  }
}

}  // namespace

int qsd_rk4_propagate(cudaStream_t st, const cplx* U, cplx* Wtmp, cplx* out, long long ld, long long sU, int Lx,
                      int Ly, int N, int T, const double* n, double* d, long long step, long long traj_base,
                      uint64_t seed, const double* gamma_dev, double J, double dt, std::string* err) {
  const int L = Lx * Ly;
  dim3 g1((unsigned)std::min<long long>(ceil_div(L, 256), 1024), T);
  qsd_diag_kernel<<<g1, 256, 0, st>>>(n, L, T, step, traj_base, (uint32_t)(seed & 0xffffffffu),
                                      (uint32_t)(seed >> 32), gamma_dev, dt, d);
  count_launch();
  const double hop = dt * J;
  dim3 g2((unsigned)std::min<long long>(ceil_div(N, 256), 64), L, T);
  // W4 = U + X U / 4 -> Wtmp;  W3 = U + X W4 / 3 -> out;  W2 = U + X W3 / 2 -> Wtmp;  U' = U + X W2 -> out
  const cplx* src[4] = {U, Wtmp, out, Wtmp};
  cplx* dst[4] = {Wtmp, out, Wtmp, out};
  for (int p = 0; p < 4; ++p) {
    horner_pass_kernel<<<g2, 256, 0, st>>>(U, src[p], dst[p], ld, sU, N, Lx, Ly, d, hop, 1.0 / (4 - p));
    count_launch();
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (err) *err = std::string("qsd_rk4: ") + cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

}  // namespace traj
