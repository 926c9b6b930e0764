// Orthonormality probe for the low-rank projective orthonormaliser (NEXT-1 option).
//
// The low-rank (Loewdin) step is exact only if U was orthonormal; its rounding accumulates as a
// slow drift of E = U^dag U - I (measured: ||E||_F grows by ~7.5e-15 per step at c3).  Instead of
// measuring the N x N Gram every step (4 L N^2 flops), estimate ||E||_F with m unit-modulus
// Rademacher probes (Hutchinson, E[x x^dag] = I):  z_j = U^dag (U x_j) - x_j = E x_j,
// est^2 = (1/m) sum_j ||z_j||^2.  Unit modulus makes the estimate exact for an error confined to
// one entry pair (|x_k| = 1).  Two HBM-bound passes over U (32 L N bytes per trajectory), no
// atomics (deterministic): Y = U X by rows, then U^dag Y by column blocks x row splits, then a
// per-trajectory finish that sums the splits and reduces ||Z - X||^2.
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "probe.h"

namespace traj {

size_t probe_x_bytes(long long N, int T) { return (size_t)T * N * PROBE_M * 16; }
size_t probe_y_bytes(long long L, int T) { return (size_t)T * L * PROBE_M * 16; }
size_t probe_partial_bytes(long long N, int T) {
  return (size_t)T * PROBE_RS_MAX * N * PROBE_M * 16 + (size_t)T * 256 * 8;
}

namespace {

constexpr double R2 = 0.70710678118654752440;

// X[t][k][j] = ((-1)^b0 + i (-1)^b1) / sqrt(2), bits from Philox (k, step, traj, 3)
__global__ void probe_gen_kernel(int N, long long step, long long traj_base, uint32_t k0, uint32_t k1, cplx* X) {
  const int t = blockIdx.y;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    const u32x4 r = philox4x32_10(u32x4{(uint32_t)k, (uint32_t)step, (uint32_t)(traj_base + t), 3u}, k0, k1);
#pragma unroll
    for (int j = 0; j < PROBE_M; ++j) {
      const uint32_t b = r.x >> (2 * j);
      X[((long long)t * N + k) * PROBE_M + j] = make_double2((b & 1) ? -R2 : R2, (b & 2) ? -R2 : R2);
    }
  }
}

// Y[t][i][j] = sum_k U[t][i][k] X[t][k][j].  CTA: 4 warps x 4 rows, k in chunks of KC staged in
// shared memory; lane-strided k (coalesced 512-byte row segments).
constexpr int PR_ROWS = 16, PR_KC = 256, PR_THREADS = 128;
__global__ void __launch_bounds__(PR_THREADS, 4) probe_rows_kernel(const cplx* __restrict__ U, long long ld, long long sU, int L,
                                                         int N, const cplx* __restrict__ X, cplx* __restrict__ Y) {
  __shared__ double2 xs[PR_KC][PROBE_M];
  const int t = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.x * PR_ROWS + warp * 4;
  const cplx* u = U + (long long)t * sU;
  const cplx* x = X + (long long)t * N * PROBE_M;
  double2 acc[4][PROBE_M];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < PROBE_M; ++j) acc[r][j] = make_double2(0.0, 0.0);
  for (int kc = 0; kc < N; kc += PR_KC) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < PR_KC * PROBE_M; idx += blockDim.x) {
      const int kk = idx / PROBE_M, j = idx % PROBE_M;
      xs[kk][j] = kc + kk < N ? x[(long long)(kc + kk) * PROBE_M + j] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = lane; kk < PR_KC && kc + kk < N; kk += 32) {
      double2 v[4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        v[r] = i0 + r < L ? u[(long long)(i0 + r) * ld + kc + kk] : make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < PROBE_M; ++j) {
        const double2 w = xs[kk][j];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          acc[r][j].x += v[r].x * w.x - v[r].y * w.y;
          acc[r][j].y += v[r].x * w.y + v[r].y * w.x;
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < PROBE_M; ++j) {
      double a = acc[r][j].x, b = acc[r][j].y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      if (lane == 0 && i0 + r < L) Y[((long long)t * L + i0 + r) * PROBE_M + j] = make_double2(a, b);
    }
}

// partial[t][s][k][j] = sum_{i in split s} conj(U[t][i][k]) Y[t][i][j].  One thread per column k;
// Y rows staged in shared memory (broadcast reads).
constexpr int PC_COLS = 256, PC_YR = 64;
__global__ void __launch_bounds__(PC_COLS) probe_cols_kernel(const cplx* __restrict__ U, long long ld, long long sU,
                                                             int L, int N, int rows_per_split,
                                                             const cplx* __restrict__ Y, cplx* __restrict__ partial) {
  __shared__ double2 ys[PC_YR][PROBE_M];
  const int t = blockIdx.z, s = blockIdx.y;
  const int k = blockIdx.x * PC_COLS + threadIdx.x;
  const int r0 = s * rows_per_split, r1 = min(L, r0 + rows_per_split);
  const cplx* u = U + (long long)t * sU;
  const cplx* y = Y + (long long)t * L * PROBE_M;
  double2 acc[PROBE_M];
#pragma unroll
  for (int j = 0; j < PROBE_M; ++j) acc[j] = make_double2(0.0, 0.0);
  for (int rc = r0; rc < r1; rc += PC_YR) {
    const int nr = min(PC_YR, r1 - rc);
    __syncthreads();
    for (int idx = threadIdx.x; idx < nr * PROBE_M; idx += blockDim.x)
      ys[idx / PROBE_M][idx % PROBE_M] = y[(long long)rc * PROBE_M + idx];
    __syncthreads();
    if (k < N) {
      for (int r = 0; r < nr; ++r) {
        const double2 v = u[(long long)(rc + r) * ld + k];
#pragma unroll
        for (int j = 0; j < PROBE_M; ++j) {
          const double2 w = ys[r][j];       // conj(v) w
          acc[j].x += v.x * w.x + v.y * w.y;
          acc[j].y += v.x * w.y - v.y * w.x;
        }
      }
    }
  }
  if (k < N) {
    cplx* p = partial + (((long long)t * PROBE_RS_MAX + s) * N + k) * PROBE_M;
#pragma unroll
    for (int j = 0; j < PROBE_M; ++j) p[j] = acc[j];
  }
}

// part2[t][b] = sum over this block's (k, j) of |sum_s partial[t][s][k][j] - X[t][k][j]|^2
constexpr int PF_BLOCKS = 256;
__global__ void probe_reduce_kernel(int N, int splits, const cplx* __restrict__ partial, const cplx* __restrict__ X,
                                    double* part2) {
  __shared__ double red[32];
  const int t = blockIdx.y;
  const long long n = (long long)N * PROBE_M;
  double acc = 0.0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n; idx += (long long)gridDim.x * blockDim.x) {
    double2 z = make_double2(0.0, 0.0);
    for (int s = 0; s < splits; ++s) {
      const double2 p = partial[((long long)t * PROBE_RS_MAX + s) * n + idx];
      z.x += p.x;
      z.y += p.y;
    }
    const double2 x = X[(long long)t * n + idx];
    const double a = z.x - x.x, b = z.y - x.y;
    acc += a * a + b * b;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    part2[(long long)t * PF_BLOCKS + blockIdx.x] = s;
  }
}

// est[t] = sqrt((1/m) sum_b part2[t][b]), fixed order
__global__ void probe_finish_kernel(int nblocks, const double* part2, double* est) {
  const int t = blockIdx.x;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += part2[(long long)t * PF_BLOCKS + b];
    est[t] = sqrt(s / PROBE_M);
  }
}

}  // namespace

int probe_orthonormality(cudaStream_t st, const cplx* U, long long ld, long long sU, int L, int N, int T,
                         long long step, long long traj_base, uint64_t seed, cplx* X, cplx* Y, cplx* partial,
                         double* est, std::string* err) {
  const uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  probe_gen_kernel<<<dim3((unsigned)ceil_div(N, 256), T), 256, 0, st>>>(N, step, traj_base, k0, k1, X);
  probe_rows_kernel<<<dim3((unsigned)ceil_div(L, PR_ROWS), T), PR_THREADS, 0, st>>>(U, ld, sU, L, N, X, Y);
  // row splits: about 4 CTAs per SM over (column blocks x splits x T), at least 64 rows per split
  const long long cblocks = ceil_div(N, PC_COLS);
  long long splits = ceil_div(4 * 148, cblocks * T);
  splits = std::max<long long>(1, std::min<long long>(std::min<long long>(splits, PROBE_RS_MAX), ceil_div(L, 64)));
  const int rows_per_split = (int)ceil_div(L, splits);
  splits = ceil_div(L, rows_per_split);
  probe_cols_kernel<<<dim3((unsigned)cblocks, (unsigned)splits, T), PC_COLS, 0, st>>>(U, ld, sU, L, N, rows_per_split,
                                                                                     Y, partial);
  // the reduction partials live after the split partials of the last trajectory's slot
  double* part2 = reinterpret_cast<double*>(partial + (size_t)T * PROBE_RS_MAX * N * PROBE_M);
  const int nb = (int)std::min<long long>(PF_BLOCKS, ceil_div((long long)N * PROBE_M, 256));
  probe_reduce_kernel<<<dim3((unsigned)nb, T), 256, 0, st>>>(N, (int)splits, partial, X, part2);
  probe_finish_kernel<<<T, 32, 0, st>>>(nb, part2, est);
  count_launch(5);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (err) *err = std::string("probe_orthonormality: ") + cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

}  // namespace traj
