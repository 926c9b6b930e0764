// Monitoring kernels of the trajectory step and small helpers.
//
// Homodyne / QSD (Eq. A3, split form, readings Q5-Q8): one CTA per row i of
// one trajectory reads the row once into registers, reduces n_i = sum_k |U_ik|^2
// (warp shuffles + one smem pass), draws Philox4x32-10 at counter
// (i, step, traj_global, 0), forms a_i = sqrt(gamma dt) z_i + (2 n_i - 1) gamma dt with
// z_i = sqrt(-2 ln(1-u0)) cos(2 pi u1) and writes exp(a_i) * row back: one HBM read and
// one write of U (32 L N bytes per trajectory-step, the HBM roofline of this phase).
//
// Projective / PM (readings Q10, Q13, Q16, Q17): sites click iff
// u0 < gamma dt; the click list S (ascending) is sampled sequentially on
// C_SS = U_S U_S^dag with the Schur-complement update of Eq. (A1) / sign-corrected (A2):
//     C <- C - C[:,t] C[t,:] / pivot,  pivot = C_tt (occupied) or C_tt - 1 (empty).
#include <math.h>
#include "common.cuh"
#include "monitor.h"
#include "zgemm.h"

namespace traj {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <int BS>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (BS == 32) return v;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < BS / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  return red[0];
}

// mode 0: occupations only; mode 1: homodyne scaling (and occupations)
template <int BS, int VPT>
__global__ void __launch_bounds__(BS) row_monitor_kernel(cplx* U, long long ld, long long sU, int L, int N, int mode,
                                                         long long step, long long traj_base, uint32_t k0, uint32_t k1,
                                                         const double* gamma, double dt, double* n_out, int site0) {
  __shared__ double red[32];
  __shared__ double fac;
  const int i = blockIdx.x, t = blockIdx.y;
  cplx* row = U + t * sU + (long long)i * ld;
  double s = 0.0;
  double2 v[VPT > 0 ? VPT : 1];
  if (VPT > 0) {
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int k = threadIdx.x + q * BS;
      v[q] = k < N ? row[k] : make_double2(0.0, 0.0);
      s += v[q].x * v[q].x + v[q].y * v[q].y;
    }
  } else {
    for (int k = threadIdx.x; k < N; k += BS) {
      const double2 w = row[k];
      s += w.x * w.x + w.y * w.y;
    }
  }
  const double n = block_sum<BS>(s, red);
  if (threadIdx.x == 0) {
    if (n_out) n_out[(long long)t * L + i] = n;
    if (mode == 1) {
      const u32x4 x =
          philox4x32_10(u32x4{(uint32_t)(site0 + i), (uint32_t)step, (uint32_t)(traj_base + t), 0u}, k0, k1);
      const double u0 = u53(x.x, x.y), u1 = u53(x.z, x.w);
      const double z = sqrt(-2.0 * log(1.0 - u0)) * cos(2.0 * M_PI * u1);
      const double gdt = gamma[t] * dt;
      fac = exp(sqrt(gdt) * z + (2.0 * n - 1.0) * gdt);
    }
  }
  if (mode != 1) return;
  __syncthreads();
  const double f = fac;
  if (VPT > 0) {
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int k = threadIdx.x + q * BS;
      if (k < N) row[k] = make_double2(f * v[q].x, f * v[q].y);
    }
  } else {
    for (int k = threadIdx.x; k < N; k += BS) {
      const double2 w = row[k];
      row[k] = make_double2(f * w.x, f * w.y);
    }
  }
}

__global__ void click_draw_kernel(int L, long long step, long long traj_base, uint32_t k0, uint32_t k1,
                                  const double* gamma, double dt, int32_t* flags, int site0) {
  const int t = blockIdx.y;
  const double p = gamma[t] * dt;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    const u32x4 x =
        philox4x32_10(u32x4{(uint32_t)(site0 + i), (uint32_t)step, (uint32_t)(traj_base + t), 0u}, k0, k1);
    flags[(long long)t * L + i] = u53(x.x, x.y) < p ? 1 : 0;
  }
}

// one CTA (1024 threads) per trajectory: ascending list of flagged sites
__global__ void __launch_bounds__(1024) compact_kernel(const int32_t* flags, int L, int32_t* list, int cap,
                                                       int32_t* count, int site0) {
  __shared__ int wsum[32];
  __shared__ int base;
  const int t = blockIdx.x;
  const int32_t* f = flags + (long long)t * L;
  int32_t* out = list + (long long)t * cap;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < L; c0 += 1024) {
    const int i = c0 + threadIdx.x;
    const int fl = i < L ? f[i] : 0;
    const unsigned b = __ballot_sync(0xffffffffu, fl);
    const int before = __popc(b & ((1u << l) - 1u));
    if (l == 0) wsum[w] = __popc(b);
    __syncthreads();
    int off = 0;
    for (int q = 0; q < w; ++q) off += wsum[q];
    const int pos = base + off + before;
    if (fl && pos < cap) out[pos] = site0 + i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int q = 0; q < 32; ++q) tot += wsum[q];
      base += tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) count[t] = base;
}

// dst[t][r][:] = src[t][idx[t][r]][:] for r < count[t]
__global__ void gather_rows_kernel(const cplx* src, long long lds, long long sS, const int32_t* idx, long long sIdx,
                                   const int32_t* count, int fixed_count, cplx* dst, long long ldd, long long sD,
                                   int ncols, int row_offset, int zero_fill) {
  const int t = blockIdx.z;
  const int r = blockIdx.y;
  const int cnt = count ? count[t] : fixed_count;
  if (r >= cnt) {
    if (zero_fill) {
      cplx* d = dst + t * sD + (long long)r * ldd;
      for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ncols; k += gridDim.x * blockDim.x)
        d[k] = make_double2(0.0, 0.0);
    }
    return;
  }
  const long long srow = idx[t * sIdx + r] - row_offset;
  const cplx* s = src + t * sS + srow * lds;
  cplx* d = dst + t * sD + (long long)r * ldd;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ncols; k += gridDim.x * blockDim.x) d[k] = s[k];
}

__device__ __forceinline__ bool decide(double p, double u1) {
  p = fmin(fmax(p, 0.0), 1.0);
  bool occ = u1 < p;
  if (occ && p < 1e-12) occ = false;
  else if (!occ && (1.0 - p) < 1e-12) occ = true;
  return occ;
}

// Blocked sequential conditional Born sampling on C_SS (readings Q13, Q16, Q17).
// Sites are visited in ascending order in panels of PB.  For a panel [s0, s0+nb) the
// kernel below runs the sequential decisions on the nb x nb diagonal block in shared memory:
//   p = Re C_tt, occupied iff u1 < p (Q17 guard), piv_t = p (occupied) or p - 1 (empty),
//   C <- C - C[:,t] C[t,:] / piv_t inside the block (Eq. A1 / sign-corrected A2),
// and returns the unit-lower multipliers as Linv = L^-1 and Dinv_Linv = diag(1/piv) L^-1.
// The trailing block then takes the same rank-nb Schur update on the GEMM:
//   Y = L^-1 C12, Z = diag(1/piv) Y, C22 <- C22 - Y^dag Z.
constexpr int PB = 64;
constexpr int PLD = PB + 1;

__global__ void __launch_bounds__(256) panel_sample_kernel(const cplx* Dw, long long ldd, long long sD,
                                                           const int32_t* S, int cap, const int32_t* count, int s0,
                                                           long long step, long long traj_base, uint32_t key0,
                                                           uint32_t key1, int32_t* occ, cplx* Linv, cplx* DLinv) {
  extern __shared__ double2 psm[];
  double2* A = psm;               // [PB][PLD] panel block, then multipliers below the diagonal
  double2* Li = psm + PB * PLD;   // [PB][PLD] L^-1
  __shared__ double inv_s;
  __shared__ double piv_s[PB];
  const int t = blockIdx.x;
  const int m = count[t] < cap ? count[t] : cap;
  if (s0 >= m) return;
  const int nb = min(PB, m - s0);
  const cplx* D = Dw + t * sD + (long long)s0 * ldd + s0;
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int i = idx / nb, k = idx % nb;
    A[i * PLD + k] = D[(long long)i * ldd + k];
  }
  __syncthreads();
  for (int r = 0; r < nb; ++r) {
    if (threadIdx.x == 0) {
      const int site = S[(long long)t * cap + s0 + r];
      const u32x4 x = philox4x32_10(u32x4{(uint32_t)site, (uint32_t)step, (uint32_t)(traj_base + t), 0u}, key0, key1);
      const double u1 = u53(x.z, x.w);
      const double p = A[r * PLD + r].x;
      const bool o = decide(p, u1);
      occ[(long long)t * cap + s0 + r] = o ? 1 : 0;
      const double pv = o ? p : p - 1.0;
      piv_s[r] = pv;
      inv_s = 1.0 / pv;
    }
    __syncthreads();
    const double inv = inv_s;
    for (int i = r + 1 + threadIdx.x; i < nb; i += blockDim.x) {     // multipliers l_ir
      const double2 v = A[i * PLD + r];
      A[i * PLD + r] = make_double2(v.x * inv, v.y * inv);
    }
    __syncthreads();
    const int mm = nb - r - 1;
    for (int idx = threadIdx.x; idx < mm * mm; idx += blockDim.x) {
      const int i = r + 1 + idx / mm, k = r + 1 + idx % mm;
      const double2 p = cmul(A[i * PLD + r], A[r * PLD + k]);
      A[i * PLD + k].x -= p.x;
      A[i * PLD + k].y -= p.y;
    }
    __syncthreads();
  }
  // L^-1 by forward substitution, one thread per column (L unit lower, multipliers in A)
  for (int k = threadIdx.x; k < PB; k += blockDim.x) {
    for (int i = 0; i < PB; ++i) {
      double2 v = make_double2(i == k ? 1.0 : 0.0, 0.0);
      if (i > k && i < nb) {
        for (int j = k; j < i; ++j) {
          const double2 p = cmul(A[i * PLD + j], Li[j * PLD + k]);
          v.x -= p.x;
          v.y -= p.y;
        }
      } else if (i >= nb) {
        v = make_double2(0.0, 0.0);
      }
      Li[i * PLD + k] = v;
    }
  }
  __syncthreads();
  cplx* lo = Linv + (long long)t * PB * PB;
  cplx* dl = DLinv + (long long)t * PB * PB;
  for (int idx = threadIdx.x; idx < PB * PB; idx += blockDim.x) {
    const int i = idx / PB, k = idx % PB;
    const double2 v = Li[i * PLD + k];
    lo[idx] = v;
    const double ip = i < nb ? 1.0 / piv_s[i] : 0.0;
    dl[idx] = make_double2(v.x * ip, v.y * ip);
  }
}

// occupied / empty site lists from the outcome flags (one thread per trajectory)
__global__ void finalize_outcomes_kernel(const int32_t* S, int cap, const int32_t* count, const int32_t* occ, int T,
                                         int32_t* pos1, int32_t* S1, int32_t* S0, int32_t* k1_out, int32_t* k0_out,
                                         int32_t* pos0) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int m = count[t] < cap ? count[t] : cap;
  const long long b = (long long)t * cap;
  int n1 = 0, n0 = 0;
  for (int r = 0; r < m; ++r) {
    if (occ[b + r]) {
      pos1[b + n1] = r;
      S1[b + n1] = S[b + r];
      ++n1;
    } else {
      if (pos0) pos0[b + n0] = r;
      S0[b + n0] = S[b + r];
      ++n0;
    }
  }
  k1_out[t] = n1;
  k0_out[t] = n0;
}

// D11[a][b] = D0[pos[a]][pos[b]]
__global__ void gather_sub_kernel(const cplx* D0, long long ld0, const int32_t* pos, int k, cplx* D11, long long ld1) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < k * k; idx += gridDim.x * blockDim.x) {
    const int a = idx / k, b = idx % k;
    D11[(long long)a * ld1 + b] = D0[(long long)pos[a] * ld0 + pos[b]];
  }
}

// D11[t][a][b] = D0[t][pos[t][a]][pos[t][b]] for a, b < k[t]; identity padding up to kmax
__global__ void gather_sub_batched_kernel(const cplx* D0, long long ld0, long long s0, const int32_t* pos, int cap,
                                          const int32_t* k, int kmax, cplx* D11, long long ld1, long long s1) {
  const int t = blockIdx.y;
  const int kt = k[t];
  const int32_t* p = pos + (long long)t * cap;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < kmax * kmax; idx += gridDim.x * blockDim.x) {
    const int a = idx / kmax, b = idx % kmax;
    double2 v = make_double2(a == b ? 1.0 : 0.0, 0.0);
    if (a < kt && b < kt) v = D0[t * s0 + (long long)p[a] * ld0 + p[b]];
    D11[t * s1 + (long long)a * ld1 + b] = v;
  }
}

__global__ void sub_identity_batched_kernel(cplx* T, long long ld, long long sT, const int32_t* S1, int cap,
                                            const int32_t* k) {
  const int t = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < k[t]) T[t * sT + (long long)S1[(long long)t * cap + c] * ld + c].x -= 1.0;
}

__global__ void zero_rows_batched_kernel(cplx* U, long long ld, long long sU, const int32_t* rows, int cap,
                                         const int32_t* k, int ncols) {
  const int t = blockIdx.z, r = blockIdx.y;
  if (r >= k[t]) return;
  cplx* p = U + t * sU + (long long)rows[(long long)t * cap + r] * ld;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x)
    p[c] = make_double2(0.0, 0.0);
}

// T[S1[c]][c] -= 1
__global__ void sub_identity_kernel(cplx* T, long long ld, const int32_t* S1, int k, int row0, int nrows,
                                    const int32_t* k_dev) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k || (k_dev && c >= *k_dev)) return;
  const int r = S1[c] - row0;
  if (r >= 0 && r < nrows) T[(long long)r * ld + c].x -= 1.0;
}

__global__ void zero_rows_kernel(cplx* U, long long ld, const int32_t* rows, int nrows, int ncols, int row0,
                                 int nlocal, const int32_t* k_dev) {
  const int r = blockIdx.y;
  if (r >= nrows || (k_dev && r >= *k_dev)) return;
  const int lr = rows[r] - row0;
  if (lr < 0 || lr >= nlocal) return;
  cplx* p = U + (long long)lr * ld;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ncols; k += gridDim.x * blockDim.x)
    p[k] = make_double2(0.0, 0.0);
}

// S = -sum[l ln l + (1-l) ln(1-l)] over n eigenvalues, l clamped to [0, 1];
// bad = 1 if some l is outside [-1e-8, 1+1e-8] or not finite.
__global__ void __launch_bounds__(256) entropy_kernel(const double* lam, int n, double* S_out, int32_t* bad) {
  __shared__ double red[32];
  __shared__ int badf;
  if (threadIdx.x == 0) badf = 0;
  __syncthreads();
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) {
    double l = lam[i];
    if (!(l >= -1e-8 && l <= 1.0 + 1e-8)) badf = 1;
    l = fmin(fmax(l, 0.0), 1.0);
    if (l > 0.0 && l < 1.0) s -= l * log(l) + (1.0 - l) * log(1.0 - l);
  }
  const double tot = block_sum<256>(s, red);
  if (threadIdx.x == 0) {
    *S_out = badf ? nan("") : tot;
    if (badf) *bad = 1;
  }
}

// rows [row0, row0 + nrows) of K = K_y (x) K_x (row-major sites), into K[0..nrows)
__global__ void build_k_kernel(cplx* K, long long ld, int Lx, int Ly, const cplx* kx, const cplx* ky, long long row0,
                               long long nrows) {
  const long long L = (long long)Lx * Ly;
  const long long total = nrows * L;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long r = idx / L, j = idx % L;
    const long long i = row0 + r;
    const int ix = (int)(i % Lx), iy = (int)(i / Lx), jx = (int)(j % Lx), jy = (int)(j / Lx);
    const int dx = ((jx - ix) % Lx + Lx) % Lx, dy = ((jy - iy) % Ly + Ly) % Ly;
    K[r * ld + j] = cmul(kx[dx], ky[dy]);
  }
}

// U[t][site_k - row0][k] = 1 for the occupied sites inside [row0, row0 + nrows)
__global__ void init_state_kernel(cplx* U, long long ld, long long sU, const int32_t* sites, int N, int row0,
                                  int nrows) {
  const int t = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const int r = sites[k] - row0;
  if (r >= 0 && r < nrows) U[t * sU + (long long)r * ld + k] = make_double2(1.0, 0.0);
}

// max over the upper triangle of |G_ij - delta_ij| (component-wise), per batch entry;
// out[t] must be zeroed (non-negative doubles order like their bit patterns).
__global__ void gram_deviation_kernel(const cplx* G, long long ld, long long sG, int n, unsigned long long* out) {
  __shared__ double red[32];
  const int t = blockIdx.y;
  const cplx* g = G + t * sG;
  const long long total = (long long)n * n;
  double m = 0.0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    if (i > j) continue;
    const double2 v = g[(long long)i * ld + j];
    const double e = fmax(fabs(v.x - (i == j ? 1.0 : 0.0)), fabs(v.y));
    m = (e > m || e != e) ? e : m;      // NaN propagates
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = fmax(b, red[w]);
    atomicMax(out + t, (unsigned long long)__double_as_longlong(b));
  }
}

// CholeskyQR2 second pass: G = I + E with |E| ~ kappa^2 eps, so R = I + F + O(E^2) with
// F = triu(E, 1) + diag(E)/2 and R^-1 = I - F + O(E^2).  X = I - F (upper, zeros below).
__global__ void first_order_inverse_kernel(const cplx* G, long long ldg, long long sG, cplx* X, long long ldx,
                                           long long sX, int n) {
  const int t = blockIdx.y;
  const cplx* g = G + t * sG;
  cplx* x = X + t * sX;
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    double2 out = make_double2(0.0, 0.0);
    if (i == j) {
      out.x = 1.0 - 0.5 * (g[(long long)i * ldg + j].x - 1.0);
    } else if (i < j) {
      const double2 v = g[(long long)i * ldg + j];
      out = make_double2(-v.x, -v.y);
    }
    x[(long long)i * ldx + j] = out;
  }
}

// gate[0] = 1 if some trajectory's max|G2 - I| exceeds thr (a NaN -- failed trajectory -- does not),
// then the full factorisation runs; counts the fallbacks on the device
__global__ void cqr2_decide_kernel(const unsigned long long* dev, int T, double thr, int32_t* gate,
                                   unsigned long long* fallbacks) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int full = 0;
  for (int t = 0; t < T; ++t) {
    const double m = __longlong_as_double((long long)dev[t]);
    if (m > thr) full = 1;
  }
  gate[0] = full;
  if (full && fallbacks) fallbacks[0] += 1ull;
}

cudaError_t last(std::string* err, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string(what) + ": " + cudaGetErrorString(e);
  return e;
}

template <int BS, int VPT>
void launch_row(cudaStream_t st, dim3 grid, cplx* U, long long ld, long long sU, int L, int N, int mode,
                long long step, long long traj_base, uint32_t k0, uint32_t k1, const double* gamma, double dt,
                double* n_out, int site0) {
  row_monitor_kernel<BS, VPT><<<grid, BS, 0, st>>>(U, ld, sU, L, N, mode, step, traj_base, k0, k1, gamma, dt, n_out,
                                                   site0);
}

}  // namespace

int row_monitor(cudaStream_t st, cplx* U, long long ld, long long sU, int L, int N, int T, int mode, long long step,
                long long traj_base, uint64_t seed, const double* gamma_dev, double dt, double* n_out,
                std::string* err, int site0) {
  dim3 grid(L, T);
  const uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
#define ROW(BS, VPT) \
  launch_row<BS, VPT>(st, grid, U, ld, sU, L, N, mode, step, traj_base, k0, k1, gamma_dev, dt, n_out, site0)
  if (N <= 32) ROW(32, 1);
  else if (N <= 64) ROW(32, 2);
  else if (N <= 128) ROW(32, 4);
  else if (N <= 256) ROW(256, 1);
  else if (N <= 512) ROW(256, 2);
  else if (N <= 1024) ROW(256, 4);
  else if (N <= 2048) ROW(256, 8);
  else if (N <= 4096) ROW(256, 16);
  else if (N <= 8192) ROW(256, 32);
  else if (N <= 16384) ROW(256, 64);
  else ROW(256, 0);
#undef ROW
  count_launch();
  return last(err, "row_monitor") == cudaSuccess ? 0 : 4;
}

int click_draw(cudaStream_t st, int L, int T, long long step, long long traj_base, uint64_t seed,
               const double* gamma_dev, double dt, int32_t* flags, std::string* err, int site0) {
  dim3 grid((unsigned)std::min<long long>(ceil_div(L, 256), 4096), T);
  click_draw_kernel<<<grid, 256, 0, st>>>(L, step, traj_base, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32),
                                          gamma_dev, dt, flags, site0);
  count_launch();
  return last(err, "click_draw") == cudaSuccess ? 0 : 4;
}

void host_click_counts(int L, int T, long long step, long long traj_base, uint64_t seed, const double* gamma,
                       double dt, int32_t* counts, int site0) {
  const uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  for (int t = 0; t < T; ++t) {
    const double p = gamma[t] * dt;
    int c = 0;
    if (p > 0)
      for (int i = 0; i < L; ++i) {
        const u32x4 x = philox4x32_10(u32x4{(uint32_t)(site0 + i), (uint32_t)step, (uint32_t)(traj_base + t), 0u}, k0, k1);
        c += u53(x.x, x.y) < p ? 1 : 0;
      }
    counts[t] = c;
  }
}

int compact(cudaStream_t st, const int32_t* flags, int L, int T, int32_t* list, int cap, int32_t* count,
            std::string* err, int site0) {
  compact_kernel<<<T, 1024, 0, st>>>(flags, L, list, cap, count, site0);
  count_launch();
  return last(err, "compact") == cudaSuccess ? 0 : 4;
}

int gather_rows(cudaStream_t st, const cplx* src, long long lds, long long sS, const int32_t* idx, long long sIdx,
                const int32_t* count_dev, int rows, int T, cplx* dst, long long ldd, long long sD, int ncols,
                std::string* err, int row_offset, int zero_fill) {
  if (rows <= 0 || T <= 0) return 0;
  dim3 grid((unsigned)std::min<long long>(ceil_div(ncols, 256), 64), rows, T);
  gather_rows_kernel<<<grid, 256, 0, st>>>(src, lds, sS, idx, sIdx, count_dev, rows, dst, ldd, sD, ncols,
                                           row_offset, zero_fill);
  count_launch();
  return last(err, "gather_rows") == cudaSuccess ? 0 : 4;
}

int sample_outcomes(cudaStream_t st, const cplx* D0, cplx* Dw, long long ldd, long long sD, const int32_t* S, int cap,
                    const int32_t* count, int maxc, int T, long long step, long long traj_base, uint64_t seed,
                    int32_t* occ, cplx* Linv, cplx* DLinv, cplx* Ybuf, cplx* Zbuf, long long ldy, int32_t* pos1,
                    int32_t* S1, int32_t* S0, int32_t* k1, int32_t* k0, std::string* err, int32_t* pos0) {
  const uint32_t key0 = (uint32_t)(seed & 0xffffffffu), key1 = (uint32_t)(seed >> 32);
  // work copy of C_SS: every batch entry's leading maxc rows (sD = 0 when unbatched)
  const size_t bytes = (size_t)((T - 1) * sD + (long long)maxc * ldd) * 16;
  if (cudaMemcpyAsync(Dw, D0, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
    if (err) *err = "sample: copy";
    return 4;
  }
  const int smem = 2 * PB * PLD * (int)sizeof(double2);
  ensure_smem((const void*)panel_sample_kernel, smem);
  for (int s0 = 0; s0 < maxc; s0 += PB) {
    panel_sample_kernel<<<T, 256, smem, st>>>(Dw, ldd, sD, S, cap, count, s0, step, traj_base, key0, key1, occ, Linv,
                                              DLinv);
    count_launch();
    if (last(err, "panel_sample") != cudaSuccess) return 4;
    const int rest = maxc - s0 - PB;
    if (rest <= 0) break;
    const cplx* C12 = Dw + (long long)s0 * ldd + s0 + PB;
    int r;
    // Y = L^-1 C12, Z = diag(1/piv) L^-1 C12  (PB x rest)
    if ((r = zgemm(st, 0, 0, PB, rest, PB, 1.0, 0.0, Linv, PB, PB * PB, C12, ldd, sD, 0.0, Ybuf, ldy, PB * ldy, T,
                   TRAJ_TRI_A_LOWER_F, err)))
      return r;
    if ((r = zgemm(st, 0, 0, PB, rest, PB, 1.0, 0.0, DLinv, PB, PB * PB, C12, ldd, sD, 0.0, Zbuf, ldy, PB * ldy, T,
                   TRAJ_TRI_A_LOWER_F, err)))
      return r;
    // C22 -= Y^dag Z
    cplx* C22 = Dw + (long long)(s0 + PB) * ldd + s0 + PB;
    if ((r = zgemm(st, 1, 0, rest, rest, PB, -1.0, 0.0, Ybuf, ldy, PB * ldy, Zbuf, ldy, PB * ldy, 1.0, C22, ldd, sD,
                   T, 0, err)))
      return r;
  }
  finalize_outcomes_kernel<<<(unsigned)ceil_div(T, 128), 128, 0, st>>>(S, cap, count, occ, T, pos1, S1, S0, k1, k0,
                                                                        pos0);
  count_launch();
  return last(err, "finalize_outcomes") == cudaSuccess ? 0 : 4;
}

int gather_sub(cudaStream_t st, const cplx* D0, long long ld0, const int32_t* pos, int k, cplx* D11, long long ld1,
               std::string* err) {
  if (k <= 0) return 0;
  gather_sub_kernel<<<(unsigned)std::min<long long>(ceil_div((long long)k * k, 256), 4096), 256, 0, st>>>(D0, ld0, pos,
                                                                                                       k, D11, ld1);
  count_launch();
  return last(err, "gather_sub") == cudaSuccess ? 0 : 4;
}

int gather_sub_batched(cudaStream_t st, const cplx* D0, long long ld0, long long s0, const int32_t* pos, int cap,
                       const int32_t* k_dev, int kmax, int T, cplx* D11, long long ld1, long long s1,
                       std::string* err) {
  if (kmax <= 0) return 0;
  dim3 grid((unsigned)std::min<long long>(ceil_div((long long)kmax * kmax, 256), 1024), T);
  gather_sub_batched_kernel<<<grid, 256, 0, st>>>(D0, ld0, s0, pos, cap, k_dev, kmax, D11, ld1, s1);
  count_launch();
  return last(err, "gather_sub_batched") == cudaSuccess ? 0 : 4;
}

int sub_identity_batched(cudaStream_t st, cplx* T, long long ld, long long sT, const int32_t* S1, int cap,
                         const int32_t* k_dev, int kmax, int nT, std::string* err) {
  if (kmax <= 0) return 0;
  dim3 grid((unsigned)ceil_div(kmax, 256), nT);
  sub_identity_batched_kernel<<<grid, 256, 0, st>>>(T, ld, sT, S1, cap, k_dev);
  count_launch();
  return last(err, "sub_identity_batched") == cudaSuccess ? 0 : 4;
}

int zero_rows_batched(cudaStream_t st, cplx* U, long long ld, long long sU, const int32_t* rows, int cap,
                      const int32_t* k_dev, int kmax, int T, int ncols, std::string* err) {
  if (kmax <= 0) return 0;
  dim3 grid((unsigned)std::min<long long>(ceil_div(ncols, 256), 64), kmax, T);
  zero_rows_batched_kernel<<<grid, 256, 0, st>>>(U, ld, sU, rows, cap, k_dev, ncols);
  count_launch();
  return last(err, "zero_rows_batched") == cudaSuccess ? 0 : 4;
}

int sub_identity(cudaStream_t st, cplx* T, long long ld, const int32_t* S1, int k, std::string* err, int row0,
                 int nrows, const int32_t* k_dev) {
  if (k <= 0) return 0;
  sub_identity_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(T, ld, S1, k, row0, nrows, k_dev);
  count_launch();
  return last(err, "sub_identity") == cudaSuccess ? 0 : 4;
}

int zero_rows(cudaStream_t st, cplx* U, long long ld, const int32_t* rows, int nrows, int ncols, std::string* err,
              int row0, int nlocal, const int32_t* k_dev) {
  if (nrows <= 0) return 0;
  dim3 grid((unsigned)std::min<long long>(ceil_div(ncols, 256), 64), nrows);
  zero_rows_kernel<<<grid, 256, 0, st>>>(U, ld, rows, nrows, ncols, row0, nlocal, k_dev);
  count_launch();
  return last(err, "zero_rows") == cudaSuccess ? 0 : 4;
}

// bins[r] += sum_{i < R, row0 + i + r < L} |C[i][row0 + i + r]|^2 for r = 1..L-1: one thread
// per distance r, rows visited in order (deterministic).  Eq. (2).
__global__ void bin_abs2_kernel(const cplx* C, long long ld, int R, int row0, int L, double* bins) {
  for (int r = 1 + blockIdx.x * blockDim.x + threadIdx.x; r < L; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    const int imax = min(R, L - r - row0);
    for (int i = 0; i < imax; ++i) {
      const double2 v = C[(long long)i * ld + row0 + i + r];
      s += v.x * v.x + v.y * v.y;
    }
    bins[r] += s;
  }
}

// part[block] = sum over rows < R, columns j with mask[j], of |C[i][j]|^2 (Eq. 5)
__global__ void masked_abs2_kernel(const cplx* C, long long ld, int R, int ncols, const int32_t* mask, double* part) {
  __shared__ double red[32];
  double s = 0.0;
  const long long total = (long long)R * ncols;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / ncols), j = (int)(idx % ncols);
    if (mask[j]) {
      const double2 v = C[(long long)i * ld + j];
      s += v.x * v.x + v.y * v.y;
    }
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// out[0] += sum of part[0..n) (one thread, fixed order: deterministic)
__global__ void accumulate_kernel(const double* part, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    out[0] += s;
  }
}

// upper triangle of each n x n batch entry set to the identity
__global__ void set_identity_kernel(cplx* G, long long ld, long long sG, int n) {
  const int t = blockIdx.y;
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    if (i <= j) G[t * sG + (long long)i * ld + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
}

// X = a X + b I on every n x n batch entry (full matrix)
__global__ void axpby_identity_kernel(cplx* X, long long ld, long long sX, int n, double a, double b) {
  const int t = blockIdx.y;
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    cplx* p = X + t * sX + (long long)i * ld + j;
    const double2 v = *p;
    *p = make_double2(a * v.x + (i == j ? b : 0.0), a * v.y);
  }
}

// out += in (n doubles): the single-GPU emulation of an all-reduce
__global__ void add_kernel(double* out, const double* in, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] += in[i];
}

int bin_abs2(cudaStream_t st, const cplx* C, long long ld, int R, int row0, int L, double* bins, std::string* err) {
  bin_abs2_kernel<<<(unsigned)ceil_div(L, 256), 256, 0, st>>>(C, ld, R, row0, L, bins);
  count_launch();
  return last(err, "bin_abs2") == cudaSuccess ? 0 : 4;
}

int masked_abs2(cudaStream_t st, const cplx* C, long long ld, int R, int ncols, const int32_t* mask, double* part,
                double* out, std::string* err) {
  const int blocks = (int)std::min<long long>(ceil_div((long long)R * ncols, 256), 1024);
  masked_abs2_kernel<<<blocks, 256, 0, st>>>(C, ld, R, ncols, mask, part);
  accumulate_kernel<<<1, 32, 0, st>>>(part, blocks, out);
  count_launch(2);
  return last(err, "masked_abs2") == cudaSuccess ? 0 : 4;
}

int axpby_identity(cudaStream_t st, cplx* X, long long ld, long long sX, int n, int T, double a, double b,
                   std::string* err) {
  dim3 grid((unsigned)std::min<long long>(ceil_div((long long)n * n, 256), 8192), T);
  axpby_identity_kernel<<<grid, 256, 0, st>>>(X, ld, sX, n, a, b);
  count_launch();
  return last(err, "axpby_identity") == cudaSuccess ? 0 : 4;
}

int set_identity(cudaStream_t st, cplx* G, long long ld, long long sG, int n, int T, std::string* err) {
  dim3 grid((unsigned)std::min<long long>(ceil_div((long long)n * n, 256), 8192), T);
  set_identity_kernel<<<grid, 256, 0, st>>>(G, ld, sG, n);
  count_launch();
  return last(err, "set_identity") == cudaSuccess ? 0 : 4;
}

int add_inplace(cudaStream_t st, double* out, const double* in, long long n, std::string* err) {
  add_kernel<<<(unsigned)std::min<long long>(ceil_div(n, 256), 148 * 32), 256, 0, st>>>(out, in, n);
  count_launch();
  return last(err, "add") == cudaSuccess ? 0 : 4;
}

int entropy_reduce(cudaStream_t st, const double* lam, int n, double* S_out, int32_t* bad, std::string* err) {
  entropy_kernel<<<1, 256, 0, st>>>(lam, n, S_out, bad);
  count_launch();
  return last(err, "entropy") == cudaSuccess ? 0 : 4;
}

int build_k(cudaStream_t st, cplx* K, long long ld, int Lx, int Ly, const cplx* kx, const cplx* ky, std::string* err,
            long long row0, long long nrows) {
  const long long L = (long long)Lx * Ly;
  if (nrows < 0) nrows = L;
  build_k_kernel<<<(unsigned)std::min<long long>(ceil_div(nrows * L, 256), 148 * 64), 256, 0, st>>>(K, ld, Lx, Ly, kx,
                                                                                                   ky, row0, nrows);
  count_launch();
  return last(err, "build_k") == cudaSuccess ? 0 : 4;
}

int gram_deviation(cudaStream_t st, const cplx* G, long long ld, long long sG, int n, int T, unsigned long long* out,
                   std::string* err) {
  if (cudaMemsetAsync(out, 0, (size_t)T * 8, st) != cudaSuccess) return 4;
  dim3 grid((unsigned)std::min<long long>(ceil_div((long long)n * n, 256), 2048), T);
  gram_deviation_kernel<<<grid, 256, 0, st>>>(G, ld, sG, n, out);
  count_launch();
  return last(err, "gram_deviation") == cudaSuccess ? 0 : 4;
}

__global__ void sum_i32_kernel(const int32_t* in, int n, int32_t* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int v = 0;
    for (int i = 0; i < n; ++i) v += in[i];
    out[0] = v;
  }
}

int sum_i32(cudaStream_t st, const int32_t* in, int n, int32_t* out, std::string* err) {
  sum_i32_kernel<<<1, 32, 0, st>>>(in, n, out);
  count_launch();
  return last(err, "sum_i32") == cudaSuccess ? 0 : 4;
}

int cqr2_decide(cudaStream_t st, const unsigned long long* dev, int T, double thr, int32_t* gate,
                unsigned long long* fallbacks, std::string* err) {
  cqr2_decide_kernel<<<1, 32, 0, st>>>(dev, T, thr, gate, fallbacks);
  count_launch();
  return last(err, "cqr2_decide") == cudaSuccess ? 0 : 4;
}

int first_order_inverse(cudaStream_t st, const cplx* G, long long ldg, long long sG, cplx* X, long long ldx,
                        long long sX, int n, int T, std::string* err) {
  dim3 grid((unsigned)std::min<long long>(ceil_div((long long)n * n, 256), 8192), T);
  first_order_inverse_kernel<<<grid, 256, 0, st>>>(G, ldg, sG, X, ldx, sX, n);
  count_launch();
  return last(err, "first_order_inverse") == cudaSuccess ? 0 : 4;
}

int init_state(cudaStream_t st, cplx* U, long long ld, long long sU, const int32_t* sites, int N, int T,
               std::string* err, int row0, int nrows) {
  dim3 grid((unsigned)ceil_div(N, 256), T);
  init_state_kernel<<<grid, 256, 0, st>>>(U, ld, sU, sites, N, row0, nrows);
  count_launch();
  return last(err, "init_state") == cudaSuccess ? 0 : 4;
}

}  // namespace traj
