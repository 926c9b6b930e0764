// Exact modular complex-FP64 products on the INT8 tensor cores (Ozaki-II / CRT; see ozaki.h).
#include "ozaki.h"
#include "igemm.h"
#include <map>
#include <mutex>
#include <set>

namespace traj {
namespace {

// pairwise coprime moduli <= 256 (the first s are used); residues are stored in [-128, 127]
__host__ __device__ constexpr int OZM(int q) {
  return q == 0 ? 256 : q == 1 ? 255 : q == 2 ? 253 : q == 3 ? 251 : q == 4 ? 247 : q == 5 ? 241 : q == 6 ? 239
       : q == 7 ? 233 : q == 8 ? 229 : q == 9 ? 227 : q == 10 ? 223 : q == 11 ? 217 : q == 12 ? 211
       : q == 13 ? 199 : q == 14 ? 197 : 193;
}
__host__ __device__ constexpr int pow2mod(int e, int m) {
  int r = 1 % m;
  for (int i = 0; i < e; ++i) r = (r * 2) % m;
  return r;
}

// CRT constants per s: X / M = frac(sum_q r_q c_q), c_q = ((M / m_q)^-1 mod m_q) / m_q = ch_q + cl_q,
// ch_q a multiple of 2^-45 (so r_q ch_q is exact for r_q < 256), M = prod m_q (as a double)
__constant__ double c_ch[OZ_MAXS + 1][OZ_MAXS];
__constant__ double c_cl[OZ_MAXS + 1][OZ_MAXS];
__constant__ double c_M[OZ_MAXS + 1];
__constant__ uint32_t c_mod[OZ_MAXS], c_c21[OZ_MAXS], c_c42[OZ_MAXS], c_magic[OZ_MAXS];

struct HostConst {
  double ch[OZ_MAXS + 1][OZ_MAXS] = {};
  double cl[OZ_MAXS + 1][OZ_MAXS] = {};
  double M[OZ_MAXS + 1] = {};
  int beta[OZ_MAXS + 1] = {};
  HostConst() {
    typedef unsigned __int128 u128;
    for (int s = 1; s <= OZ_MAXS; ++s) {
      u128 Mp = 1;
      for (int q = 0; q < s; ++q) Mp *= (u128)OZM(q);
      // double of M and floor(log2(M))
      M[s] = (double)(uint64_t)(Mp >> 64) * 18446744073709551616.0 + (double)(uint64_t)Mp;
      int lg = 0;
      for (u128 x = Mp; x > 1; x >>= 1) ++lg;
      beta[s] = lg / 2 - 1;
      for (int q = 0; q < s; ++q) {
        const int m = OZM(q);
        const int Mi = (int)((Mp / (u128)m) % (u128)m);
        int inv = 0;
        for (int x = 1; x < m; ++x)
          if ((long long)Mi * x % m == 1) {
            inv = x;
            break;
          }
        // n = round(inv 2^45 / m); cl = (inv 2^45 - n m) / (m 2^45)
        const long long num = (long long)inv << 45;
        const long long n = (num + m / 2) / m;
        ch[s][q] = (double)n * 0x1p-45;
        cl[s][q] = (double)(num - n * m) / (double)m * 0x1p-45;
      }
    }
  }
};

const HostConst& host_const() {
  static HostConst c;
  return c;
}

int ensure_device_constants(const int** moduli_dev, std::string* err) {
  static std::mutex mu;
  static std::map<int, int*> mods;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    if (err) *err = "ozaki: cudaGetDevice";
    return 4;
  }
  std::lock_guard<std::mutex> g(mu);
  auto it = mods.find(dev);
  if (it == mods.end()) {
    const HostConst& h = host_const();
    int* d = nullptr;
    int mh[OZ_MAXS];
    for (int q = 0; q < OZ_MAXS; ++q) mh[q] = OZM(q);
    uint32_t tm[4][OZ_MAXS];
    for (int q = 0; q < OZ_MAXS; ++q) {
      const uint32_t m = OZM(q);
      tm[0][q] = m;
      tm[1][q] = pow2mod(21, m);
      tm[2][q] = pow2mod(42, m);
      tm[3][q] = (uint32_t)(4294967296ULL / m);
    }
    if (cudaMemcpyToSymbol(c_mod, tm[0], sizeof(tm[0])) != cudaSuccess ||
        cudaMemcpyToSymbol(c_c21, tm[1], sizeof(tm[1])) != cudaSuccess ||
        cudaMemcpyToSymbol(c_c42, tm[2], sizeof(tm[2])) != cudaSuccess ||
        cudaMemcpyToSymbol(c_magic, tm[3], sizeof(tm[3])) != cudaSuccess ||
        cudaMemcpyToSymbol(c_ch, h.ch, sizeof(h.ch)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_cl, h.cl, sizeof(h.cl)) != cudaSuccess ||
        cudaMemcpyToSymbol(c_M, h.M, sizeof(h.M)) != cudaSuccess || cudaMalloc(&d, sizeof(mh)) != cudaSuccess ||
        cudaMemcpy(d, mh, sizeof(mh), cudaMemcpyHostToDevice) != cudaSuccess) {
      if (err) *err = "ozaki: constant upload";
      return 4;
    }
    it = mods.emplace(dev, d).first;
  }
  *moduli_dev = it->second;
  return 0;
}

// exponent e with nu 2^e < 2^beta (nu = the row's / column's 2-norm of |re| + |im|); 0 for a zero row
__device__ __forceinline__ int scale_exp(double nu2, int beta) {
  if (!(nu2 > 0.0)) return 0;
  return beta - ilogb(sqrt(nu2)) - 1;
}

// residue in [0, m) of the integer x (|x| < 2^62), by 21-bit digits: every partial sum < 2^30
template <int Q>
__device__ __forceinline__ uint32_t res_of(long long x) {
  constexpr int m = OZM(Q);
  constexpr uint32_t c21 = pow2mod(21, m), c42 = pow2mod(42, m);
  const unsigned long long u = x < 0 ? (unsigned long long)(-x) : (unsigned long long)x;
  const uint32_t x0 = (uint32_t)(u & 0x1FFFFF), x1 = (uint32_t)((u >> 21) & 0x1FFFFF), x2 = (uint32_t)(u >> 42);
  uint32_t r = (x2 * c42 + x1 * c21 + x0) % (uint32_t)m;
  if (x < 0 && r) r = m - r;
  return r;
}

// [0, m) -> the symmetric int8 representative as a byte
template <int Q>
__device__ __forceinline__ uint32_t sym8(uint32_t r) {
  constexpr int m = OZM(Q);
  return (uint32_t)(uint8_t)(int8_t)((int)r > (m - 1) / 2 ? (int)r - m : (int)r);
}

template <int Q>
__device__ __forceinline__ void planes_of(long long vr, long long vi, int conj, uint32_t (&b)[4]) {
  constexpr uint32_t m = OZM(Q);
  const uint32_t a = res_of<Q>(vr);
  uint32_t c = res_of<Q>(vi);
  if (conj && c) c = m - c;
  uint32_t s = a + c;
  s -= s >= m ? m : 0;
  uint32_t d = a + m - c;
  d -= d >= m ? m : 0;
  b[0] = sym8<Q>(a);
  b[1] = sym8<Q>(c);
  b[2] = sym8<Q>(s);
  b[3] = sym8<Q>(d);
}

__device__ __forceinline__ long long to_int(double v, int e) { return __double2ll_rn(scalbn(v, e)); }

template <int S, int NP, int Q = 0>
struct RowStore {
  // 4 consecutive elements -> one 32-bit word per (plane, modulus)
  __device__ __forceinline__ static void run(const long long (&vr)[4], const long long (&vi)[4], int conj, int8_t* R,
                                             long long pstride, long long qstride) {
    if constexpr (Q < S) {
      uint32_t w[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) w[p] = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t b[4];
        planes_of<Q>(vr[k], vi[k], conj, b);
#pragma unroll
        for (int p = 0; p < NP; ++p) w[p] |= b[p] << (8 * k);
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) *reinterpret_cast<uint32_t*>(R + p * pstride + Q * qstride) = w[p];
      RowStore<S, NP, Q + 1>::run(vr, vi, conj, R, pstride, qstride);
    }
  }
};

template <int S, int NP>
__global__ void __launch_bounds__(256) oz_split_rows_kernel(const cplx* __restrict__ X, long long ldx, long long sX,
                                                            int rows, int cols_cap, int T, int conj, int8_t* R,
                                                            long long ldr, int* e, long long sE, int beta,
                                                            const int32_t* gate, const int32_t* cdev) {
  if (gate && *gate == 0) return;
  const int row = blockIdx.x, t = blockIdx.y;
  const cplx* x = X + t * sX + (long long)row * ldx;
  const int cols = cdev ? min(cols_cap, cdev[t]) : cols_cap;   // past it: zero residues
  __shared__ double red[8];
  __shared__ int ex_s;
  double acc = 0.0;
  for (int j = threadIdx.x; j < cols; j += 256) {
    const cplx v = x[j];
    const double a = fabs(v.x) + fabs(v.y);
    acc = fma(a, a, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    ex_s = scale_exp(s, beta);
    e[t * sE + row] = ex_s;
  }
  __syncthreads();
  const int ex = ex_s;
  const long long qstride = (long long)T * rows * ldr, pstride = (long long)S * qstride;
  int8_t* Rrow = R + (long long)t * rows * ldr + (long long)row * ldr;
  for (int j0 = 4 * threadIdx.x; j0 < cols_cap; j0 += 1024) {
    long long vr[4], vi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (j0 + k < cols) {
        const cplx v = x[j0 + k];
        vr[k] = to_int(v.x, ex);
        vi[k] = to_int(v.y, ex);
      } else {
        vr[k] = vi[k] = 0;
      }
    }
    RowStore<S, NP>::run(vr, vi, conj, Rrow + j0, pstride, qstride);
  }
}

// per-column partial sums of (|re| + |im|)^2 over 8 row chunks: part[(c T + t) cols + j]
__global__ void __launch_bounds__(256) oz_colnorm_kernel(const cplx* __restrict__ X, long long ldx, long long sX,
                                                         int rows, int cols, int T, double* part, int subI,
                                                         const int32_t* gate) {
  if (gate && *gate == 0) return;
  const int j = blockIdx.x * 32 + threadIdx.x, c = blockIdx.y, t = blockIdx.z;
  const int per = (rows + 7) / 8, r0 = c * per, r1 = min(rows, r0 + per);
  double acc = 0.0;
  if (j < cols) {
    const cplx* x = X + t * sX + j;
    for (int i = r0 + threadIdx.y; i < r1; i += 8) {
      const cplx v = x[(long long)i * ldx];
      const double a = fabs(v.x - (subI && i == j ? 1.0 : 0.0)) + fabs(v.y);
      acc = fma(a, a, acc);
    }
  }
  __shared__ double red[8][33];
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && j < cols) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
    part[((long long)c * T + t) * cols + j] = s;
  }
}

constexpr int CT = 64;   // column-split tile: 64 columns of X x 64 rows of X

// the 21-bit digits of |x| (|x| < 2^62) and its sign
struct Digits {
  uint32_t d0, d1, d2;
  bool neg;
};
__device__ __forceinline__ Digits digits_of(long long x) {
  const unsigned long long u = x < 0 ? (unsigned long long)(-x) : (unsigned long long)x;
  return Digits{(uint32_t)(u & 0x1FFFFF), (uint32_t)((u >> 21) & 0x1FFFFF), (uint32_t)(u >> 42), x < 0};
}
// residue in [0, m_q) with run-time tables (the column split's 16 values per thread leave no
// registers for a fully unrolled modulus loop)
__device__ __forceinline__ uint32_t res_rt(const Digits& d, int q) {
  const uint32_t m = c_mod[q];
  const uint32_t y = d.d2 * c_c42[q] + d.d1 * c_c21[q] + d.d0;   // < 2^30
  uint32_t r = y - __umulhi(y, c_magic[q]) * m;                 // in [0, m + 64)
  r -= r >= m ? m : 0;
  if (d.neg && r) r = m - r;
  return r;
}
__device__ __forceinline__ uint32_t sym8_rt(uint32_t r, uint32_t m) {
  return (uint32_t)(uint8_t)(int8_t)((int)r > ((int)m - 1) / 2 ? (int)r - (int)m : (int)r);
}

template <int S, int NP>
__device__ __forceinline__ void col_store(const Digits (&dr)[16], const Digits (&di)[16], int8_t* R, long long pstride,
                                          long long qstride) {
#pragma unroll 1
  for (int q = 0; q < S; ++q) {
    const uint32_t m = c_mod[q];
    uint32_t w[NP][4];
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int i = 0; i < 4; ++i) w[p][i] = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t a = res_rt(dr[k], q), c = res_rt(di[k], q);
      uint32_t sm = a + c;
      sm -= sm >= m ? m : 0;
      uint32_t df = a + m - c;
      df -= df >= m ? m : 0;
      const uint32_t b[4] = {sym8_rt(a, m), sym8_rt(c, m), sym8_rt(sm, m), sym8_rt(df, m)};
#pragma unroll
      for (int p = 0; p < NP; ++p) w[p][k >> 2] |= b[p] << (8 * (k & 3));
    }
#pragma unroll
    for (int p = 0; p < NP; ++p)
      *reinterpret_cast<uint4*>(R + p * pstride + q * qstride) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
  }
}

template <int S, int NP>
__global__ void __launch_bounds__(256) oz_split_cols_kernel(const cplx* __restrict__ X, long long ldx, long long sX,
                                                            int rows, int cols, int T, int8_t* R, long long ldr,
                                                            int* e, long long sE, const double* part, int beta,
                                                            int subI, const int32_t* gate, const int32_t* cdev) {
  if (gate && *gate == 0) return;
  extern __shared__ cplx tile[];   // [CT rows][CT + 1]
  const int j0 = blockIdx.x * CT, i0 = blockIdx.y * CT, t = blockIdx.z;
  const int cz = cdev ? min(cols, cdev[t]) : cols;   // columns past cz are taken as zero
  const cplx* x = X + t * sX;
  for (int r = threadIdx.x / CT; r < CT; r += 256 / CT) {
    const int i = i0 + r, j = j0 + (threadIdx.x % CT);
    cplx v = (i < rows && j < cz) ? x[(long long)i * ldx + j] : make_double2(0.0, 0.0);
    if (subI && i == j) v.x -= 1.0;
    tile[r * (CT + 1) + (threadIdx.x % CT)] = v;
  }
  __syncthreads();
  const int jj = threadIdx.x >> 2, ig = (threadIdx.x & 3) * 16, j = j0 + jj;
  if (j >= cols || i0 + ig >= rows) return;
  double nu2 = 0.0;
  if (j < cz) {
#pragma unroll
    for (int c = 0; c < 8; ++c) nu2 += part[((long long)c * T + t) * cols + j];
  }
  const int ex = scale_exp(nu2, beta);
  if (blockIdx.y == 0 && ig == 0) e[t * sE + j] = ex;
  Digits dr[16], di[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const cplx v = tile[(ig + k) * (CT + 1) + jj];
    dr[k] = digits_of(to_int(v.x, ex));
    di[k] = digits_of(to_int(v.y, ex));
  }
  const long long qstride = (long long)T * cols * ldr, pstride = (long long)S * qstride;
  col_store<S, NP>(dr, di, R + (long long)t * cols * ldr + (long long)j * ldr + i0 + ig, pstride, qstride);
}

template <int S, int Q = 0>
struct Crt {
  // accumulate sum_q frac(r_q ch_q) (exact) and sum_q r_q cl_q for the real and imaginary parts
  __device__ __forceinline__ static void run(const uint8_t* P, long long qstride, long long pstride, int flags,
                                             double (&sr)[4], double (&lr)[4], double (&si)[4], double (&li)[4]) {
    if constexpr (Q < S) {
      constexpr int m = OZM(Q);
      const uchar4 p1 = *reinterpret_cast<const uchar4*>(P + Q * qstride);
      const uchar4 p2 = *reinterpret_cast<const uchar4*>(P + pstride + Q * qstride);
      const uchar4 p3 = *reinterpret_cast<const uchar4*>(P + 2 * pstride + Q * qstride);
      const int a1[4] = {p1.x, p1.y, p1.z, p1.w}, a2[4] = {p2.x, p2.y, p2.z, p2.w}, a3[4] = {p3.x, p3.y, p3.z, p3.w};
      const double ch = c_ch[S][Q], cl = c_cl[S][Q];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int re, im;
        if (flags & OZ_NEG_P2) {
          re = a1[k] + a2[k];
          im = a3[k] - a1[k] + a2[k] + m;
        } else {
          re = a1[k] - a2[k] + m;
          im = a3[k] - a1[k] - a2[k] + 2 * m;
        }
        re %= m;
        im %= m;
        double tr = (double)re * ch, ti = (double)im * ch;
        tr -= rint(tr);
        ti -= rint(ti);
        sr[k] += tr;
        si[k] += ti;
        lr[k] = fma((double)re, cl, lr[k]);
        li[k] = fma((double)im, cl, li[k]);
      }
      Crt<S, Q + 1>::run(P, qstride, pstride, flags, sr, lr, si, li);
    }
  }
};

__device__ __forceinline__ double crt_value(double s, double l, double M) {
  double f = s - rint(s);   // exact
  f += l;
  f -= rint(f);
  return f * M;
}

template <int S>
__global__ void __launch_bounds__(128) oz_combine_kernel(const uint8_t* __restrict__ P, long long ldp, int M, int N,
                                                         int T, const int* __restrict__ eA, long long sEA, int a_traj,
                                                         const int* __restrict__ eB, long long sEB, int flags, cplx* C,
                                                         long long ldc, long long sC, const cplx* base,
                                                         const int32_t* gate, const int32_t* ndev) {
  if (gate && *gate == 0) return;
  const int i = blockIdx.y, t = blockIdx.z;
  const int j0 = (blockIdx.x * 128 + threadIdx.x) * 4;
  if (ndev) N = min(N, ndev[t]);
  if (j0 >= N) return;
  if ((flags & OZ_UPPER) && j0 + 3 < i) return;
  const long long qstride = (long long)T * M * ldp, pstride = (long long)S * qstride;
  const uint8_t* p = P + ((long long)t * M + i) * ldp + j0;
  double sr[4] = {0, 0, 0, 0}, lr[4] = {0, 0, 0, 0}, si[4] = {0, 0, 0, 0}, li[4] = {0, 0, 0, 0};
  Crt<S>::run(p, qstride, pstride, flags, sr, lr, si, li);
  const double Md = c_M[S];
  const int ea = eA[(a_traj ? t : 0) * sEA + i];
  cplx* c = C + t * sC + (long long)i * ldc;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = j0 + k;
    if (j >= N || ((flags & OZ_UPPER) && j < i)) continue;
    const int sc = -(ea + eB[t * sEB + j]);
    double2 v = make_double2(scalbn(crt_value(sr[k], lr[k], Md), sc), scalbn(crt_value(si[k], li[k], Md), sc));
    if (flags & OZ_NEGATE) {
      v.x = -v.x;
      v.y = -v.y;
    }
    if (base) {
      const double2 o = base[t * sC + (long long)i * ldc + j];
      v.x += o.x;
      v.y += o.y;
    } else if (flags & OZ_ACCUMULATE) {
      const double2 o = c[j];
      v.x += o.x;
      v.y += o.y;
    }
    c[j] = v;
  }
}

template <template <int> class F, typename... A>
int dispatch_s(int s, A... args) {
  switch (s) {
    case 4: return F<4>::go(args...);
    case 6: return F<6>::go(args...);
    case 8: return F<8>::go(args...);
    case 10: return F<10>::go(args...);
    case 12: return F<12>::go(args...);
    case 14: return F<14>::go(args...);
    case 16: return F<16>::go(args...);
  }
  return 1;
}

template <int S>
struct LaunchRows {
  static int go(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T, int conj,
                int8_t* R, long long ldr, int* e, long long sE, int beta, const int32_t* gate, const int32_t* cdev,
                int np) {
    if (np == 4)
      oz_split_rows_kernel<S, 4><<<dim3(rows, T), 256, 0, st>>>(X, ldx, sX, rows, cols, T, conj, R, ldr, e, sE, beta,
                                                                gate, cdev);
    else
      oz_split_rows_kernel<S, 3><<<dim3(rows, T), 256, 0, st>>>(X, ldx, sX, rows, cols, T, conj, R, ldr, e, sE, beta,
                                                                gate, cdev);
    return 0;
  }
};

template <int S>
struct LaunchCols {
  static int go(cudaStream_t st, int np, const cplx* X, long long ldx, long long sX, int rows, int cols, int T,
                int8_t* R, long long ldr, int* e, long long sE, const double* part, int beta, int subI,
                const int32_t* gate, const int32_t* cdev) {
    const int smem = CT * (CT + 1) * 16;
    dim3 grid(ceil_div(cols, CT), ceil_div(rows, CT), T);
    if (np == 4) {
      if (ensure_smem((const void*)oz_split_cols_kernel<S, 4>, smem) != cudaSuccess) return 4;
      oz_split_cols_kernel<S, 4><<<grid, 256, smem, st>>>(X, ldx, sX, rows, cols, T, R, ldr, e, sE, part, beta, subI,
                                                          gate, cdev);
    } else {
      if (ensure_smem((const void*)oz_split_cols_kernel<S, 3>, smem) != cudaSuccess) return 4;
      oz_split_cols_kernel<S, 3><<<grid, 256, smem, st>>>(X, ldx, sX, rows, cols, T, R, ldr, e, sE, part, beta, subI,
                                                          gate, cdev);
    }
    return 0;
  }
};

template <int S>
struct LaunchCombine {
  static int go(cudaStream_t st, const OzProduct& p) {
    dim3 grid(ceil_div(p.N, 512), p.M, p.T);
    oz_combine_kernel<S><<<grid, 128, 0, st>>>(p.RC, oz_ld(p.N), p.M, p.N, p.T, p.eA, p.sEA, p.a_traj, p.eB, p.sEB,
                                               p.flags, p.C, p.ldc, p.sC, p.base, p.gate, p.ndev);
    return 0;
  }
};

int launched(const char* what, std::string* err) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (err) *err = std::string(what) + ": " + cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

}  // namespace

int oz_supported(int s) { return s >= 4 && s <= 16 && s % 2 == 0; }
int oz_beta(int s) { return oz_supported(s) ? host_const().beta[s] : 0; }

int oz_split_rows(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T, int conj,
                  int s, int8_t* R, int* e, long long sE, std::string* err, const int32_t* gate, const int32_t* cdev,
                  int nplanes) {
  if (rows <= 0 || cols <= 0 || T <= 0) return 0;
  const int* md;
  if (!oz_supported(s) || rows >= 65536 * 32 || T > 65535) {
    if (err) *err = "oz_split_rows: unsupported modulus count or shape";
    return 1;
  }
  if (int r = ensure_device_constants(&md, err)) return r;
  if (nplanes != 3 && nplanes != 4) {
    if (err) *err = "oz_split_rows: 3 or 4 planes";
    return 1;
  }
  dispatch_s<LaunchRows>(s, st, X, ldx, sX, rows, cols, T, conj, R, oz_ld(cols), e, sE, oz_beta(s), gate, cdev, nplanes);
  return launched("oz_split_rows", err);
}

int oz_split_cols(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T, int nplanes,
                  int s, int8_t* R, int* e, long long sE, double* part, std::string* err, int sub_identity,
                  const int32_t* gate, const int32_t* cdev) {
  if (rows <= 0 || cols <= 0 || T <= 0) return 0;
  const int* md;
  if (!oz_supported(s) || (nplanes != 3 && nplanes != 4) || T > 65535 || ceil_div(rows, CT) > 65535) {
    if (err) *err = "oz_split_cols: unsupported modulus count, plane count or shape";
    return 1;
  }
  if (int r = ensure_device_constants(&md, err)) return r;
  oz_colnorm_kernel<<<dim3(ceil_div(cols, 32), 8, T), dim3(32, 8), 0, st>>>(X, ldx, sX, rows, cols, T, part,
                                                                            sub_identity, gate);
  if (int r = launched("oz_colnorm", err)) return r;
  if (dispatch_s<LaunchCols>(s, st, nplanes, X, ldx, sX, rows, cols, T, R, oz_ld(rows), e, sE, part, oz_beta(s),
                             sub_identity, gate, cdev)) {
    if (err) *err = "oz_split_cols: shared memory attribute";
    return 4;
  }
  return launched("oz_split_cols", err);
}

int oz_product(cudaStream_t st, const OzProduct& p, std::string* err) {
  if (int r = oz_product_mma(st, p, err)) return r;
  return oz_product_combine(st, p, err);
}

int oz_product_combine(cudaStream_t st, const OzProduct& p, std::string* err) {
  if (p.M <= 0 || p.N <= 0 || p.T <= 0) return 0;
  dispatch_s<LaunchCombine>(p.s, st, p);
  return launched("oz_combine", err);
}

int oz_product_mma(cudaStream_t st, const OzProduct& p, std::string* err) {
  if (p.M <= 0 || p.N <= 0 || p.T <= 0) return 0;
  const int* md;
  if (!oz_supported(p.s) || p.K <= 0 || p.M > 65535 * 8 || p.T > 65535) {
    if (err) *err = "oz_product: unsupported modulus count or shape";
    return 1;
  }
  if (int r = ensure_device_constants(&md, err)) return r;
  if (p.M > 65535) {
    if (err) *err = "oz_product: M > 65535";
    return 1;
  }
  IgemmArgs g;
  g.M = p.M;
  g.N = p.N;
  g.K = p.K;
  g.batch = 3LL * p.s * p.T;
  g.A = p.RA;
  g.lda = oz_ld(p.K);
  g.strideA = (long long)p.M * g.lda;
  g.B = p.RB;
  g.ldb = oz_ld(p.K);
  g.strideB = (long long)p.N * g.ldb;
  g.C = p.RC;
  g.ldc = oz_ld(p.N);
  g.strideC = (long long)p.M * g.ldc;
  g.out = IG_OUT_MOD;
  g.moduli = md;
  g.flags = ((p.flags & OZ_UPPER) ? IG_UPPER : 0) | ((p.flags & OZ_TRI_B) ? IG_TRI_B : 0);
  g.oz_s = p.s;
  g.oz_T = p.T;
  for (int i = 0; i < 3; ++i) {
    g.oz_pa[i] = p.pa[i];
    g.oz_pb[i] = p.pb[i];
  }
  g.oz_a_traj = p.a_traj;
  g.oz_b_traj = 1;
  g.oz_na = p.a_planes * p.s * (p.a_traj ? p.T : 1);
  g.oz_nb = p.b_planes * p.s * p.T;
  g.gate = p.gate;
  g.kdev = p.kdev;
  g.ndev = p.ndev;
  return igemm(st, g, err);
}

}  // namespace traj
