// Exact modular complex-FP64 products on the INT8 tensor cores (Ozaki-II / CRT; see ozaki.h).
#include "ozaki.h"
#include "igemm.h"
#include <algorithm>
#include <map>
#include <mutex>
#include <set>

namespace traj {
namespace {

// pairwise coprime odd moduli <= 256 (the first s are used) whose prime factors are all = 1 (mod 4), so
// that -1 is a square mod each of them (221 = 13 17, 205 = 5 41, the rest prime); residues are stored
// in [-128, 127]
__host__ __device__ constexpr int OZM(int q) {
  return q == 0 ? 241 : q == 1 ? 233 : q == 2 ? 229 : q == 3 ? 221 : q == 4 ? 205 : q == 5 ? 197 : q == 6 ? 193
       : q == 7 ? 181 : q == 8 ? 173 : q == 9 ? 157 : q == 10 ? 149 : q == 11 ? 137 : q == 12 ? 113
       : q == 13 ? 109 : q == 14 ? 101 : q == 15 ? 97 : q == 16 ? 89 : 73;
}
// the smallest j with j^2 = -1 (mod m)
__host__ __device__ constexpr int sqrt_minus_one(int m) {
  for (int x = 1; x < m; ++x)
    if (x * x % m == m - 1) return x;
  return 0;
}
__host__ __device__ constexpr int OZJ(int q) { return sqrt_minus_one(OZM(q)); }
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
    for (int s = 1; s <= OZ_MAXS; ++s) {
      // M as a double (the product in 64-bit-mantissa long double, rounded once) and floor(log2(M))
      long double Ml = 1.0L;
      for (int q = 0; q < s; ++q) Ml *= (long double)OZM(q);
      M[s] = (double)Ml;
      int lg = 0;
      {
        long double x = Ml;
        while (x >= 2.0L) {
          x *= 0.5L;
          ++lg;
        }
      }
      // both sides below 2^beta keep |2 Re|, |2 Im| (the combine reconstructs twice the product)
      // below 2^(2 beta + 1) <= 2^(lg - 1) <= M / 2; the 21-bit digit split of the operands needs
      // |x| < 2^62
      beta[s] = std::min(lg / 2 - 1, 61);
      // the moduli in pairs (q = 2p, 2p + 1), mu_p = m_2p m_2p+1 < 2^16 (s even); c_p = inv_p / mu_p,
      // inv_p = (M / mu_p)^-1 mod mu_p; n = round(inv_p 2^36 / mu_p), ch = n 2^-36, cl = c_p - ch (the
      // representatives r < 2^16 + 768 keep every r ch exact in 53 bits)
      for (int q = 0; 2 * q + 1 < s; ++q) {
        const long long mu = (long long)OZM(2 * q) * OZM(2 * q + 1);
        long long Mi = 1;   // (M / mu) mod mu
        for (int r = 0; r < s; ++r)
          if (r != 2 * q && r != 2 * q + 1) Mi = Mi * OZM(r) % mu;
        long long inv = 0;
        {   // extended Euclid
          long long r0 = mu, r1 = Mi, t0 = 0, t1 = 1;
          while (r1) {
            const long long k = r0 / r1;
            long long tmp = r0 - k * r1;
            r0 = r1;
            r1 = tmp;
            tmp = t0 - k * t1;
            t0 = t1;
            t1 = tmp;
          }
          inv = ((t0 % mu) + mu) % mu;
        }
        const long long num = inv << 36;
        const long long n = (num + mu / 2) / mu;
        ch[s][q] = (double)n * 0x1p-36;
        cl[s][q] = (double)(num - n * mu) / (double)mu * 0x1p-36;
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

// exponent e with nu 2^e < 2^beta (nu = the row's / column's 2-norm of |re| + |im|); 0 for a zero row;
// OZ_NONFINITE for a row holding a NaN or an infinity: its residues are written as zeros and the combine
// returns NaN for every output it meets (as an FP64 product would), so a failed trajectory stays failed
constexpr int OZ_NONFINITE = 1 << 20;
__device__ __forceinline__ int scale_exp(double nu2, int beta) {
  if (!(nu2 <= 1.7e308)) return OZ_NONFINITE;   // NaN or infinite
  if (!(nu2 > 0.0)) return 0;
  return beta - ilogb(sqrt(nu2)) - 1;
}

// v 2^e rounded to an integer (|v 2^e| < 2^62 by the choice of e); the power of two is built
// directly unless it leaves the normal range
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
__device__ __forceinline__ long long to_int(double v, int e, double p2) {
  if (e == OZ_NONFINITE) return 0;
  return __double2ll_rn((e > -1000 && e < 1000) ? v * p2 : scalbn(v, e));
}

// x (|x| < 2^62) by the eight bytes of x + 2^62 >= 0 (two words: no digit extraction)
struct Dig {
  uint32_t lo, hi;
};
__device__ __forceinline__ Dig dig_of(long long x) {
  const unsigned long long u = (unsigned long long)x + (1ull << 62);
  return Dig{(uint32_t)u, (uint32_t)(u >> 32)};
}
// one reduction step of v in [0, k m): v <- v - m when v >= m (unsigned wrap-around makes it a min)
__device__ __forceinline__ uint32_t red1(uint32_t v, uint32_t m) { return min(v, v - m); }

// bytes (256^k c mod m) for k = k0 .. k0 + 3, packed for dp4a
__host__ __device__ constexpr uint32_t pow256_word(int k0, uint32_t c, uint32_t m) {
  uint32_t w = 0;
  for (int k = 0; k < 4; ++k) w |= (uint32_t)((unsigned long long)pow2mod(8 * (k0 + k), (int)m) * c % m) << (8 * k);
  return w;
}

// The residues of z+ = re + j im and z- = re - j im mod m_Q straight from the bytes b_k of re + 2^62 and
// im + 2^62: R = sum_k b_k (256^k mod m) -- two dp4a -- is congruent to re + 2^62, I = sum_k b_k
// (256^k j mod m) to j (im + 2^62), both <= 8 255 (m - 1) < 2^19, so
//   (z+ + 128) mod m = (R + I + offP) mod m,   (z- + 128) mod m = (R + (KM - I) + offM) mod m
// with KM the least multiple of m >= 8 255 (m - 1) and the offsets removing the 2^62 shifts.  Every sum S is
// below 2^21, where floor(S / m) = umulhi(S, ceil(2^32 / m)) exactly (S (ceil(2^32 / m) m - 2^32) < 2^32):
// one multiply-high and one multiply-subtract per plane.
template <int Q>
struct Mod {
  static constexpr uint32_t m = OZM(Q);
  static constexpr uint32_t j = OZJ(Q);   // j^2 = -1 (mod m)
  static constexpr uint32_t p62 = pow2mod(62, m);
  static constexpr uint32_t cr0 = pow256_word(0, 1, m), cr1 = pow256_word(4, 1, m);
  static constexpr uint32_t ci0 = pow256_word(0, j, m), ci1 = pow256_word(4, j, m);
  static constexpr uint32_t offP = (128 % m + 2 * m * m - p62 * (1 + j)) % m;   // 128 - 2^62 (1 + j)
  static constexpr uint32_t offM = (128 + m - p62 + p62 * j) % m;               // 128 - 2^62 (1 - j)
  static constexpr uint32_t KM = m * ((8u * 255u * (m - 1) + m - 1) / m);
  static constexpr uint32_t magic = (uint32_t)((0x100000000ull + m - 1) / m);
  static_assert(8ull * 255 * (m - 1) + KM + 2 * m < (1ull << 21), "sums stay below 2^21");
  static_assert((unsigned long long)(1u << 21) * ((unsigned long long)magic * m - 0x100000000ull) < 0x100000000ull,
                "the multiply-high quotient is exact below 2^21");
  __device__ __forceinline__ static uint32_t mod(uint32_t v) { return v - __umulhi(v, magic) * m; }
  __device__ __forceinline__ static void planes(const Dig& dr, const Dig& di, uint32_t& zp, uint32_t& zm) {
    const uint32_t R = __dp4a(dr.hi, cr1, __dp4a(dr.lo, cr0, 0u));
    const uint32_t I = __dp4a(di.hi, ci1, __dp4a(di.lo, ci0, 0u));
    zp = mod(R + I + offP);
    zm = mod(R + (KM - I) + offM);
  }
};

__device__ __forceinline__ uint32_t pack4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410) ^ 0x80808080u;
}

// residues of the two planes z+ = re + j im and z- = re - j im (the images of re + i im under the two
// ring homomorphisms Z[i] -> Z_m, i -> +-j) of E consecutive elements, packed 4 per word; the stored
// int8 is ((z + 128) mod m) - 128, a residue of z in [-128, 127], i.e. the byte ((z + 128) mod m) ^ 0x80
template <int Q, int E>
__device__ __forceinline__ void plane_words(const Dig (&dr)[E], const Dig (&di)[E], uint32_t (&w)[2][E / 4]) {
#pragma unroll
  for (int g = 0; g < E / 4; ++g) {
    uint32_t b[2][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) Mod<Q>::planes(dr[4 * g + k], di[4 * g + k], b[0][k], b[1][k]);
#pragma unroll
    for (int p = 0; p < 2; ++p) w[p][g] = pack4(b[p][0], b[p][1], b[p][2], b[p][3]);
  }
}

template <int S, int Q = 0>
struct RowStore {
  // 4 consecutive elements -> one 32-bit word per (plane, modulus)
  __device__ __forceinline__ static void run(const Dig (&dr)[4], const Dig (&di)[4], int8_t* R, long long pstride,
                                             long long qstride) {
    if constexpr (Q < S) {
      uint32_t w[2][1];
      plane_words<Q, 4>(dr, di, w);
#pragma unroll
      for (int p = 0; p < 2; ++p) *reinterpret_cast<uint32_t*>(R + p * pstride + Q * qstride) = w[p][0];
      RowStore<S, Q + 1>::run(dr, di, R, pstride, qstride);
    }
  }
};

template <int S>
__global__ void __launch_bounds__(256) oz_split_rows_kernel(const cplx* __restrict__ X, long long ldx, long long sX,
                                                            int rows, int cols_cap, int T, int conj, int8_t* R,
                                                            long long ldr, int* e, long long sE, int beta,
                                                            const int32_t* gate, const int32_t* cdev,
                                                            const int32_t* rdev) {
  if (gate && *gate == 0) return;
  const int row = blockIdx.x, t = blockIdx.y;
  const cplx* x = X + t * sX + (long long)row * ldx;
  // past cdev (columns) or rdev (rows): zero residues
  const int cols = (rdev && row >= rdev[t]) ? 0 : (cdev ? min(cols_cap, cdev[t]) : cols_cap);
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
  const double p2 = pow2(ex);
  const long long qstride = (long long)T * rows * ldr, pstride = (long long)S * qstride;
  int8_t* Rrow = R + (long long)t * rows * ldr + (long long)row * ldr;
  for (int j0 = 4 * threadIdx.x; j0 < cols_cap; j0 += 1024) {
    Dig dr[4], di[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      long long vr = 0, vi = 0;
      if (j0 + k < cols) {
        const cplx v = x[j0 + k];
        vr = to_int(v.x, ex, p2);
        vi = to_int(v.y, ex, p2);
        if (conj) vi = -vi;
      }
      dr[k] = dig_of(vr);
      di[k] = dig_of(vi);
    }
    RowStore<S>::run(dr, di, Rrow + j0, pstride, qstride);
  }
}

// per-column partial sums of (|re| + |im|)^2 over 8 row chunks: part[(c T + t) cols + j]
__global__ void __launch_bounds__(256) oz_colnorm_kernel(const cplx* __restrict__ X, long long ldx, long long sX,
                                                         int rows, int cols, int T, double* part, int subI,
                                                         const int32_t* gate, const int32_t* rdev) {
  if (gate && *gate == 0) return;
  const int j = blockIdx.x * 32 + threadIdx.x, c = blockIdx.y, t = blockIdx.z;
  const int rz = rdev ? min(rows, rdev[t]) : rows;
  const int per = (rows + 7) / 8, r0 = c * per, r1 = min(rz, r0 + per);
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

constexpr int CTI = 64, CTJ = 32;   // column-split tile: 64 rows (k) x 32 columns (residue rows) of X

template <int S, int Q = 0>
struct ColStore {
  // 8 consecutive k of one residue row -> one 8-byte store per (plane, modulus)
  __device__ __forceinline__ static void run(const Dig (&dr)[8], const Dig (&di)[8], int8_t* R, long long pstride,
                                             long long qstride) {
    if constexpr (Q < S) {
      uint32_t w[2][2];
      plane_words<Q, 8>(dr, di, w);
#pragma unroll
      for (int p = 0; p < 2; ++p) *reinterpret_cast<uint2*>(R + p * pstride + Q * qstride) = make_uint2(w[p][0], w[p][1]);
      ColStore<S, Q + 1>::run(dr, di, R, pstride, qstride);
    }
  }
};

template <int S>
__global__ void __launch_bounds__(256) oz_split_cols_kernel(const cplx* __restrict__ X, long long ldx, long long sX,
                                                            int rows, int cols, int T, int8_t* R, long long ldr,
                                                            int* e, long long sE, const double* part, int beta,
                                                            int subI, const int32_t* gate, const int32_t* cdev,
                                                            const int32_t* rdev, const int* e_in) {
  if (gate && *gate == 0) return;
  // column index rotated by the row group (ii >> 3): the 8 threads of a 128-bit load phase (same column, rows 8
  // apart) then fall into 8 different bank groups
  __shared__ cplx tile[CTI][CTJ];
  const int j0 = blockIdx.x * CTJ, i0 = blockIdx.y * CTI, t = blockIdx.z;
  const int cz = cdev ? min(cols, cdev[t]) : cols;   // columns past cz are taken as zero
  const int rz = rdev ? min(rows, rdev[t]) : rows;   // rows past rz too
  const cplx* x = X + t * sX;
#pragma unroll
  for (int r = 0; r < CTI * CTJ / 256; ++r) {
    const int el = threadIdx.x + 256 * r, ii = el / CTJ, jj = el % CTJ;
    const int i = i0 + ii, j = j0 + jj;
    cplx v = (i < rz && j < cz) ? x[(long long)i * ldx + j] : make_double2(0.0, 0.0);
    if (subI && i == j) v.x -= 1.0;
    tile[ii][(jj + (ii >> 3)) & (CTJ - 1)] = v;
  }
  __syncthreads();
  const int jj = threadIdx.x >> 3, ig = (threadIdx.x & 7) * 8, j = j0 + jj;
  if (j >= cols || i0 + ig >= rows) return;
  int ex;
  if (e_in) {
    ex = e_in[t * sE + j];
  } else {
    double nu2 = 0.0;
    if (j < cz) {
#pragma unroll
      for (int c = 0; c < 8; ++c) nu2 += part[((long long)c * T + t) * cols + j];
    }
    ex = scale_exp(nu2, beta);
    if (blockIdx.y == 0 && ig == 0) e[t * sE + j] = ex;
  }
  const double p2 = pow2(ex);
  Dig dr[8], di[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const cplx v = tile[ig + k][(jj + (ig >> 3)) & (CTJ - 1)];
    dr[k] = dig_of(to_int(v.x, ex, p2));
    di[k] = dig_of(to_int(v.y, ex, p2));
  }
  const long long qstride = (long long)T * cols * ldr, pstride = (long long)S * qstride;
  ColStore<S>::run(dr, di, R + (long long)t * cols * ldr + (long long)j * ldr + i0 + ig, pstride, qstride);
}

// ---- CRT combine.  Moduli are taken in pairs (m_a, m_b) -> one residue mod mu = m_a m_b < 2^16
// (Garner's step), then X / M = frac(sum_p r_p c_p) over the 8 pairs with c_p = ch_p + cl_p, ch_p a
// multiple of 2^-36: every r_p ch_p (r_p < 2^16) and the sum of their fractional parts are exact.
__host__ __device__ constexpr int modinv(int a, int m) {
  int r = 1;
  for (int x = 1; x < m; ++x)
    if ((a % m) * x % m == 1) r = x;
  return r;
}

// residues of twice the real and imaginary parts from the two product residues a+ = P+ mod m and
// a- = P- mod m (bytes < m; P+- = A+- B+-, the product's images under i -> +-j): 2 Re = P+ + P- is left
// unreduced in [0, 2m) (the Garner step below takes any non-negative representative); 2 Im =
// (P+ - P-) / j = -j (P+ - P-) takes one multiplication and one modulo
template <int Q>
__device__ __forceinline__ void reim(uint32_t ap, uint32_t am, uint32_t& re, uint32_t& im) {
  constexpr uint32_t m = OZM(Q), nj = OZM(Q) - OZJ(Q);
  re = ap + am;
  im = ((ap + m - am) * nj) % m;
}

// the residues of 4 consecutive outputs of one (product, modulus): with split-K, the chunks' residues
// summed and reduced mod m
template <int Q, bool KS1>
__device__ __forceinline__ void res4(const uint8_t* p, long long kstride, int ks, uint32_t (&v)[4]) {
  uchar4 a = *reinterpret_cast<const uchar4*>(p);
  v[0] = a.x;
  v[1] = a.y;
  v[2] = a.z;
  v[3] = a.w;
  if (!KS1 && ks > 1) {
    for (int c = 1; c < ks; ++c) {
      a = *reinterpret_cast<const uchar4*>(p + c * kstride);
      v[0] += a.x;
      v[1] += a.y;
      v[2] += a.z;
      v[3] += a.w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] %= (uint32_t)OZM(Q);
  }
}

__device__ __forceinline__ double u32_to_double(uint32_t r) {
  return __dadd_rn(__hiloint2double(0x43300000, (int)r), -4503599627370496.0);
}
__device__ __forceinline__ double round_magic(double x) {
  return __dadd_rn(__dadd_rn(x, 6755399441055744.0), -6755399441055744.0);
}

template <int S, bool KS1, int PQ = 0>
struct CrtPair {
  __device__ __forceinline__ static void run(const uint8_t* P, long long qstride, long long pstride, long long kstride,
                                             int ks, double (&sr)[4], double (&lr)[4], double (&si)[4],
                                             double (&li)[4]) {
    if constexpr (2 * PQ < S) {
      constexpr int QA = 2 * PQ, QB = 2 * PQ + 1;
      constexpr uint32_t ma = OZM(QA), mb = OZM(QB);
      constexpr uint32_t inv = (uint32_t)modinv((int)(ma % mb), (int)mb);   // m_a^-1 mod m_b
      uint32_t A1[4], A2[4], B1[4], B2[4];
      res4<QA, KS1>(P + QA * qstride, kstride, ks, A1);
      res4<QA, KS1>(P + pstride + QA * qstride, kstride, ks, A2);
      res4<QB, KS1>(P + QB * qstride, kstride, ks, B1);
      res4<QB, KS1>(P + pstride + QB * qstride, kstride, ks, B2);
      const double ch = c_ch[S][PQ], cl = c_cl[S][PQ];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t rea, ima, reb, imb;
        reim<QA>(A1[k], A2[k], rea, ima);
        reim<QB>(B1[k], B2[k], reb, imb);
        // Garner: r = r_a + m_a ((r_b - r_a) m_a^-1 mod m_b) in [0, mu + m_a) (r_a, r_b in [0, 2m)
        // unreduced, 2 m_a < 4 m_b for the adjacent moduli of a pair; one modulo per component), then one
        // step to the canonical residue in [0, mu): a zero
        // product must come out as exactly 0 (a zero row has exponent 0, so any CRT residual of a
        // non-canonical representative would be amplified)
        constexpr uint32_t mu = ma * mb;
        const uint32_t rr = red1(rea + ma * (((reb + 4 * mb - rea) * inv) % mb), mu);
        const uint32_t ri = red1(ima + ma * (((imb + 4 * mb - ima) * inv) % mb), mu);
        // (double)r and rint() without the conversion pipe: 2^52 + r is the double with r in its low
        // mantissa word, and x + 1.5 2^52 - 1.5 2^52 rounds |x| < 2^51 to the nearest-even integer
        const double dr = u32_to_double(rr), di = u32_to_double(ri);
        double tr = dr * ch, ti = di * ch;
        tr -= round_magic(tr);
        ti -= round_magic(ti);
        sr[k] += tr;
        si[k] += ti;
        lr[k] = fma(dr, cl, lr[k]);
        li[k] = fma(di, cl, li[k]);
      }
      CrtPair<S, KS1, PQ + 1>::run(P, qstride, pstride, kstride, ks, sr, lr, si, li);
    }
  }
};

__device__ __forceinline__ double crt_value(double s, double l, double M) {
  double f = s - rint(s);   // exact
  f += l;
  f -= rint(f);
  return f * M;
}

template <int S, bool KS1>
__global__ void __launch_bounds__(128) oz_combine_kernel(const uint8_t* __restrict__ P, long long ldp, int M, int N,
                                                         int T, const int* __restrict__ eA, long long sEA, int a_traj,
                                                         const int* __restrict__ eB, long long sEB, int flags, cplx* C,
                                                         long long ldc, long long sC, const cplx* base,
                                                         const int32_t* gate, const int32_t* ndev, int ks) {
  if (gate && *gate == 0) return;
  const int i = blockIdx.y, t = blockIdx.z;
  const int j0 = (blockIdx.x * 128 + threadIdx.x) * 4;
  if (ndev) N = min(N, ndev[t]);
  if (j0 >= N) return;
  if ((flags & OZ_UPPER) && j0 + 3 < i) return;
  const long long kstride = (long long)M * ldp, qstride = (long long)T * ks * kstride, pstride = (long long)S * qstride;
  const uint8_t* p = P + ((long long)t * ks * M + i) * ldp + j0;
  double sr[4] = {0, 0, 0, 0}, lr[4] = {0, 0, 0, 0}, si[4] = {0, 0, 0, 0}, li[4] = {0, 0, 0, 0};
  CrtPair<S, KS1>::run(p, qstride, pstride, kstride, ks, sr, lr, si, li);
  const double Md = c_M[S];
  const int ea = eA[(a_traj ? t : 0) * sEA + i];
  cplx* c = C + t * sC + (long long)i * ldc;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = j0 + k;
    if (j >= N || ((flags & OZ_UPPER) && j < i)) continue;
    const int eb = eB[t * sEB + j];
    const int sc = -(ea + eb) - 1;   // the CRT value is twice the product
    double2 v = make_double2(crt_value(sr[k], lr[k], Md), crt_value(si[k], li[k], Md));
    if (ea == OZ_NONFINITE || eb == OZ_NONFINITE) v = make_double2(__longlong_as_double(0x7ff8000000000000LL),
                                                                   __longlong_as_double(0x7ff8000000000000LL));
    if (sc > -1000 && sc < 1000) {
      const double f = pow2(sc);
      v.x *= f;
      v.y *= f;
    } else {
      v.x = scalbn(v.x, sc);
      v.y = scalbn(v.y, sc);
    }
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
    case 18: return F<18>::go(args...);
  }
  return 1;
}

template <int S>
struct LaunchRows {
  static int go(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T, int conj,
                int8_t* R, long long ldr, int* e, long long sE, int beta, const int32_t* gate, const int32_t* cdev,
                int np, const int32_t* rdev) {
    oz_split_rows_kernel<S><<<dim3(rows, T), 256, 0, st>>>(X, ldx, sX, rows, cols, T, conj, R, ldr, e, sE, beta, gate,
                                                           cdev, rdev);
    return 0;
  }
};

template <int S>
struct LaunchCols {
  static int go(cudaStream_t st, int np, const cplx* X, long long ldx, long long sX, int rows, int cols, int T,
                int8_t* R, long long ldr, int* e, long long sE, const double* part, int beta, int subI,
                const int32_t* gate, const int32_t* cdev, const int32_t* rdev, const int* e_in) {
    dim3 grid(ceil_div(cols, CTJ), ceil_div(rows, CTI), T);
    oz_split_cols_kernel<S><<<grid, 256, 0, st>>>(X, ldx, sX, rows, cols, T, R, ldr, e, sE, part, beta, subI, gate,
                                                  cdev, rdev, e_in);
    return 0;
  }
};

template <int S>
struct LaunchCombine {
  static int go(cudaStream_t st, const OzProduct& p) {
    dim3 grid(ceil_div(p.N, 512), p.M, p.T);
    if (p.ksplit > 1)
      oz_combine_kernel<S, false><<<grid, 128, 0, st>>>(p.RC, oz_ld(p.N), p.M, p.N, p.T, p.eA, p.sEA, p.a_traj, p.eB,
                                                        p.sEB, p.flags, p.C, p.ldc, p.sC, p.base, p.gate, p.ndev,
                                                        p.ksplit);
    else
      oz_combine_kernel<S, true><<<grid, 128, 0, st>>>(p.RC, oz_ld(p.N), p.M, p.N, p.T, p.eA, p.sEA, p.a_traj, p.eB,
                                                       p.sEB, p.flags, p.C, p.ldc, p.sC, p.base, p.gate, p.ndev, 1);
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

int oz_supported(int s) { return s >= 4 && s <= OZ_MAXS && s % 2 == 0; }

int oz_constants(int s, int* moduli, int* beta, double* ch, double* cl, double* M) {
  if (!oz_supported(s)) return 1;
  const HostConst& h = host_const();
  for (int q = 0; q < s; ++q) moduli[q] = OZM(q);
  *beta = h.beta[s];
  for (int p = 0; p < s / 2; ++p) {
    ch[p] = h.ch[s][p];
    cl[p] = h.cl[s][p];
  }
  *M = h.M[s];
  return 0;
}
int oz_beta(int s) { return oz_supported(s) ? host_const().beta[s] : 0; }
int oz_roots(int s, int* roots) {
  if (!oz_supported(s)) return 1;
  for (int q = 0; q < s; ++q) roots[q] = OZJ(q);
  return 0;
}

int oz_split_rows(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T, int conj,
                  int s, int8_t* R, int* e, long long sE, std::string* err, const int32_t* gate, const int32_t* cdev,
                  int nplanes, const int32_t* rdev) {
  if (rows <= 0 || cols <= 0 || T <= 0) return 0;
  const int* md;
  if (!oz_supported(s) || rows >= 65536 * 32 || T > 65535) {
    if (err) *err = "oz_split_rows: unsupported modulus count or shape";
    return 1;
  }
  if (int r = ensure_device_constants(&md, err)) return r;
  dispatch_s<LaunchRows>(s, st, X, ldx, sX, rows, cols, T, conj, R, oz_ld(cols), e, sE, oz_beta(s), gate, cdev, nplanes,
                         rdev);
  return launched("oz_split_rows", err);
}

int oz_split_cols(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T, int nplanes,
                  int s, int8_t* R, int* e, long long sE, double* part, std::string* err, int sub_identity,
                  const int32_t* gate, const int32_t* cdev, const int32_t* rdev) {
  if (rows <= 0 || cols <= 0 || T <= 0) return 0;
  const int* md;
  if (!oz_supported(s) || T > 65535 || ceil_div(rows, CTI) > 65535) {
    if (err) *err = "oz_split_cols: unsupported modulus count, plane count or shape";
    return 1;
  }
  if (int r = ensure_device_constants(&md, err)) return r;
  oz_colnorm_kernel<<<dim3(ceil_div(cols, 32), 8, T), dim3(32, 8), 0, st>>>(X, ldx, sX, rows, cols, T, part,
                                                                            sub_identity, gate, rdev);
  if (int r = launched("oz_colnorm", err)) return r;
  if (dispatch_s<LaunchCols>(s, st, nplanes, X, ldx, sX, rows, cols, T, R, oz_ld(rows), e, sE, part, oz_beta(s),
                             sub_identity, gate, cdev, rdev, nullptr)) {
    if (err) *err = "oz_split_cols: shared memory attribute";
    return 4;
  }
  return launched("oz_split_cols", err);
}

namespace {
__global__ void oz_colsum_kernel(const double* __restrict__ part, int cols, int T, double* nu2, long long sN, int acc) {
  const int j = blockIdx.x * 256 + threadIdx.x, t = blockIdx.y;
  if (j >= cols) return;
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += part[((long long)c * T + t) * cols + j];
  nu2[t * sN + j] = acc ? nu2[t * sN + j] + s : s;
}
__global__ void oz_exponents_kernel(const double* __restrict__ nu2, long long sN, int cols, int beta, int* e,
                                    long long sE) {
  const int j = blockIdx.x * 256 + threadIdx.x, t = blockIdx.y;
  if (j < cols) e[t * sE + j] = scale_exp(nu2[t * sN + j], beta);
}
}  // namespace

int oz_colnorm_accumulate(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T,
                          double* part, double* nu2, long long sN, int accumulate, std::string* err,
                          int sub_identity) {
  if (cols <= 0 || T <= 0) return 0;
  oz_colnorm_kernel<<<dim3(ceil_div(cols, 32), 8, T), dim3(32, 8), 0, st>>>(X, ldx, sX, rows, cols, T, part,
                                                                            sub_identity, nullptr, nullptr);
  if (int r = launched("oz_colnorm", err)) return r;
  oz_colsum_kernel<<<dim3(ceil_div(cols, 256), T), 256, 0, st>>>(part, cols, T, nu2, sN, accumulate);
  return launched("oz_colsum", err);
}

namespace {
// gate[1] = !gate[0] && max nu2 <= thr2, gate[2] = !gate[0] && !(max nu2 <= thr2); a NaN (failed
// trajectory) does not raise the tier
__global__ void __launch_bounds__(1024) oz_tier_decide_kernel(const double* __restrict__ nu2, long long n, double thr2,
                                                               int32_t* gate) {
  __shared__ int over;
  if (threadIdx.x == 0) over = 0;
  __syncthreads();
  int o = 0;
  for (long long i = threadIdx.x; i < n; i += 1024) o |= nu2[i] > thr2;
  if (o) over = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int full = gate[0];
    gate[1] = !full && !over;
    gate[2] = !full && over;
  }
}
}  // namespace

int oz_tier_decide(cudaStream_t st, const double* nu2, long long n, double thr2, int32_t* gate, std::string* err) {
  oz_tier_decide_kernel<<<1, 1024, 0, st>>>(nu2, n, thr2, gate);
  return launched("oz_tier_decide", err);
}

int oz_exponents(cudaStream_t st, const double* nu2, long long sN, int cols, int T, int s, int* e, long long sE,
                 std::string* err) {
  if (cols <= 0 || T <= 0) return 0;
  if (!oz_supported(s)) {
    if (err) *err = "oz_exponents: unsupported modulus count";
    return 1;
  }
  oz_exponents_kernel<<<dim3(ceil_div(cols, 256), T), 256, 0, st>>>(nu2, sN, cols, oz_beta(s), e, sE);
  return launched("oz_exponents", err);
}

int oz_split_cols_e(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T,
                    int nplanes, int s, int8_t* R, const int* e_in, long long sE, std::string* err) {
  if (rows <= 0 || cols <= 0 || T <= 0) return 0;
  const int* md;
  if (!oz_supported(s) || !e_in) {
    if (err) *err = "oz_split_cols_e: unsupported modulus / plane count or no exponents";
    return 1;
  }
  if (int r = ensure_device_constants(&md, err)) return r;
  if (dispatch_s<LaunchCols>(s, st, nplanes, X, ldx, sX, rows, cols, T, R, oz_ld(rows), nullptr, sE, nullptr,
                             oz_beta(s), 0, nullptr, nullptr, nullptr, e_in)) {
    if (err) *err = "oz_split_cols_e: launch";
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
  // a conjugated operand (the callers' pa[2] / pb[2] == 3, the 3M scheme's (re - im) plane) swaps its two
  // planes: conj(z)+- = z-+
  const int ca = p.pa[2] == 3 ? 1 : 0, cb = p.pb[2] == 3 ? 1 : 0;
  g.oz_np = 2;
  g.batch = 2LL * p.s * p.T;
  g.A = p.RA;
  g.lda = p.lda_override ? p.lda_override : oz_ld(p.K);
  g.strideA = (long long)p.M * g.lda;
  g.B = p.RB;
  g.ldb = oz_ld(p.K);
  g.strideB = (long long)p.N * g.ldb;
  g.C = p.RC;
  g.ldc = oz_ld(p.N);
  g.strideC = (long long)p.M * g.ldc;
  g.out = p.mma_accumulate ? IG_OUT_MOD_ACC : IG_OUT_MOD;
  g.moduli = md;
  g.flags = ((p.flags & OZ_UPPER) ? IG_UPPER : 0) | ((p.flags & OZ_TRI_B) ? IG_TRI_B : 0);
  g.oz_s = p.s;
  g.oz_T = p.T;
  g.oz_pa[0] = ca;
  g.oz_pa[1] = 1 - ca;
  g.oz_pb[0] = cb;
  g.oz_pb[1] = 1 - cb;
  g.oz_pa[2] = g.oz_pb[2] = 0;
  g.oz_a_traj = p.a_traj;
  g.oz_b_traj = 1;
  g.oz_na = 2LL * p.s * (p.a_traj ? p.T : 1);
  g.oz_nb = 2LL * p.s * p.T;
  g.gate = p.gate;
  g.kdev = p.kdev;
  g.ndev = p.ndev;
  g.ksplit = std::max(1, p.ksplit);
  return igemm(st, g, err);
}

}  // namespace traj
