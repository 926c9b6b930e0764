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

// Strassen's algorithm on every real product of the planar 3M propagator, LV = 1, 2 or 3 levels.  With
// A = K's plane q and B = U's plane q in 2 x 2 blocks:
//   M1 = (A11 + A22)(B11 + B22)  M2 = (A21 + A22) B11  M3 = A11 (B12 - B22)  M4 = A22 (B21 - B11)
//   M5 = (A11 + A12) B22         M6 = (A21 - A11)(B11 + B12)             M7 = (A12 - A22)(B21 + B22)
//   C11 = M1 + M4 - M5 + M7,  C12 = M3 + M5,  C21 = M2 + M4,  C22 = M1 - M2 + M3 + M6
// -- seven half-size products instead of eight; applied again to each of the seven (LV = 2), 49
// quarter-size products instead of 64; once more (LV = 3), 343 eighth-size products instead of 512.  The operand / recombination coefficients over the 2 x 2
// blocks (11, 12, 21, 22) are the tables below; one thread handles one element of the leaf grid and
// all 2^LV x 2^LV positions it stands for, so each pass reads and writes every matrix once.  K's
// operands are formed once (strassen_k), U's per step (strassen_b), the leaf products are
// recombined together with the complex 3M recombination in one pass (strassen_c).
__constant__ int8_t kSA[7][4] = {{1, 0, 0, 1}, {0, 0, 1, 1}, {1, 0, 0, 0}, {0, 0, 0, 1},
                                 {1, 1, 0, 0}, {-1, 0, 1, 0}, {0, 1, 0, -1}};
__constant__ int8_t kSB[7][4] = {{1, 0, 0, 1}, {1, 0, 0, 0}, {0, 1, 0, -1}, {-1, 0, 1, 0},
                                 {0, 0, 0, 1}, {1, 1, 0, 0}, {0, 0, 1, 1}};
__constant__ int8_t kSC[4][7] = {{1, 0, 0, 1, -1, 0, 1}, {0, 0, 1, 0, 1, 0, 0},
                                 {0, 1, 0, 1, 0, 0, 0}, {1, -1, 1, 0, 0, 1, 0}};

template <int LV>
struct P7 {
  static constexpr int v = 7 * P7<LV - 1>::v;
};
template <>
struct P7<0> {
  static constexpr int v = 1;
};

// the 7^LV operands of a matrix given on its 2^LV x 2^LV grid of leaf blocks x[R][C] (one element each):
// operand s1 of the top split over the four half-blocks, then recursively its 7^(LV-1) operands
template <int LV>
struct StrassenOps {
  static __device__ __forceinline__ void run(const double (&x)[1 << LV][1 << LV], const int8_t (&co)[7][4],
                                             double* out, long long bs) {
    constexpr int H = 1 << (LV - 1);
#pragma unroll
    for (int s = 0; s < 7; ++s) {
      double h[H][H];
#pragma unroll
      for (int r = 0; r < H; ++r)
#pragma unroll
        for (int c = 0; c < H; ++c)
          h[r][c] = co[s][0] * x[r][c] + co[s][1] * x[r][H + c] + co[s][2] * x[H + r][c] + co[s][3] * x[H + r][H + c];
      StrassenOps<LV - 1>::run(h, co, out + (long long)s * P7<LV - 1>::v * bs, bs);
    }
  }
};
template <>
struct StrassenOps<0> {
  static __device__ __forceinline__ void run(const double (&x)[1][1], const int8_t (&)[7][4], double* out,
                                             long long) {
    out[0] = x[0][0];
  }
};

// c[R][C] = the 2^LV x 2^LV blocks of the product recombined from its 7^LV leaf products m[k * bs]
template <int LV>
struct StrassenComb {
  static __device__ __forceinline__ void run(const double* m, long long bs, double (&c)[1 << LV][1 << LV]) {
    constexpr int H = 1 << (LV - 1);
#pragma unroll
    for (int r = 0; r < 2 * H; ++r)
#pragma unroll
      for (int q = 0; q < 2 * H; ++q) c[r][q] = 0.0;
    auto add = [&](int s) {
      double ch[H][H];
      StrassenComb<LV - 1>::run(m + (long long)s * P7<LV - 1>::v * bs, bs, ch);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double k = kSC[b][s];
#pragma unroll
        for (int r = 0; r < H; ++r)
#pragma unroll
          for (int q = 0; q < H; ++q) c[(b >> 1) * H + r][(b & 1) * H + q] += k * ch[r][q];
      }
    };
    if constexpr (LV >= 3) {   // one top-level product at a time: 49 loads live, not 343
#pragma unroll 1
      for (int s = 0; s < 7; ++s) add(s);
    } else {
#pragma unroll
      for (int s = 0; s < 7; ++s) add(s);
    }
  }
};
template <>
struct StrassenComb<0> {
  static __device__ __forceinline__ void run(const double* m, long long, double (&c)[1][1]) { c[0][0] = m[0]; }
};

// Ks[q][s][i][j] (s < 7^LV) from K's planes: leaf grid h = L / 2^LV
template <int LV>
__global__ void strassen_a_kernel(const double* __restrict__ Kp, long long ldk, long long pk, int h,
                                  double* __restrict__ Ks, long long ldks) {
  constexpr int G = 1 << LV, NS = P7<LV>::v;
  const int q = blockIdx.z, i = blockIdx.y;
  const double* k = Kp + q * pk;
  const long long bs = (long long)h * ldks;
  double* o = Ks + (long long)q * NS * bs + (long long)i * ldks;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < h; j += gridDim.x * blockDim.x) {
    double x[G][G];
#pragma unroll
    for (int R = 0; R < G; ++R)
#pragma unroll
      for (int C = 0; C < G; ++C) x[R][C] = k[(long long)(R * h + i) * ldk + C * h + j];
    StrassenOps<LV>::run(x, kSA, o + j, bs);
  }
}

// Bc[q][s][t][i][j]: the operands of the planes (re, im, re + im) of U[t]; leaf grid h x nh.  PL < 0: all
// three planes in one pass; PL = q: plane q only (the three-level pass, whose 64 positions per thread
// leave no registers for three planes)
template <int LV, int PL>
__global__ void strassen_b_kernel(const cplx* __restrict__ U, long long ldu, long long sU, int h, int nh, int T,
                                  double* __restrict__ Bc, long long ldb) {
  constexpr int G = 1 << LV, NS = P7<LV>::v;
  const int t = blockIdx.z, i = blockIdx.y;
  const cplx* u = U + t * sU;
  const long long bs = (long long)T * h * ldb;          // stride between (q, s) entries
  double* o = Bc + (long long)t * h * ldb + (long long)i * ldb;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nh; j += gridDim.x * blockDim.x) {
    double2 v[G][G];
#pragma unroll
    for (int R = 0; R < G; ++R)
#pragma unroll
      for (int C = 0; C < G; ++C) v[R][C] = u[(long long)(R * h + i) * ldu + C * nh + j];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (PL >= 0 && q != PL) continue;
      double x[G][G];
#pragma unroll
      for (int R = 0; R < G; ++R)
#pragma unroll
        for (int C = 0; C < G; ++C) x[R][C] = q == 0 ? v[R][C].x : (q == 1 ? v[R][C].y : v[R][C].x + v[R][C].y);
      StrassenOps<LV>::run(x, kSB, o + (long long)q * NS * bs + j, bs);
    }
  }
}

// U[t] (+)= the product recombined from the leaf products: per plane the 2^LV x 2^LV blocks, then
// (P1 - P2) + i (P3 - P1 - P2).  PL < 0: all planes; PL = q: plane q's share only, added to U
// (plane 0 writes or accumulates per `accumulate`, planes 1 and 2 always accumulate)
template <int LV, int PL>
__global__ void strassen_c_kernel(const double* __restrict__ Mb, long long ldb, int h, int nh, int T,
                                  cplx* __restrict__ U, long long ldu, long long sU, int accumulate) {
  constexpr int G = 1 << LV, NS = P7<LV>::v;
  const int t = blockIdx.z, i = blockIdx.y;
  const long long bs = (long long)T * h * ldb;
  const double* m = Mb + (long long)t * h * ldb + (long long)i * ldb;
  cplx* u = U + t * sU;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nh; j += gridDim.x * blockDim.x) {
    if (PL >= 0) {   // plane PL's share: (re, im) += (sr, si) x its product
      double c[G][G];
      StrassenComb<LV>::run(m + (long long)PL * NS * bs + j, bs, c);
      const double sr = PL == 0 ? 1.0 : (PL == 1 ? -1.0 : 0.0), si = PL == 2 ? 1.0 : -1.0;
      const bool acc = PL > 0 || accumulate;
#pragma unroll
      for (int R = 0; R < G; ++R)
#pragma unroll
        for (int C = 0; C < G; ++C) {
          cplx* p = u + (long long)(R * h + i) * ldu + C * nh + j;
          double2 v = make_double2(sr * c[R][C], si * c[R][C]);
          if (acc) {
            const double2 o = *p;
            v.x += o.x;
            v.y += o.y;
          }
          *p = v;
        }
      continue;
    }
    double c[3][G][G];
#pragma unroll
    for (int q = 0; q < 3; ++q) StrassenComb<LV>::run(m + (long long)q * NS * bs + j, bs, c[q]);
#pragma unroll
    for (int R = 0; R < G; ++R)
#pragma unroll
      for (int C = 0; C < G; ++C) {
        cplx* p = u + (long long)(R * h + i) * ldu + C * nh + j;
        double2 v = make_double2(c[0][R][C] - c[1][R][C], c[2][R][C] - c[0][R][C] - c[1][R][C]);
        if (accumulate) {
          const double2 o = *p;
          v.x += o.x;
          v.y += o.y;
        }
        *p = v;
      }
  }
}

}  // namespace

namespace {

// the three-level recombination, one plane, one top-level quadrant b1 = blockIdx.z per thread (one
// trajectory): c = sum over the top-level products s1 feeding b1 of kSC[b1][s1] x their two-level
// recombination -- 16 outputs and at most 4 x 49 loads per thread instead of 64 and 343
template <int PL>
__global__ void __launch_bounds__(256, 2) strassen_c3_kernel(const double* __restrict__ Mb, long long ldb, int h, int nh,
                                   cplx* __restrict__ U, long long ldu, int accumulate) {
  const int i = blockIdx.y, b1 = blockIdx.z;
  const long long bs = (long long)h * ldb;
  const double* m = Mb + (long long)PL * 343 * bs + (long long)i * ldb;
  const double sr = PL == 0 ? 1.0 : (PL == 1 ? -1.0 : 0.0), si = PL == 2 ? 1.0 : -1.0;
  const bool acc = PL > 0 || accumulate;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nh; j += gridDim.x * blockDim.x) {
    double c[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) c[r][q] = 0.0;
#pragma unroll 1
    for (int s1 = 0; s1 < 7; ++s1) {
      const double k = kSC[b1][s1];
      if (k == 0.0) continue;
      double ch[4][4];
      StrassenComb<2>::run(m + (long long)s1 * 49 * bs + j, bs, ch);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) c[r][q] += k * ch[r][q];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int R = (b1 >> 1) * 4 + r, C = (b1 & 1) * 4 + q;
        cplx* p = U + (long long)(R * h + i) * ldu + C * nh + j;
        double2 v = make_double2(sr * c[r][q], si * c[r][q]);
        if (acc) {
          const double2 o = *p;
          v.x += o.x;
          v.y += o.y;
        }
        *p = v;
      }
  }
}

}  // namespace

int strassen_k(cudaStream_t st, int levels, const double* Kp, long long ldk, long long pk, int L, double* Ks,
               long long ldks, std::string* err) {
  const int h = L >> levels;
  dim3 grid((unsigned)std::min<long long>(ceil_div(h, 256), 16), h, 3);
  if (levels == 3) strassen_a_kernel<3><<<grid, 256, 0, st>>>(Kp, ldk, pk, h, Ks, ldks);
  else if (levels == 2) strassen_a_kernel<2><<<grid, 256, 0, st>>>(Kp, ldk, pk, h, Ks, ldks);
  else strassen_a_kernel<1><<<grid, 256, 0, st>>>(Kp, ldk, pk, h, Ks, ldks);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("strassen_k: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

int strassen_b(cudaStream_t st, int levels, const cplx* U, long long ldu, long long sU, int L, int N, int T,
               double* Bc, long long ldb, std::string* err) {
  const int h = L >> levels, nh = N >> levels;
  dim3 grid((unsigned)std::min<long long>(ceil_div(nh, 256), 16), h, T);
  if (levels == 3) {
    strassen_b_kernel<3, 0><<<grid, 256, 0, st>>>(U, ldu, sU, h, nh, T, Bc, ldb);
    strassen_b_kernel<3, 1><<<grid, 256, 0, st>>>(U, ldu, sU, h, nh, T, Bc, ldb);
    strassen_b_kernel<3, 2><<<grid, 256, 0, st>>>(U, ldu, sU, h, nh, T, Bc, ldb);
    count_launch(2);
  } else if (levels == 2) {
    strassen_b_kernel<2, -1><<<grid, 256, 0, st>>>(U, ldu, sU, h, nh, T, Bc, ldb);
  } else {
    strassen_b_kernel<1, -1><<<grid, 256, 0, st>>>(U, ldu, sU, h, nh, T, Bc, ldb);
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("strassen_b: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

int strassen_c(cudaStream_t st, int levels, const double* Mb, long long ldb, int L, int N, int T, cplx* U,
               long long ldu, long long sU, std::string* err, int accumulate) {
  const int h = L >> levels, nh = N >> levels;
  dim3 grid((unsigned)std::min<long long>(ceil_div(nh, 256), 16), h, T);
  if (levels == 3) {   // one trajectory (traj_api.cu): grid.z = the top-level quadrant
    if (T != 1) {
      if (err) *err = "strassen_c: three levels need one trajectory";
      return 1;
    }
    dim3 g3(grid.x, h, 4);
    strassen_c3_kernel<0><<<g3, 256, 0, st>>>(Mb, ldb, h, nh, U, ldu, accumulate);
    strassen_c3_kernel<1><<<g3, 256, 0, st>>>(Mb, ldb, h, nh, U, ldu, accumulate);
    strassen_c3_kernel<2><<<g3, 256, 0, st>>>(Mb, ldb, h, nh, U, ldu, accumulate);
    count_launch(2);
  } else if (levels == 2) {
    strassen_c_kernel<2, -1><<<grid, 256, 0, st>>>(Mb, ldb, h, nh, T, U, ldu, sU, accumulate);
  } else {
    strassen_c_kernel<1, -1><<<grid, 256, 0, st>>>(Mb, ldb, h, nh, T, U, ldu, sU, accumulate);
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) *err = std::string("strassen_c: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

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
