// Fused small-lattice trajectory step (rows a1-a3 of SURVEY §8(a) in one kernel).
//
// c1 (L = 64, N = 32) is latency-bound on the general path: ~20 launches and two host round trips
// per step for a few hundred kFLOP.  Here one CTA owns one trajectory; U stays in shared memory
// for a whole run of steps and every step is
//   (a1) U <- K U                                   (K read through L1/L2, shared by the batch)
//   (a2) homodyne: n_i = sum_k |U_ik|^2, U_i. *= exp(sqrt(gamma dt) z_i + (2 n_i - 1) gamma dt)
//        (Eq. A3, split form, readings Q5-Q8; z_i Box-Muller of the site's Philox pair), or
//        projective: sites with u0 < gamma dt in ascending order (Q10, Q16); conditional Born
//        sampling on C_SS = U_S U_S^dag with the Eq. (A1) / sign-corrected (A2) Schur update
//        (Q13, Q15, Q17; C_SS in the idle scratch buffer, or in global memory when the click
//        list is longer); each occupied site j then maps U <- U - (U w - e_j) w^dag with
//        w = conj(U_j.)/|U_j.|, and the rows of the empty sites are zeroed
//   (a3) CholeskyQR2 (P:209 orthonormalisation; north star (c)): twice G = U^dag U, G = R^dag R,
//        U <- U R^-1
// with the same Philox counters (site, step, traj_global, 0) as monitor.cu.  The occupied-site
// projections are applied one at a time instead of monitor.cu's block rank-k update: both give
// span(E_S1) + Z_S0 U null(U_S1) (the projectors of distinct sites commute), i.e. the same
// C = U U^dag after CholeskyQR2.  The Cholesky factor's inverse comes from Gaussian elimination
// of [G | I] on unscaled rows (two pivots per barrier), U R^-1 is then one product.  The three
// GEMM-shaped phases (K U, U^dag U, U X) run on the FP64 tensor pipe (m8n8k4 DMMA, 8 x 8 complex
// tiles, one per warp at a time); the rest is DFMA with rows on warps and columns on lanes.
#include <math.h>
#include "common.cuh"
#include "small_step.h"

namespace traj {

namespace {

constexpr int SB = 512;   // threads per CTA (one trajectory)
constexpr int NW = SB / 32;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // conj(a) b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cmulcb(double2 a, double2 b) {  // a conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// C (8 x 8 complex, lane: row g, columns 2 slot, 2 slot + 1) += op(A) B over k < K on the FP64
// tensor pipe: four real m8n8k4 DMMAs per k-step of 4.  fa(m, k) returns A[m0 + m][k] and
// fb(k, n) returns B[k][n0 + n] (zero outside the operands); op(A) = conj(A) when CONJ_A.
template <bool CONJ_A, class FA, class FB>
__device__ __forceinline__ void ztile(FA fa, FB fb, int K, int g, int slot, double* cr, double* ci) {
  // two accumulator sets (even / odd k-steps) halve the dependent DMMA chains
  double r1[2] = {0.0, 0.0}, i1[2] = {0.0, 0.0};
  int k0 = 0;
  for (; k0 + 4 < K; k0 += 8) {
    const double2 av = fa(g, k0 + slot), aw = fa(g, k0 + 4 + slot);
    const double2 bv = fb(k0 + slot, g), bw = fb(k0 + 4 + slot, g);
    const double ai = CONJ_A ? -av.y : av.y, aj = CONJ_A ? -aw.y : aw.y;
    dmma_8x8x4(cr[0], cr[1], av.x, bv.x);
    dmma_8x8x4(r1[0], r1[1], aw.x, bw.x);
    dmma_8x8x4(ci[0], ci[1], av.x, bv.y);
    dmma_8x8x4(i1[0], i1[1], aw.x, bw.y);
    dmma_8x8x4(cr[0], cr[1], -ai, bv.y);
    dmma_8x8x4(r1[0], r1[1], -aj, bw.y);
    dmma_8x8x4(ci[0], ci[1], ai, bv.x);
    dmma_8x8x4(i1[0], i1[1], aj, bw.x);
  }
  if (k0 < K) {
    const double2 av = fa(g, k0 + slot);
    const double2 bv = fb(k0 + slot, g);
    const double ai = CONJ_A ? -av.y : av.y;
    dmma_8x8x4(cr[0], cr[1], av.x, bv.x);
    dmma_8x8x4(ci[0], ci[1], av.x, bv.y);
    dmma_8x8x4(cr[0], cr[1], -ai, bv.y);
    dmma_8x8x4(ci[0], ci[1], ai, bv.x);
  }
  cr[0] += r1[0];
  cr[1] += r1[1];
  ci[0] += i1[0];
  ci[1] += i1[1];
}

__device__ __forceinline__ bool decide_born(double p, double u1) {   // readings Q13, Q17
  p = fmin(fmax(p, 0.0), 1.0);
  bool occ = u1 < p;
  if (occ && p < 1e-12) occ = false;
  else if (!occ && (1.0 - p) < 1e-12) occ = true;
  return occ;
}

struct Carve {
  double2 *A, *B, *G, *uw, *wv;
  double *piv, *u0, *u1, *red;
  int *S, *occ, *misc;
};

__host__ __device__ inline size_t carve_small(int L, int N, bool proj, char* base, Carve* c) {
  const size_t ld = N + 1;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + o : nullptr;
    o += (bytes + 15) & ~size_t(15);
    return p;
  };
  Carve k;
  k.A = reinterpret_cast<double2*>(take(L * ld * 16));
  k.B = reinterpret_cast<double2*>(take(L * ld * 16));
  k.G = reinterpret_cast<double2*>(take(N * ld * 16));
  k.uw = reinterpret_cast<double2*>(take(L * 16));
  k.wv = reinterpret_cast<double2*>(take(N * 16));
  k.piv = reinterpret_cast<double*>(take(N * 8));
  k.u0 = reinterpret_cast<double*>(take(L * 8));
  k.u1 = reinterpret_cast<double*>(take(L * 8));
  k.red = reinterpret_cast<double*>(take(NW * 8));
  k.S = reinterpret_cast<int*>(take(L * 4));
  k.occ = reinterpret_cast<int*>(take(L * 4));
  k.misc = reinterpret_cast<int*>(take(8 * 4));
  if (c) *c = k;
  return o;
}

__global__ void __launch_bounds__(SB, 1) small_step_kernel(SmallStepArgs a) {
  extern __shared__ __align__(16) char smraw[];
  const int L = a.L, N = a.N, ld = N + 1;
  const bool proj = a.projective != 0;
  Carve c;
  carve_small(L, N, proj, smraw, &c);
  double2* A = c.A;
  double2* B = c.B;
  double2* G = c.G;
  // every element loop maps rows to warps and columns to lanes (no integer division)
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.failed[t]) return;
  cplx* Ug = a.U + t * a.sU;
  for (int i = warp; i < L; i += NW)
    for (int k = lane; k < N; k += 32) A[i * ld + k] = Ug[(long long)i * a.ldU + k];
  const double gdt = a.gamma[t] * a.dt;
  const uint32_t tr = (uint32_t)(a.traj_base + t);
  const uint32_t key0 = (uint32_t)(a.seed & 0xffffffffu), key1 = (uint32_t)(a.seed >> 32);
  bool bad = false;
  __syncthreads();
  for (long long s = 0; s < a.n_steps && !bad; ++s) {
    const uint32_t step = (uint32_t)(a.step0 + s);
    // ---- (a1) B = K A on the DMMA pipe: one 8 x 8 complex tile per warp at a time
    {
      const int NT = (N + 7) >> 3, MT = (L + 7) >> 3;
      for (int tile = warp; tile < MT * NT; tile += NW) {
        const int m0 = (tile / NT) * 8, n0 = (tile % NT) * 8;
        double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
        const double2* Ad = A;
        ztile<false>(
            [&](int m, int k) {
              return (m0 + m < L && k < L) ? __ldg(a.K + (long long)(m0 + m) * a.ldK + k) : make_double2(0.0, 0.0);
            },
            [&](int k, int n) { return (k < L && n0 + n < N) ? Ad[k * ld + n0 + n] : make_double2(0.0, 0.0); }, L,
            lane >> 2, lane & 3, cr, ci);
        const int r = m0 + (lane >> 2), c0 = n0 + 2 * (lane & 3);
        if (r < L) {
          if (c0 < N) B[r * ld + c0] = make_double2(cr[0], ci[0]);
          if (c0 + 1 < N) B[r * ld + c0 + 1] = make_double2(cr[1], ci[1]);
        }
      }
    }
    __syncthreads();
    {
      double2* tmp = A;
      A = B;
      B = tmp;
    }
    // ---- (a2) monitor
    if (!proj) {
      for (int i = warp; i < L; i += NW) {   // one warp per row
        double n = 0.0;
        for (int k = lane; k < N; k += 32) {
          const double2 v = A[i * ld + k];
          n += v.x * v.x + v.y * v.y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
        double f = 0.0;
        if (lane == 0) {
          const u32x4 x = philox4x32_10(u32x4{(uint32_t)i, step, tr, 0u}, key0, key1);
          const double u0 = u53(x.x, x.y), u1 = u53(x.z, x.w);
          const double z = sqrt(-2.0 * log(1.0 - u0)) * cos(2.0 * M_PI * u1);
          f = exp(sqrt(gdt) * z + (2.0 * n - 1.0) * gdt);
        }
        f = __shfl_sync(0xffffffffu, f, 0);
        for (int k = lane; k < N; k += 32) {
          const double2 v = A[i * ld + k];
          A[i * ld + k] = make_double2(f * v.x, f * v.y);
        }
      }
      __syncthreads();
    } else {
      for (int i = tid; i < L; i += SB) {
        const u32x4 x = philox4x32_10(u32x4{(uint32_t)i, step, tr, 0u}, key0, key1);
        c.u0[i] = u53(x.x, x.y);
        c.u1[i] = u53(x.z, x.w);
      }
      __syncthreads();
      if (warp == 0) {   // ascending click list S
        int m = 0;
        for (int c0 = 0; c0 < L; c0 += 32) {
          const int i = c0 + lane;
          const bool fl = i < L && c.u0[i] < gdt;
          const unsigned b = __ballot_sync(0xffffffffu, fl);
          if (fl) c.S[m + __popc(b & ((1u << lane) - 1u))] = i;
          m += __popc(b);
        }
        if (lane == 0) c.misc[0] = m;
      }
      __syncthreads();
      const int m = c.misc[0];
      if (m > a.cap) {   // the general path's click-list overflow (TRAJ_ENUMERIC there)
        bad = true;
        break;
      }
      // C_SS = U_S U_S^dag in the free scratch buffer B when it fits, else in global memory
      const bool in_smem = (long long)m * (m + 1) <= (long long)L * ld;
      double2* D = in_smem ? B : a.Dg + t * a.sDg;
      const int ldd = in_smem ? m + 1 : (int)a.ldDg;
      for (int p = warp; p < m; p += NW) {
        const double2* up = A + c.S[p] * ld;
        for (int q = lane; q < m; q += 32) {
          const double2* uq = A + c.S[q] * ld;
          double2 acc = make_double2(0.0, 0.0);
          for (int k = 0; k < N; ++k) {
            const double2 v = cmulcb(up[k], uq[k]);
            acc.x += v.x;
            acc.y += v.y;
          }
          D[p * ldd + q] = acc;
        }
      }
      __syncthreads();
      // sequential conditional sampling: pivot p (occupied) or p - 1 (empty),
      // C <- C - C[:, r] C[r, :] / pivot on the trailing block
      for (int r = 0; r < m; ++r) {
        const double p = D[r * ldd + r].x;
        const bool o = decide_born(p, c.u1[c.S[r]]);
        const double inv = 1.0 / (o ? p : p - 1.0);
        if (tid == 0) c.occ[r] = o ? 1 : 0;
        for (int i = r + 1 + warp; i < m; i += NW) {
          const double2 l = D[i * ldd + r];
          const double lx = l.x * inv, ly = l.y * inv;
          for (int k = r + 1 + lane; k < m; k += 32) {
            const double2 d = D[r * ldd + k];
            D[i * ldd + k].x -= lx * d.x - ly * d.y;
            D[i * ldd + k].y -= lx * d.y + ly * d.x;
          }
        }
        __syncthreads();
      }
      // occupied sites, ascending: U <- U - (U w - e_j) w^dag, w = conj(U_j.) / |U_j.|
      int k1 = 0;
      for (int r = 0; r < m; ++r) {
        if (!c.occ[r]) continue;
        ++k1;
        const int j = c.S[r];
        if (warp == 0) {
          double n = 0.0;
          for (int k = lane; k < N; k += 32) {
            const double2 v = A[j * ld + k];
            n += v.x * v.x + v.y * v.y;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
          const double rn = 1.0 / sqrt(n);
          for (int k = lane; k < N; k += 32) {
            const double2 v = A[j * ld + k];
            c.wv[k] = make_double2(v.x * rn, -v.y * rn);   // w_k
          }
        }
        __syncthreads();
        for (int i = warp; i < L; i += NW) {   // (U w)_i - delta_ij, one warp per row
          double2 acc = make_double2(0.0, 0.0);
          for (int k = lane; k < N; k += 32) {
            const double2 v = cmul(A[i * ld + k], c.wv[k]);
            acc.x += v.x;
            acc.y += v.y;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
          }
          if (i == j) acc.x -= 1.0;
          if (lane == 0) c.uw[i] = acc;
        }
        __syncthreads();
        for (int i = warp; i < L; i += NW) {
          const double2 u = c.uw[i];
          for (int k = lane; k < N; k += 32) {
            const double2 v = cmulcb(u, c.wv[k]);
            A[i * ld + k].x -= v.x;
            A[i * ld + k].y -= v.y;
          }
        }
        __syncthreads();
      }
      for (int r = warp; r < m; r += NW)   // empty sites: rows zeroed
        if (!c.occ[r])
          for (int k = lane; k < N; k += 32) A[c.S[r] * ld + k] = make_double2(0.0, 0.0);
      if (tid == 0) {
        c.misc[1] = m - k1;   // zeroed rows
        if (s == a.n_steps - 1) {
          a.last[2 * t] = m;
          a.last[2 * t + 1] = k1;
        }
      }
      __syncthreads();
    }
    // ---- (a3) CholeskyQR2.  Per pass: G = A^dag A (upper); Gaussian elimination of [G | I] on
    // unscaled rows, G = L D L^dag, W = L^-1 (in B); X = R^-1 = W^dag D^-1/2 (into G's upper
    // triangle); B = A X.  N + 3 barriers per pass.
    // projective: the occupied-site maps are exact isometries and K is unitary, so with no row
    // zeroed U is orthonormal to rounding and pass 1 has R = I (the general path's rule with the
    // low-rank first Gram on; pass 2 still measures the Gram and certifies the result)
    const bool skip1 = proj && a.skip_orthonormal_pass && c.misc[1] == 0;
    for (int pass = skip1 ? 1 : 0; pass < 2 && !bad; ++pass) {
      double2* W = B;
      double dev = 0.0;
      for (int p = warp; p < N; p += NW)
        for (int q = lane; q < N; q += 32) W[p * ld + q] = make_double2(p == q ? 1.0 : 0.0, 0.0);
      {   // G = A^dag A, tiles on and above the diagonal (DMMA)
        const int NT = (N + 7) >> 3;
        for (int tile = warp; tile < NT * NT; tile += NW) {
          const int pt = tile / NT, qt = tile % NT;
          if (pt > qt) continue;
          const int p0 = pt * 8, q0 = qt * 8;
          double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
          const double2* Ad = A;
          ztile<true>([&](int m, int k) { return (k < L && p0 + m < N) ? Ad[k * ld + p0 + m] : make_double2(0.0, 0.0); },
                      [&](int k, int n) { return (k < L && q0 + n < N) ? Ad[k * ld + q0 + n] : make_double2(0.0, 0.0); },
                      L, lane >> 2, lane & 3, cr, ci);
          const int r = p0 + (lane >> 2), c0 = q0 + 2 * (lane & 3);
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cc = c0 + e;
            if (r < N && cc < N) {
              G[r * ld + cc] = make_double2(cr[e], ci[e]);
              if (r <= cc) {   // max |G - I| over the upper triangle (NaN propagates)
                const double d = fmax(fabs(cr[e] - (r == cc ? 1.0 : 0.0)), fabs(ci[e]));
                dev = (d > dev || d != d) ? d : dev;
              }
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, dev, o);
        dev = (v > dev || v != v) ? v : dev;
      }
      if (lane == 0) c.red[warp] = dev;
      __syncthreads();
      // second pass: G = I + E with |E| ~ kappa^2 eps, R^-1 = I - triu(E, 1) - diag(E) / 2 up to
      // O(N |E|^2), exact to rounding when N max|E|^2 < 1e-18 (the general path's rule and
      // threshold, monitor.cu first_order_inverse); otherwise the full factorisation
      bool first_order = false;
      if (pass == 1 && !a.full_cqr2) {
        double mx = 0.0;
        for (int w = 0; w < NW; ++w) mx = (c.red[w] > mx || c.red[w] != c.red[w]) ? c.red[w] : mx;
        first_order = mx <= 1e-9 / sqrt((double)N);
        if (!first_order && tid == 0) atomicAdd(a.fallbacks, 1ull);
      }
      if (first_order) {
        for (int p = warp; p < N; p += NW)
          for (int q = p + lane; q < N; q += 32) {
            const double2 v = G[p * ld + q];
            G[p * ld + q] = q == p ? make_double2(1.0 - 0.5 * (v.x - 1.0), 0.0) : make_double2(-v.x, -v.y);
          }
        __syncthreads();
      }
      if (!first_order) {
        // two pivots (a, a + 1) per barrier: row a + 1 after pivot a is formed on the fly,
        //   m = conj(G_a,a+1) / p_a,  G'_a+1,k = G_a+1,k - m G_a,k,  p_a+1 = G'_a+1,a+1,
        // and each row i > a + 1 takes  row_i -= c_a row_a + c_b row_a+1  (G: k >= i; W: k <= a + 1)
        // with l_a = conj(G_a,i) / p_a, c_b = conj(G'_a+1,i) / p_a+1, c_a = l_a - c_b m.  W's row
        // a + 1 itself becomes W_a+1 - m W_a in the next phase (nobody reads it there).
        int prev = -1;   // first pivot of the previous pair: W row prev + 1 still pending
        for (int j = 0; j < N; j += 2) {
          const bool pair = j + 1 < N;
          const double pa = G[j * ld + j].x;
          if (!(pa > 0.0) || !isfinite(pa)) {   // the same values in every thread: uniform exit
            bad = true;
            break;
          }
          const double ia = 1.0 / pa;
          double2 mm = make_double2(0.0, 0.0);
          double ib = 0.0;
          if (pair) {
            const double2 gab = G[j * ld + j + 1];
            mm = make_double2(gab.x * ia, -gab.y * ia);
            const double pb = G[(j + 1) * ld + j + 1].x - (gab.x * gab.x + gab.y * gab.y) * ia;
            if (!(pb > 0.0) || !isfinite(pb)) {
              bad = true;
              break;
            }
            ib = 1.0 / pb;
            if (tid == 0) c.piv[j + 1] = pb;
          }
          if (tid == 0) c.piv[j] = pa;
          if (prev >= 0 && warp == NW - 1) {   // the previous pair's pending W row
            const double2 g = G[prev * ld + prev + 1];
            const double ip = 1.0 / c.piv[prev];
            const double mx = g.x * ip, my = -g.y * ip;
            for (int k = lane; k <= prev; k += 32) {
              const double2 w = W[prev * ld + k];
              W[(prev + 1) * ld + k].x -= mx * w.x - my * w.y;
              W[(prev + 1) * ld + k].y -= mx * w.y + my * w.x;
            }
          }
          const int b = pair ? j + 1 : j;
          for (int i = b + 1 + warp; i < N; i += NW) {
            const double2 gai = G[j * ld + i];
            const double lax = gai.x * ia, lay = -gai.y * ia;              // l_a
            double cax = lax, cay = lay, cbx = 0.0, cby = 0.0;
            if (pair) {
              const double2 gbi = G[(j + 1) * ld + i];
              const double2 gpi = make_double2(gbi.x - (mm.x * gai.x - mm.y * gai.y),
                                               gbi.y - (mm.x * gai.y + mm.y * gai.x));   // G'_a+1,i
              cbx = gpi.x * ib;
              cby = -gpi.y * ib;
              cax = lax - (cbx * mm.x - cby * mm.y);
              cay = lay - (cbx * mm.y + cby * mm.x);
            }
            for (int k = i + lane; k < N; k += 32) {   // G row i, upper part
              const double2 ra = G[j * ld + k];
              double2 v = G[i * ld + k];
              v.x -= cax * ra.x - cay * ra.y;
              v.y -= cax * ra.y + cay * ra.x;
              if (pair) {
                const double2 rb = G[(j + 1) * ld + k];
                v.x -= cbx * rb.x - cby * rb.y;
                v.y -= cbx * rb.y + cby * rb.x;
              }
              G[i * ld + k] = v;
            }
            for (int k = lane; k <= b; k += 32) {      // W row i, columns <= b
              const double2 wa = W[j * ld + k];
              double2 v = W[i * ld + k];
              v.x -= cax * wa.x - cay * wa.y;
              v.y -= cax * wa.y + cay * wa.x;
              if (pair) {
                const double2 wb = W[(j + 1) * ld + k];
                v.x -= cbx * wb.x - cby * wb.y;
                v.y -= cbx * wb.y + cby * wb.x;
              }
              W[i * ld + k] = v;
            }
          }
          prev = pair ? j : -1;
          __syncthreads();
        }
        if (!bad && prev >= 0) {   // the last pair's pending W row
          if (warp == NW - 1) {
            const double2 g = G[prev * ld + prev + 1];
            const double ip = 1.0 / c.piv[prev];
            const double mx = g.x * ip, my = -g.y * ip;
            for (int k = lane; k <= prev; k += 32) {
              const double2 w = W[prev * ld + k];
              W[(prev + 1) * ld + k].x -= mx * w.x - my * w.y;
              W[(prev + 1) * ld + k].y -= mx * w.y + my * w.x;
            }
          }
          __syncthreads();
        }
        if (bad) break;
        for (int i = warp; i < N; i += NW) {   // X_ki = conj(W_ik) / sqrt(p_i), k <= i
          const double ir = 1.0 / sqrt(c.piv[i]);
          for (int k = lane; k <= i; k += 32) {
            const double2 w = W[i * ld + k];
            G[k * ld + i] = make_double2(w.x * ir, -w.y * ir);
          }
        }
        __syncthreads();
      }
      {   // B = A X (DMMA), X upper triangular in G: k-steps past the tile's last column skipped
        const int NT = (N + 7) >> 3, MT = (L + 7) >> 3;
        for (int tile = warp; tile < MT * NT; tile += NW) {
          const int m0 = (tile / NT) * 8, n0 = (tile % NT) * 8;
          double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
          const double2* Ad = A;
          const double2* Xd = G;
          ztile<false>([&](int m, int k) { return (m0 + m < L && k < N) ? Ad[(m0 + m) * ld + k] : make_double2(0.0, 0.0); },
                       [&](int k, int n) {
                         return (k <= n0 + n && n0 + n < N) ? Xd[k * ld + n0 + n] : make_double2(0.0, 0.0);
                       },
                       min(N, n0 + 8), lane >> 2, lane & 3, cr, ci);
          const int r = m0 + (lane >> 2), c0 = n0 + 2 * (lane & 3);
          if (r < L) {
            if (c0 < N) B[r * ld + c0] = make_double2(cr[0], ci[0]);
            if (c0 + 1 < N) B[r * ld + c0 + 1] = make_double2(cr[1], ci[1]);
          }
        }
      }
      __syncthreads();
      double2* tmp = A;
      A = B;
      B = tmp;
    }
  }
  if (bad && tid == 0) a.failed[t] = 1;
  for (int i = warp; i < L; i += NW)
    for (int k = lane; k < N; k += 32) Ug[(long long)i * a.ldU + k] = A[i * ld + k];
}

}  // namespace

size_t small_step_smem_bytes(int L, int N, bool projective) {
  return carve_small(L, N, projective, nullptr, nullptr);
}

bool small_step_fits(int L, int N, bool projective) {
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  return L > 0 && N > 0 && small_step_smem_bytes(L, N, projective) <= (size_t)optin;
}

int small_steps(cudaStream_t st, const SmallStepArgs& a, std::string* err) {
  if (a.n_steps <= 0 || a.T <= 0) return 0;
  const size_t smem = small_step_smem_bytes(a.L, a.N, a.projective != 0);
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // the attribute is raised once per device to the opt-in maximum (any (L, N) that fits)
  if (e == cudaSuccess) e = ensure_smem(reinterpret_cast<const void*>(small_step_kernel), optin);
  if (e == cudaSuccess && smem > (size_t)optin) e = cudaErrorInvalidValue;
  if (e == cudaSuccess) {
    small_step_kernel<<<a.T, SB, smem, st>>>(a);
    count_launch();
    e = cudaGetLastError();
  }
  if (e != cudaSuccess && err) *err = std::string("small_steps: ") + cudaGetErrorString(e);
  return e == cudaSuccess ? 0 : 4;
}

}  // namespace traj
