// Complex-FP64 GEMM on the B200 FP64 tensor pipe (DMMA.8x8x4), TMA-fed.
//
//   C_b = alpha * op(A_b) * op(B_b) + beta * C_b,  op in {N, C(onjugate transpose)}
//
// Used for every contraction of the step: U <- K U (a1),
// G = U^dag U and U <- U R^-1 (a3, CholeskyQR2 for the QR of P:209), the Cholesky /
// triangular-inverse recursion, the projective rank-k update (a2) and C_A = U_A U_A^dag (a4).
//
// Design (sm_100a):
//  * tcgen05 has no f64 kind; the FP64 tensor path is mma.sync.m8n8k4.f64 -> DMMA.8x8x4
//    (measured 37.1 TF/s chip peak, profiles/r01_fp64_microbench.txt).
//  * Complex product as 4 real products folded into 2 real MMAs over an interleaved
//    k axis: k_real = (complex k, component c).  With op(A) = a_r + i sa a_i and
//    op(B) = b_r + i sb b_i (sa, sb = -1 for a conjugated operand):
//        Cr += [a_r, -sa*sb*a_i] . [b_r, b_i]      (B fragment: the raw interleaved double)
//        Ci += [sb*a_r,  sa*a_i] . [b_i, b_r]      (B fragment: the swapped double)
//    so every B fragment is a plain 64-bit shared load and the signs are sign-bit XORs
//    on the A fragment (ALU pipe; a DADD negation would sit on the FP64 pipe and stall
//    the dependent DMMA).
//  * CTA tile 128 x 64 complex, 8 warps of 32 x 32 complex (64 accumulator doubles
//    each, up to 255 registers: 2 warps per SM sub-partition).  Lane 0 of warp 0 also
//    issues the TMA loads (cp.async.bulk.tensor) STAGES-1 stages ahead into a 6-stage
//    mbarrier ring of 24 KB stages (8 complex k per stage); a separate producer warp
//    would put 3 warps on one sub-partition and cap registers at 168.
//  * Every smem tile is made of 128-byte lines with the TMA 128B swizzle; each MMA
//    k-step pairs complex k with k+4, which makes all four operand layouts
//    (k-contiguous or m/n-contiguous) bank-conflict free.
//  * Out-of-range rows / k are zero-filled by TMA, so ragged M, N, K need no masks
//    except in the epilogue.
#include "common.cuh"
#include "zgemm.h"
#include <stdlib.h>

namespace traj {

namespace {

constexpr int BM = 128;
constexpr int BN = 64;
constexpr int BKC = 8;                 // complex k per stage
constexpr int STAGES = 6;
constexpr int CONSUMER_WARPS = 8;
constexpr int THREADS = CONSUMER_WARPS * 32;
constexpr int A_BYTES = BM * 128;
constexpr int B_BYTES = BN * 128;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8;
constexpr int GROUP_M = 8;

struct Args {
  int M, N, K;
  int tiles_m, tiles_n;
  int flags;
  int a_batched, b_batched;
  int a_4d, b_4d;          // m/n-contiguous operand mapped as one 4D box per stage
  double alpha_re, alpha_im, beta;
  cplx* C;
  long long ldc, strideC;
  int m_off, n_off;        // global row / column of this call's (0, 0): triangle and upper-tile tests
  // device-side bounds (zgemm.h DevBounds): read once per CTA
  const int32_t* gate;     // nullptr, or the launch does nothing unless *gate != 0
  const int32_t* mbd;      // nullptr, or C's needed rows per batch entry: tiles at m0 >= mbd exit
  const int32_t* nbd;      // nullptr, or C's needed columns per batch entry: tiles at n0 >= nbd exit
  const int32_t* kbd;      // nullptr, or the reduction extent per batch entry (k-blocks past it skipped)
  int db_per_batch;        // 1: bounds indexed by the batch entry; 0: entry 0 for every batch entry
};

// the device-side bounds of zgemm.h DevBounds, evaluated uniformly by the whole CTA
#define TRAJ_DEV_BOUNDS(n0)                                      \
  if (args.gate && *args.gate == 0) return;                      \
  const int dbz_ = args.db_per_batch ? z : 0;                    \
  if (args.nbd && (n0) >= args.nbd[dbz_]) return;                \
  if (args.mbd && m0 >= args.mbd[dbz_]) return;                  \
  const int Kz = args.kbd ? min(args.K, args.kbd[dbz_]) : args.K;

// byte offset of complex element (r, k) in a k-contiguous tile: line r, chunk k (swizzled)
__device__ __forceinline__ uint32_t off_kc(int r, int k) { return r * 128 + ((k ^ (r & 7)) << 4); }
// byte offset in an m/n-contiguous tile made of [8 k-lines][8 complex] 1 KB sub-boxes
__device__ __forceinline__ uint32_t off_mn(int r, int k) {
  return (r >> 3) * 1024 + k * 128 + (((r & 7) ^ k) << 4);
}

template <bool CONJ_A, bool CONJ_B>
__global__ void __launch_bounds__(THREADS, 1)
    zgemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const Args args) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the 128B swizzle, by pointer arithmetic so loads stay LDS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  // ---- tile coordinates (grouped raster for L2 reuse of the A row-panel)
  const int t = blockIdx.x;
  const int group = GROUP_M * args.tiles_n;
  const int first_m = (t / group) * GROUP_M;
  const int gm = min(GROUP_M, args.tiles_m - first_m);
  const int pid_m = first_m + (t % group) % gm;
  const int pid_n = (t % group) / gm;
  const int m0 = pid_m * BM, n0 = pid_n * BN;
  const int z = blockIdx.z;
  if ((args.flags & TRAJ_C_UPPER_F) && m0 + args.m_off > n0 + args.n_off + BN - 1) return;   // tile entirely below the diagonal
  TRAJ_DEV_BOUNDS(n0)

  int kb = 0, ke = Kz;
  if (args.flags & TRAJ_TRI_A_UPPER_F) kb = max(kb, m0 + args.m_off);
  if (args.flags & TRAJ_TRI_A_LOWER_F) ke = min(ke, m0 + args.m_off + BM);
  if (args.flags & TRAJ_TRI_B_UPPER_F) ke = min(ke, n0 + args.n_off + BN);
  if (args.flags & TRAJ_TRI_B_LOWER_F) kb = max(kb, n0 + args.n_off);
  const int nk = ke > kb ? (ke - kb + BKC - 1) / BKC : 0;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ================= TMA issue (warp 0, lane 0), STAGES-1 stages ahead
  const bool issuer = (warp == 0 && lane == 0);
  const int za = args.a_batched ? z : 0, zb = args.b_batched ? z : 0;
  auto issue = [&](int it) {
    const int s = it % STAGES;
    mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
    const int k0 = kb + it * BKC;
    uint8_t* sA = smem + s * STAGE_BYTES;
    uint8_t* sB = sA + A_BYTES;
    if (!CONJ_A) {
      tma_load_3d(sA, &tmA, 2 * k0, m0, za, &full[s]);                 // [BM rows][8 k]
    } else if (args.a_4d) {
      tma_load_4d(sA, &tmA, 0, k0, m0 / 8, za, &full[s]);              // [BM/8 chunks][8 k][8 m]
    } else {
#pragma unroll
      for (int c = 0; c < BM / 8; ++c) tma_load_3d(sA + c * 1024, &tmA, 2 * (m0 + 8 * c), k0, za, &full[s]);
    }
    if (CONJ_B) {
      tma_load_3d(sB, &tmB, 2 * k0, n0, zb, &full[s]);                 // [BN rows][8 k]
    } else if (args.b_4d) {
      tma_load_4d(sB, &tmB, 0, k0, n0 / 8, zb, &full[s]);              // [BN/8 chunks][8 k][8 n]
    } else {
#pragma unroll
      for (int c = 0; c < BN / 8; ++c) tma_load_3d(sB + c * 1024, &tmB, 2 * (n0 + 8 * c), k0, zb, &full[s]);
    }
  };
  // Stage x reuses the slot of stage x-STAGES, free once all 8 warps released it.  The
  // issuer polls (test_wait) instead of blocking so that warp 0 is not held back by the
  // slowest warp; it blocks only if the stage it is about to consume is not in flight.
  int issued = 0;
  auto try_issue = [&](int it, bool must) {
    while (issued < nk && issued <= it + STAGES - 1) {
      if (issued >= STAGES) {
        const uint32_t par = ((issued / STAGES) + 1) & 1;
        if (must && issued <= it) mbar_wait(&empty[issued % STAGES], par);
        else if (!mbar_test(&empty[issued % STAGES], par)) break;
      }
      issue(issued);
      ++issued;
    }
  };
  if (issuer) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    try_issue(0, true);
  }

  // ================= DMMA consumers
  const int warp_m = warp & 3, warp_n = warp >> 2;
  const int g = lane >> 2;          // fragment row (A) / column (B)
  const int slot = lane & 3;        // k slot of the 8x8x4 MMA
  const int c = slot & 1;           // component of the interleaved complex k
  const int khalf = (slot >> 1) * 4;
  constexpr unsigned long long SIGN = 0x8000000000000000ull;
  // A1 = [a_r, -sa*sb*a_i]: flip the imaginary lane when sa*sb = +1
  const unsigned long long mask1 = (c == 1 && CONJ_A == CONJ_B) ? SIGN : 0ull;
  // A2 = [sb*a_r, sa*a_i]
  const unsigned long long mask2 = ((c == 0 && CONJ_B) || (c == 1 && CONJ_A)) ? SIGN : 0ull;

  double acc[4][4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int p = 0; p < 2; ++p) acc[i][j][p][0] = acc[i][j][p][1] = 0.0;

  for (int it = 0; it < nk; ++it) {
    const int s = it % STAGES;
    if (issuer) try_issue(it, true);
    mbar_wait(&full[s], (it / STAGES) & 1);
    const uint8_t* sA = smem + s * STAGE_BYTES;
    const uint8_t* sB = sA + A_BYTES;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = q + khalf;
      unsigned long long a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = warp_m * 32 + 8 * i + g;
        const uint32_t o = (CONJ_A ? off_mn(r, k) : off_kc(r, k)) + 8 * c;
        a[i] = *reinterpret_cast<const unsigned long long*>(sA + o);
      }
      double b1[4], b2[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = warp_n * 32 + 8 * j + g;
        const uint32_t o = CONJ_B ? off_kc(r, k) : off_mn(r, k);
        b1[j] = *reinterpret_cast<const double*>(sB + o + 8 * c);
        b2[j] = *reinterpret_cast<const double*>(sB + o + 8 * (1 - c));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double a1 = __longlong_as_double((long long)(a[i] ^ mask1));
        const double a2 = __longlong_as_double((long long)(a[i] ^ mask2));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma_8x8x4(acc[i][j][0][0], acc[i][j][0][1], a1, b1[j]);
          dmma_8x8x4(acc[i][j][1][0], acc[i][j][1][1], a2, b2[j]);
        }
      }
      if (q == 1 && issuer) try_issue(it, false);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ---- epilogue: thread holds C(row g, cols 2*slot, 2*slot+1) of each 8x8 block
  cplx* C = args.C + (long long)z * args.strideC;
  const bool upper = args.flags & TRAJ_C_UPPER_F;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + warp_m * 32 + 8 * i + g;
    if (row >= args.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + warp_n * 32 + 8 * j + 2 * slot + e;
        if (col >= args.N || (upper && row + args.m_off > col + args.n_off)) continue;
        const double vr = acc[i][j][0][e], vi = acc[i][j][1][e];
        double2 out;
        out.x = args.alpha_re * vr - args.alpha_im * vi;
        out.y = args.alpha_re * vi + args.alpha_im * vr;
        cplx* p = C + (long long)row * args.ldc + col;
        if (args.beta != 0.0) {
          const double2 old = *p;
          out.x += args.beta * old.x;
          out.y += args.beta * old.y;
        }
        *p = out;
      }
    }
  }
}


// ------------------------------------------------------------------ 3M (Gauss) variant
// op(A) = A' = a_r + i a_i', op(B) = B' = b_r + i b_i' (a_i' = sa a_i, b_i' = sb b_i):
//   P1 = a_r b_r,  P2 = a_i' b_i',  P3 = (a_r + a_i')(b_r + b_i')
//   Re C = P1 - P2,  Im C = P3 - P1 - P2
// Three real DMMA products over the complex k axis instead of four over the interleaved
// one: 6mnk instead of 8mnk tensor-pipe flops, the same FP64 arithmetic (the standard
// ZGEMM3M trade: the imaginary part's error bound carries |a_r|+|a_i| factors).
// CTA 64 x 64, 8 warps of 32 x 16 (three accumulator sets: 96 registers); a stage holds 16
// complex k as two 8-k sub-tiles per operand (6 stages of 32 KB).  MMA k-step q takes complex
// k = (q & 1) + 2 s of sub-tile q >> 1 for k-slot s: rows m, m+1 of a quarter-warp then hit
// chunks of opposite parity, so the 128-bit fragment loads of all layouts are conflict free.
// Fragments of the next k-step are loaded before the current k-step's MMAs.
namespace g3 {
constexpr int BM = 64, BN = 64, STAGES = 6, KSUB = 2;
constexpr int A_SUB = BM * 128, B_SUB = BN * 128;
constexpr int A_BYTES = KSUB * A_SUB, B_BYTES = KSUB * B_SUB, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8;
}  // namespace g3

template <bool CONJ_A, bool CONJ_B>
__global__ void __launch_bounds__(THREADS, 1)
    zgemm3m_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const Args args) {
  constexpr int BM3 = g3::BM, BN3 = g3::BN, ST3 = g3::STAGES, SB3 = g3::STAGE_BYTES;
  constexpr int KS = BKC * g3::KSUB;     // complex k per stage
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST3 * SB3);
  uint64_t* empty = full + ST3;
  const int t = blockIdx.x;
  const int group = GROUP_M * args.tiles_n;
  const int first_m = (t / group) * GROUP_M;
  const int gm = min(GROUP_M, args.tiles_m - first_m);
  const int pid_m = first_m + (t % group) % gm;
  const int pid_n = (t % group) / gm;
  const int m0 = pid_m * BM3, n0 = pid_n * BN3;
  const int z = blockIdx.z;
  if ((args.flags & TRAJ_C_UPPER_F) && m0 + args.m_off > n0 + args.n_off + BN3 - 1) return;
  TRAJ_DEV_BOUNDS(n0)
  int kb = 0, ke = Kz;
  if (args.flags & TRAJ_TRI_A_UPPER_F) kb = max(kb, m0 + args.m_off);
  if (args.flags & TRAJ_TRI_A_LOWER_F) ke = min(ke, m0 + args.m_off + BM3);
  if (args.flags & TRAJ_TRI_B_UPPER_F) ke = min(ke, n0 + args.n_off + BN3);
  if (args.flags & TRAJ_TRI_B_LOWER_F) kb = max(kb, n0 + args.n_off);
  const int nk = ke > kb ? (ke - kb + KS - 1) / KS : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST3; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const bool issuer = (warp == 0 && lane == 0);
  const int za = args.a_batched ? z : 0, zb = args.b_batched ? z : 0;
  auto issue = [&](int it) {
    const int s = it % ST3;
    mbar_arrive_expect_tx(&full[s], SB3);
#pragma unroll
    for (int h = 0; h < g3::KSUB; ++h) {
      const int k0 = kb + it * KS + h * BKC;
      uint8_t* sA = smem + s * SB3 + h * g3::A_SUB;
      uint8_t* sB = smem + s * SB3 + g3::A_BYTES + h * g3::B_SUB;
      if (!CONJ_A) {
        tma_load_3d(sA, &tmA, 2 * k0, m0, za, &full[s]);
      } else if (args.a_4d) {
        tma_load_4d(sA, &tmA, 0, k0, m0 / 8, za, &full[s]);
      } else {
#pragma unroll
        for (int c = 0; c < BM3 / 8; ++c) tma_load_3d(sA + c * 1024, &tmA, 2 * (m0 + 8 * c), k0, za, &full[s]);
      }
      if (CONJ_B) {
        tma_load_3d(sB, &tmB, 2 * k0, n0, zb, &full[s]);
      } else if (args.b_4d) {
        tma_load_4d(sB, &tmB, 0, k0, n0 / 8, zb, &full[s]);
      } else {
#pragma unroll
        for (int c = 0; c < BN3 / 8; ++c) tma_load_3d(sB + c * 1024, &tmB, 2 * (n0 + 8 * c), k0, zb, &full[s]);
      }
    }
  };
  int issued = 0;
  auto try_issue = [&](int it, bool must) {
    while (issued < nk && issued <= it + ST3 - 1) {
      if (issued >= ST3) {
        const uint32_t par = ((issued / ST3) + 1) & 1;
        if (must && issued <= it) mbar_wait(&empty[issued % ST3], par);
        else if (!mbar_test(&empty[issued % ST3], par)) break;
      }
      issue(issued);
      ++issued;
    }
  };
  if (issuer) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    try_issue(0, true);
  }
  const int warp_m = warp & 1, warp_n = warp >> 1;    // 2 x 4 warps of 32 x 16
  const int g = lane >> 2, slot = lane & 3;
  constexpr unsigned long long SIGN = 0x8000000000000000ull;
  constexpr unsigned long long ma = CONJ_A ? SIGN : 0ull, mb = CONJ_B ? SIGN : 0ull;
  double acc[4][2][3][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int p = 0; p < 3; ++p) acc[i][j][p][0] = acc[i][j][p][1] = 0.0;
  // fragment address for k-step q: k = (q & 1) + 2*slot in sub-tile q >> 1.  The swizzle
  // XORs the chunk with (row & 7) for k-contiguous tiles and (k) for m/n-contiguous ones;
  // (q & 1) flips bit 0 of k, handled by recomputing the offset.
  auto addrA = [&](const uint8_t* base, int q, int i) -> const double2* {
    const int r = warp_m * 32 + 8 * i + g, k = (q & 1) + 2 * slot;
    return reinterpret_cast<const double2*>(base + (q >> 1) * g3::A_SUB +
                                            (CONJ_A ? off_mn(r, k) : off_kc(r, k)));
  };
  auto addrB = [&](const uint8_t* base, int q, int j) -> const double2* {
    const int r = warp_n * 16 + 8 * j + g, k = (q & 1) + 2 * slot;
    return reinterpret_cast<const double2*>(base + g3::A_BYTES + (q >> 1) * g3::B_SUB +
                                            (CONJ_B ? off_kc(r, k) : off_mn(r, k)));
  };
  for (int it = 0; it < nk; ++it) {
    const int s = it % ST3;
    if (issuer) try_issue(it, true);
    mbar_wait(&full[s], (it / ST3) & 1);
    const uint8_t* base = smem + s * SB3;
    double2 va[4], vb[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) va[i] = *addrA(base, 0, i);
#pragma unroll
    for (int j = 0; j < 2; ++j) vb[j] = *addrB(base, 0, j);
#pragma unroll
    for (int q = 0; q < 2 * g3::KSUB; ++q) {
      double a1[4], a2[4], a3[4], b1[2], b2[2], b3[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a1[i] = va[i].x;
        a2[i] = __longlong_as_double((long long)((unsigned long long)__double_as_longlong(va[i].y) ^ ma));
        a3[i] = a1[i] + a2[i];
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        b1[j] = vb[j].x;
        b2[j] = __longlong_as_double((long long)((unsigned long long)__double_as_longlong(vb[j].y) ^ mb));
        b3[j] = b1[j] + b2[j];
      }
      if (q + 1 < 2 * g3::KSUB) {      // prefetch the next k-step's fragments
#pragma unroll
        for (int i = 0; i < 4; ++i) va[i] = *addrA(base, q + 1, i);
#pragma unroll
        for (int j = 0; j < 2; ++j) vb[j] = *addrB(base, q + 1, j);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma_8x8x4(acc[i][j][0][0], acc[i][j][0][1], a1[i], b1[j]);
          dmma_8x8x4(acc[i][j][1][0], acc[i][j][1][1], a2[i], b2[j]);
        }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][2][0], acc[i][j][2][1], a3[i], b3[j]);
      if (q == 1 && issuer) try_issue(it, false);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  cplx* C = args.C + (long long)z * args.strideC;
  const bool upper = args.flags & TRAJ_C_UPPER_F;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + warp_m * 32 + 8 * i + g;
    if (row >= args.M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + warp_n * 16 + 8 * j + 2 * slot + e;
        if (col >= args.N || (upper && row + args.m_off > col + args.n_off)) continue;
        const double p1 = acc[i][j][0][e], p2 = acc[i][j][1][e], p3 = acc[i][j][2][e];
        const double vr = p1 - p2, vi = p3 - p1 - p2;
        double2 out;
        out.x = args.alpha_re * vr - args.alpha_im * vi;
        out.y = args.alpha_re * vi + args.alpha_im * vr;
        cplx* pc = C + (long long)row * args.ldc + col;
        if (args.beta != 0.0) {
          const double2 old = *pc;
          out.x += args.beta * old.x;
          out.y += args.beta * old.y;
        }
        *pc = out;
      }
    }
  }
}

// Wide variant: CTA 128 x 64, 8 warps of 32 x 32 (three accumulator sets = 192 registers, the
// fragments loaded per k-step without a prefetch buffer), 4 stages of 48 KB.
namespace g3w {
constexpr int BM = 128, BN = 64, STAGES = 4, KSUB = 2;
constexpr int A_SUB = BM * 128, B_SUB = BN * 128;
constexpr int A_BYTES = KSUB * A_SUB, B_BYTES = KSUB * B_SUB, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8;
}  // namespace g3w

template <bool CONJ_A, bool CONJ_B>
__global__ void __launch_bounds__(THREADS, 1)
    zgemm3mw_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const Args args) {
  constexpr int BM3 = g3w::BM, BN3 = g3w::BN, ST3 = g3w::STAGES, SB3 = g3w::STAGE_BYTES;
  constexpr int KS = BKC * g3w::KSUB;     // complex k per stage
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST3 * SB3);
  uint64_t* empty = full + ST3;
  const int t = blockIdx.x;
  const int group = GROUP_M * args.tiles_n;
  const int first_m = (t / group) * GROUP_M;
  const int gm = min(GROUP_M, args.tiles_m - first_m);
  const int pid_m = first_m + (t % group) % gm;
  const int pid_n = (t % group) / gm;
  const int m0 = pid_m * BM3, n0 = pid_n * BN3;
  const int z = blockIdx.z;
  if ((args.flags & TRAJ_C_UPPER_F) && m0 + args.m_off > n0 + args.n_off + BN3 - 1) return;
  TRAJ_DEV_BOUNDS(n0)
  int kb = 0, ke = Kz;
  if (args.flags & TRAJ_TRI_A_UPPER_F) kb = max(kb, m0 + args.m_off);
  if (args.flags & TRAJ_TRI_A_LOWER_F) ke = min(ke, m0 + args.m_off + BM3);
  if (args.flags & TRAJ_TRI_B_UPPER_F) ke = min(ke, n0 + args.n_off + BN3);
  if (args.flags & TRAJ_TRI_B_LOWER_F) kb = max(kb, n0 + args.n_off);
  const int nk = ke > kb ? (ke - kb + KS - 1) / KS : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST3; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const bool issuer = (warp == 0 && lane == 0);
  const int za = args.a_batched ? z : 0, zb = args.b_batched ? z : 0;
  auto issue = [&](int it) {
    const int s = it % ST3;
    mbar_arrive_expect_tx(&full[s], SB3);
#pragma unroll
    for (int h = 0; h < g3w::KSUB; ++h) {
      const int k0 = kb + it * KS + h * BKC;
      uint8_t* sA = smem + s * SB3 + h * g3w::A_SUB;
      uint8_t* sB = smem + s * SB3 + g3w::A_BYTES + h * g3w::B_SUB;
      if (!CONJ_A) {
        tma_load_3d(sA, &tmA, 2 * k0, m0, za, &full[s]);
      } else if (args.a_4d) {
        tma_load_4d(sA, &tmA, 0, k0, m0 / 8, za, &full[s]);
      } else {
#pragma unroll
        for (int c = 0; c < BM3 / 8; ++c) tma_load_3d(sA + c * 1024, &tmA, 2 * (m0 + 8 * c), k0, za, &full[s]);
      }
      if (CONJ_B) {
        tma_load_3d(sB, &tmB, 2 * k0, n0, zb, &full[s]);
      } else if (args.b_4d) {
        tma_load_4d(sB, &tmB, 0, k0, n0 / 8, zb, &full[s]);
      } else {
#pragma unroll
        for (int c = 0; c < BN3 / 8; ++c) tma_load_3d(sB + c * 1024, &tmB, 2 * (n0 + 8 * c), k0, zb, &full[s]);
      }
    }
  };
  int issued = 0;
  auto try_issue = [&](int it, bool must) {
    while (issued < nk && issued <= it + ST3 - 1) {
      if (issued >= ST3) {
        const uint32_t par = ((issued / ST3) + 1) & 1;
        if (must && issued <= it) mbar_wait(&empty[issued % ST3], par);
        else if (!mbar_test(&empty[issued % ST3], par)) break;
      }
      issue(issued);
      ++issued;
    }
  };
  if (issuer) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    try_issue(0, true);
  }
  const int warp_m = warp & 3, warp_n = warp >> 2;    // 4 x 2 warps of 32 x 32
  const int g = lane >> 2, slot = lane & 3;
  constexpr unsigned long long SIGN = 0x8000000000000000ull;
  constexpr unsigned long long ma = CONJ_A ? SIGN : 0ull, mb = CONJ_B ? SIGN : 0ull;
  double acc[4][4][3][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int p = 0; p < 3; ++p) acc[i][j][p][0] = acc[i][j][p][1] = 0.0;
  // fragment address for k-step q: k = (q & 1) + 2*slot in sub-tile q >> 1.  The swizzle
  // XORs the chunk with (row & 7) for k-contiguous tiles and (k) for m/n-contiguous ones;
  // (q & 1) flips bit 0 of k, handled by recomputing the offset.
  auto addrA = [&](const uint8_t* base, int q, int i) -> const double2* {
    const int r = warp_m * 32 + 8 * i + g, k = (q & 1) + 2 * slot;
    return reinterpret_cast<const double2*>(base + (q >> 1) * g3w::A_SUB +
                                            (CONJ_A ? off_mn(r, k) : off_kc(r, k)));
  };
  auto addrB = [&](const uint8_t* base, int q, int j) -> const double2* {
    const int r = warp_n * 32 + 8 * j + g, k = (q & 1) + 2 * slot;
    return reinterpret_cast<const double2*>(base + g3w::A_BYTES + (q >> 1) * g3w::B_SUB +
                                            (CONJ_B ? off_kc(r, k) : off_mn(r, k)));
  };
  for (int it = 0; it < nk; ++it) {
    const int s = it % ST3;
    if (issuer) try_issue(it, true);
    mbar_wait(&full[s], (it / ST3) & 1);
    const uint8_t* base = smem + s * SB3;
#pragma unroll
    for (int q = 0; q < 2 * g3w::KSUB; ++q) {
      double2 va[4], vb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) va[i] = *addrA(base, q, i);
#pragma unroll
      for (int j = 0; j < 4; ++j) vb[j] = *addrB(base, q, j);
      if (CONJ_A) {   // sign-bit XOR (ALU), not a DADD negation on the FP64 pipe
#pragma unroll
        for (int i = 0; i < 4; ++i)
          va[i].y = __longlong_as_double((long long)((unsigned long long)__double_as_longlong(va[i].y) ^ ma));
      }
      if (CONJ_B) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          vb[j].y = __longlong_as_double((long long)((unsigned long long)__double_as_longlong(vb[j].y) ^ mb));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma_8x8x4(acc[i][j][0][0], acc[i][j][0][1], va[i].x, vb[j].x);
          dmma_8x8x4(acc[i][j][1][0], acc[i][j][1][1], va[i].y, vb[j].y);
        }
      double b3[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) b3[j] = vb[j].x + vb[j].y;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double a3 = va[i].x + va[i].y;
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][2][0], acc[i][j][2][1], a3, b3[j]);
      }
      if (q == 1 && issuer) try_issue(it, false);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  cplx* C = args.C + (long long)z * args.strideC;
  const bool upper = args.flags & TRAJ_C_UPPER_F;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + warp_m * 32 + 8 * i + g;
    if (row >= args.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + warp_n * 32 + 8 * j + 2 * slot + e;
        if (col >= args.N || (upper && row + args.m_off > col + args.n_off)) continue;
        const double p1 = acc[i][j][0][e], p2 = acc[i][j][1][e], p3 = acc[i][j][2][e];
        const double vr = p1 - p2, vi = p3 - p1 - p2;
        double2 out;
        out.x = args.alpha_re * vr - args.alpha_im * vi;
        out.y = args.alpha_re * vi + args.alpha_im * vr;
        cplx* pc = C + (long long)row * args.ldc + col;
        if (args.beta != 0.0) {
          const double2 old = *pc;
          out.x += args.beta * old.x;
          out.y += args.beta * old.y;
        }
        *pc = out;
      }
    }
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t get_encode() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}

// Map a batch of row-major complex matrices [rows][cols] (ld, batch stride in complex
// elements) as a 3D FP64 tensor {2*cols, rows, batch} with boxes {16, box_rows, 1}.
bool make_map(CUtensorMap* map, const void* base, long long rows, long long cols, long long ld, long long stride,
              long long batch, int box_rows) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return false;
  const bool batched = stride != 0 && batch > 1;
  cuuint64_t dims[3] = {(cuuint64_t)(2 * cols), (cuuint64_t)rows, (cuuint64_t)(batched ? batch : 1)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 16), (cuuint64_t)((batched ? stride : ld * rows) * 16)};
  cuuint32_t box[3] = {16, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// m/n-contiguous operand [rows = k][cols] as a 4D tensor {16 doubles, rows, chunks of 8
// complex (stride 128 B), batch}; one box {16, 8, box_chunks, 1} fills a whole stage tile.
// Column chunks are read whole, so this is used only when round_up(cols, 8) <= ld (the
// extra columns then stay inside each row and only feed discarded outputs).
bool make_map_4d(CUtensorMap* map, const void* base, long long rows, long long cols, long long ld, long long stride,
                 long long batch, int box_chunks) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return false;
  const bool batched = stride != 0 && batch > 1;
  cuuint64_t dims[4] = {16, (cuuint64_t)rows, (cuuint64_t)ceil_div(cols, 8), (cuuint64_t)(batched ? batch : 1)};
  cuuint64_t strides[3] = {(cuuint64_t)(ld * 16), 128, (cuuint64_t)((batched ? stride : ld * rows) * 16)};
  cuuint32_t box[4] = {16, 8, (cuuint32_t)box_chunks, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool CA, bool CB>
cudaError_t launch(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const Args& args, int batch) {
  {
    cudaError_t e = ensure_smem((const void*)zgemm_dmma_kernel<CA, CB>, SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(args.tiles_m * args.tiles_n, 1, batch);
  zgemm_dmma_kernel<CA, CB><<<grid, THREADS, SMEM_BYTES, st>>>(a, b, args);
  count_launch();
  return cudaGetLastError();
}

template <bool CA, bool CB>
cudaError_t launch3m(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const Args& args, int batch) {
  {
    cudaError_t e = ensure_smem((const void*)zgemm3m_dmma_kernel<CA, CB>, g3::SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(args.tiles_m * args.tiles_n, 1, batch);
  zgemm3m_dmma_kernel<CA, CB><<<grid, THREADS, g3::SMEM_BYTES, st>>>(a, b, args);
  count_launch();
  return cudaGetLastError();
}

template <bool CA, bool CB>
cudaError_t launch3mw(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const Args& args, int batch) {
  {
    cudaError_t e = ensure_smem((const void*)zgemm3mw_dmma_kernel<CA, CB>, g3w::SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(args.tiles_m * args.tiles_n, 1, batch);
  zgemm3mw_dmma_kernel<CA, CB><<<grid, THREADS, g3w::SMEM_BYTES, st>>>(a, b, args);
  count_launch();
  return cudaGetLastError();
}

std::atomic<int> g_algo{-1};

}  // namespace

int zgemm_algorithm() {
  int a = g_algo.load();
  if (a < 0) {
    const char* e = getenv("TRAJ_ZGEMM_3M");     // default 3M; TRAJ_ZGEMM_3M=0 selects 4M
    a = (e && e[0] == '0') ? 0 : 1;
    g_algo.store(a);
  }
  return a;
}

void set_zgemm_algorithm(int algo) { g_algo.store(algo ? 1 : 0); }

int zgemm(cudaStream_t st, int opA, int opB, long long M, long long N, long long K, double alpha_re,
          double alpha_im, const cplx* A, long long lda, long long strideA, const cplx* B, long long ldb,
          long long strideB, double beta, cplx* C, long long ldc, long long strideC, long long batch, int flags,
          std::string* err, long long m_off, long long n_off, const DevBounds* db) {
  if (M <= 0 || N <= 0 || batch <= 0) return 0;
  if (M > (1ll << 30) || N > (1ll << 30) || K > (1ll << 30) || batch > 65535) {
    if (err) *err = "zgemm: dimension too large";
    return 1;
  }
  if (K > 0 && (lda <= 0 || ldb <= 0 || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))) {
    if (err) *err = "zgemm: bad lda/ldb or misaligned operand";
    return 1;
  }
  CUtensorMap ma, mb;
  const long long Ka = K > 0 ? K : 1;
  int algo = zgemm_algorithm();
  // 3M shape policy: the 128 x 64 (32 x 32 warp tiles) variant for large N x N products
  // (better fragment reuse; K.U +3%), the 64 x 64 one otherwise (Gram upper tiles, skinny and
  // small GEMMs of the Cholesky recursion get more CTAs and less diagonal waste)
  if (algo == 1 && opA == 0 && opB == 0 && ceil_div(M, g3w::BM) * ceil_div(N, g3w::BN) * batch >= 4 * 148) algo = 2;
  const bool m3 = algo >= 1;
  const int bm = algo == 2 ? g3w::BM : (m3 ? g3::BM : BM), bn = algo == 2 ? g3w::BN : (m3 ? g3::BN : BN);
  // op(A) = A: stored [M][K], k-contiguous tile [BM rows][8 k]; op(A) = A^dag: stored [K][M].
  const bool a4 = opA == 1 && round_up(M, 8) <= lda && !getenv("TRAJ_NO_TMA4D");
  const bool b4 = opB == 0 && round_up(N, 8) <= ldb && !getenv("TRAJ_NO_TMA4D");
  bool ok = opA == 0 ? make_map(&ma, A, M, Ka, lda, strideA, batch, bm)
                     : (a4 ? make_map_4d(&ma, A, Ka, M, lda, strideA, batch, bm / 8)
                           : make_map(&ma, A, Ka, M, lda, strideA, batch, 8));
  ok = ok && (opB == 0 ? (b4 ? make_map_4d(&mb, B, Ka, N, ldb, strideB, batch, bn / 8)
                             : make_map(&mb, B, Ka, N, ldb, strideB, batch, 8))
                       : make_map(&mb, B, N, Ka, ldb, strideB, batch, bn));
  if (!ok) {
    if (err) *err = "zgemm: cuTensorMapEncodeTiled failed";
    return 4;
  }
  Args args;
  args.M = (int)M;
  args.N = (int)N;
  args.K = (int)K;
  args.tiles_m = (int)ceil_div(M, bm);
  args.tiles_n = (int)ceil_div(N, bn);
  args.flags = flags;
  args.a_batched = strideA != 0 && batch > 1;
  args.b_batched = strideB != 0 && batch > 1;
  args.a_4d = a4;
  args.b_4d = b4;
  args.alpha_re = alpha_re;
  args.alpha_im = alpha_im;
  args.beta = beta;
  args.C = C;
  args.ldc = ldc;
  args.strideC = strideC;
  args.m_off = (int)m_off;
  args.n_off = (int)n_off;
  args.gate = db ? db->gate : nullptr;
  args.nbd = db ? db->n : nullptr;
  args.mbd = db ? db->m : nullptr;
  args.kbd = db ? db->k : nullptr;
  args.db_per_batch = db ? db->per_batch : 0;
  cudaError_t e;
  if (algo == 2) {
    if (opA == 0 && opB == 0) e = launch3mw<false, false>(st, ma, mb, args, (int)batch);
    else if (opA == 0) e = launch3mw<false, true>(st, ma, mb, args, (int)batch);
    else if (opB == 0) e = launch3mw<true, false>(st, ma, mb, args, (int)batch);
    else e = launch3mw<true, true>(st, ma, mb, args, (int)batch);
  } else if (m3) {
    if (opA == 0 && opB == 0) e = launch3m<false, false>(st, ma, mb, args, (int)batch);
    else if (opA == 0) e = launch3m<false, true>(st, ma, mb, args, (int)batch);
    else if (opB == 0) e = launch3m<true, false>(st, ma, mb, args, (int)batch);
    else e = launch3m<true, true>(st, ma, mb, args, (int)batch);
  } else if (opA == 0 && opB == 0) e = launch<false, false>(st, ma, mb, args, (int)batch);
  else if (opA == 0) e = launch<false, true>(st, ma, mb, args, (int)batch);
  else if (opB == 0) e = launch<true, false>(st, ma, mb, args, (int)batch);
  else e = launch<true, true>(st, ma, mb, args, (int)batch);
  if (e != cudaSuccess) {
    if (err) *err = std::string("zgemm launch: ") + cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

}  // namespace traj
