// Real FP64 GEMM on the DMMA pipe for the planar 3M complex product (csrc/zgemm.cu's interleaved
// 3M keeps three accumulator sets per warp -- 192 registers, no room for larger warp tiles; the
// planar form runs the three real products P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi) as one
// batched real GEMM with a single accumulator set per warp).
//
// C_z = alpha op(A_z) B_z + beta C_z, row-major real matrices, z < batch.  CTA 128 x 128, 8 warps of
// 32 x 64 (64 accumulator doubles), 16 real k per stage, a 4-deep TMA ring (3, 5 and 6 stages and
// other refill points measured no better, tools/dgemm_bench.py) whose lane 0 of warp 0 issues;
// 128B-swizzled tiles: A [128 m][16 k] (one 3D box; op(A) = A^T: the 4D box of B), B [8 chunks of
// 16 n][16 k][16 n] (one 4D box).  DMMA m8n8k4: A fragment A[g][k], B fragment B[k][g], k = 4 q + slot.
#include <cuda.h>
#include <stdlib.h>

#include <string>

#include "common.cuh"
#include "dgemm.h"

namespace traj {

namespace {

constexpr int DBM = 128, DBN = 128, DBK = 16, DSTAGES = 4, DWARPS = 8, DTHREADS = DWARPS * 32;
constexpr int DA_BYTES = DBM * DBK * 8, DB_BYTES = DBK * DBN * 8, DSTAGE = DA_BYTES + DB_BYTES;
constexpr int DSMEM = DSTAGES * DSTAGE + 1024 + 2 * DSTAGES * 8;
constexpr int DGROUP_M = 8;

struct DArgs {
  int M, N, K;
  int tiles_m, tiles_n;
  int a_batched, b_batched;
  int a_div;               // batch entries per A entry (A_z = A entry z / a_div)
  int flags;               // DG_TRI_B_UPPER, DG_C_UPPER (dgemm.h)
  int m_off, n_off;        // global row / column of C(0, 0) for the triangle tests
  double alpha, beta;
  double* C;
  long long ldc, strideC;
};

// A(r, k) in a [rows][16 k] tile of 128-byte lines
__device__ __forceinline__ uint32_t doff_a(int r, int k) { return r * 128 + ((((k >> 1) ^ (r & 7))) << 4) + (k & 1) * 8; }
// B(k, n) in a [n / 16][16 k][16 n] tile
__device__ __forceinline__ uint32_t doff_b(int k, int n) {
  return ((n >> 4) * 16 + k) * 128 + (((((n & 15) >> 1) ^ (k & 7))) << 4) + (n & 1) * 8;
}

// TA: op(A) = A^T with A stored [K][M] (m-contiguous tiles, the same 4D box as B)
template <bool TA>
__global__ void __launch_bounds__(DTHREADS, 1)
    dgemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const DArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DSTAGES * DSTAGE);
  uint64_t* empty = full + DSTAGES;
  const int t = blockIdx.x;
  const int group = DGROUP_M * args.tiles_n;
  const int first_m = (t / group) * DGROUP_M;
  const int gm = min(DGROUP_M, args.tiles_m - first_m);
  const int m0 = (first_m + (t % group) % gm) * DBM, n0 = ((t % group) / gm) * DBN;
  const int z = blockIdx.z;
  if ((args.flags & DG_C_UPPER) && m0 + args.m_off > n0 + args.n_off + DBN - 1) return;   // below the diagonal
  int ke = args.K;
  if (args.flags & DG_TRI_B_UPPER) ke = min(ke, n0 + args.n_off + DBN);
  const int nk = (ke + DBK - 1) / DBK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < DSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], DWARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const bool issuer = warp == 0 && lane == 0;
  const int za = args.a_batched ? z / args.a_div : 0, zb = args.b_batched ? z : 0;
  auto issue = [&](int it) {
    const int s = it % DSTAGES;
    mbar_arrive_expect_tx(&full[s], DSTAGE);
    uint8_t* sA = smem + s * DSTAGE;
    if (TA) tma_load_4d(sA, &tmA, 0, it * DBK, m0 / 16, za, &full[s]);
    else tma_load_3d(sA, &tmA, it * DBK, m0, za, &full[s]);
    tma_load_4d(sA + DA_BYTES, &tmB, 0, it * DBK, n0 / 16, zb, &full[s]);
  };
  int issued = 0;
  auto try_issue = [&](int it, bool must) {
    while (issued < nk && issued <= it + DSTAGES - 1) {
      if (issued >= DSTAGES) {
        const uint32_t par = ((issued / DSTAGES) + 1) & 1;
        if (must && issued <= it) mbar_wait(&empty[issued % DSTAGES], par);
        else if (!mbar_test(&empty[issued % DSTAGES], par)) break;
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
  const int warp_m = warp & 3, warp_n = warp >> 2;   // 4 x 2 warps of 32 x 64
  const int g = lane >> 2, slot = lane & 3;
  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int it = 0; it < nk; ++it) {
    const int s = it % DSTAGES;
    if (issuer) try_issue(it, true);
    mbar_wait(&full[s], (it / DSTAGES) & 1);
    const uint8_t* sA = smem + s * DSTAGE;
    const uint8_t* sB = sA + DA_BYTES;
#pragma unroll
    for (int q = 0; q < DBK / 4; ++q) {
      const int k = 4 * q + slot;
      double a[4], b[8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        a[i] = *reinterpret_cast<const double*>(sA + (TA ? doff_b(k, warp_m * 32 + 8 * i + g)
                                                          : doff_a(warp_m * 32 + 8 * i + g, k)));
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = *reinterpret_cast<const double*>(sB + doff_b(k, warp_n * 64 + 8 * j + g));
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      if (q == 1 && issuer) try_issue(it, false);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  double* C = args.C + (long long)z * args.strideC;
  const bool upper = args.flags & DG_C_UPPER;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + warp_m * 32 + 8 * i + g;
    if (row >= args.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int col = n0 + warp_n * 64 + 8 * j + 2 * slot;
      double* p = C + (long long)row * args.ldc + col;
      if (upper && row + args.m_off > col + args.n_off) {   // one of the pair may still be on/above
        if (row + args.m_off <= col + 1 + args.n_off && col + 1 < args.N) {
          double v = args.alpha * acc[i][j][1];
          if (args.beta != 0.0) v += args.beta * p[1];
          p[1] = v;
        }
        continue;
      }
      if (col + 1 < args.N) {
        double2 v = make_double2(args.alpha * acc[i][j][0], args.alpha * acc[i][j][1]);
        if (args.beta != 0.0) {
          const double2 o = *reinterpret_cast<const double2*>(p);
          v.x += args.beta * o.x;
          v.y += args.beta * o.y;
        }
        *reinterpret_cast<double2*>(p) = v;
      } else if (col < args.N) {
        double v = args.alpha * acc[i][j][0];
        if (args.beta != 0.0) v += args.beta * p[0];
        p[0] = v;
      }
    }
  }
}

typedef CUresult (*PFN_encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encode_t encode_fn() {
  static PFN_encode_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encode_t>(p);
  }
  return fn;
}

}  // namespace

int dgemm(cudaStream_t st, int opA, long long M, long long N, long long K, double alpha, const double* A,
          long long lda, long long strideA, const double* B, long long ldb, long long strideB, double beta, double* C,
          long long ldc, long long strideC, long long batch, int flags, std::string* err, long long m_off,
          long long n_off, int a_div) {
  if (M <= 0 || N <= 0 || batch <= 0) return 0;
  if (K <= 0 || (lda & 1) || (ldb & 15) || round_up(N, 16) > ldb || (ldc & 1) ||
      (opA == 1 && ((lda & 15) || round_up(M, 16) > lda)) || (opA != 0 && opA != 1) ||
      (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) ||
      (reinterpret_cast<uintptr_t>(C) & 15) || batch > 65535) {
    if (err) *err = "dgemm: needs K > 0, even lda/ldc, ldb (and lda for op(A) = A^T) a multiple of 16 >= N (M) rounded up to 16, 16-B alignment";
    return 1;
  }
  PFN_encode_t enc = encode_fn();
  if (!enc) {
    if (err) *err = "dgemm: cuTensorMapEncodeTiled unavailable";
    return 4;
  }
  if (a_div < 1 || batch % a_div) {
    if (err) *err = "dgemm: a_div must divide the batch";
    return 1;
  }
  const long long na = batch / a_div;   // A entries
  const bool ab = strideA != 0 && na > 1, bb = strideB != 0 && batch > 1;
  CUtensorMap ma, mb;
  if (opA == 0) {
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)M, (cuuint64_t)(ab ? na : 1)};
    cuuint64_t strides[2] = {(cuuint64_t)(lda * 8), (cuuint64_t)((ab ? strideA : lda * M) * 8)};
    cuuint32_t box[3] = {DBK, DBM, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(A), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      if (err) *err = "dgemm: A tensor map";
      return 4;
    }
  } else {   // A stored [K][M]: 16-column chunks of m, like B
    cuuint64_t dims[4] = {16, (cuuint64_t)K, (cuuint64_t)ceil_div(M, 16), (cuuint64_t)(ab ? na : 1)};
    cuuint64_t strides[3] = {(cuuint64_t)(lda * 8), 128, (cuuint64_t)((ab ? strideA : lda * K) * 8)};
    cuuint32_t box[4] = {16, DBK, DBM / 16, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(A), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      if (err) *err = "dgemm: A^T tensor map";
      return 4;
    }
  }
  {
    cuuint64_t dims[4] = {16, (cuuint64_t)K, (cuuint64_t)ceil_div(N, 16), (cuuint64_t)(bb ? batch : 1)};
    cuuint64_t strides[3] = {(cuuint64_t)(ldb * 8), 128, (cuuint64_t)((bb ? strideB : ldb * K) * 8)};
    cuuint32_t box[4] = {16, DBK, DBN / 16, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(B), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      if (err) *err = "dgemm: B tensor map";
      return 4;
    }
  }
  DArgs args;
  args.M = (int)M;
  args.N = (int)N;
  args.K = (int)K;
  args.tiles_m = (int)ceil_div(M, DBM);
  args.tiles_n = (int)ceil_div(N, DBN);
  args.a_batched = ab;
  args.a_div = a_div;
  args.b_batched = bb;
  args.flags = flags;
  args.m_off = (int)m_off;
  args.n_off = (int)n_off;
  args.alpha = alpha;
  args.beta = beta;
  args.C = C;
  args.ldc = ldc;
  args.strideC = strideC;
  {
    const void* kern = opA ? (const void*)dgemm_dmma_kernel<true> : (const void*)dgemm_dmma_kernel<false>;
    if (ensure_smem(kern, DSMEM) != cudaSuccess) {
      if (err) *err = "dgemm: shared memory attribute";
      return 4;
    }
  }
  dim3 grid((unsigned)(args.tiles_m * args.tiles_n), 1, (unsigned)batch);
  if (opA) dgemm_dmma_kernel<true><<<grid, DTHREADS, DSMEM, st>>>(ma, mb, args);
  else dgemm_dmma_kernel<false><<<grid, DTHREADS, DSMEM, st>>>(ma, mb, args);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (err) *err = std::string("dgemm: ") + cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

}  // namespace traj
