// INT8 tensor-core GEMM for sm_100a: tcgen05.mma.kind::i8, accumulators in TMEM, operands staged by
// TMA as 128B-swizzled K-major tiles, one persistent CTA per SM.
//
// C_z = A_z B_z^T (A_z: M x K, B_z: N x K, both K-major int8), exact in int32.  This is the building
// block of the modular complex-FP64 products (ozaki.cu): each residue product is one batch entry and
// the epilogue reduces the exact int32 dot product mod that entry's modulus.
//
// CTA: 192 threads, warp 0 = TMA producer, warp 1 = MMA issuer (one elected lane) and TMEM owner,
// warps 2..5 = epilogue (warp w reads TMEM lanes 32 (w % 4) .. + 31: one accumulator row per thread).
// Tile 128 x 256 x 128 (one MMA 128 x 256 x 32 per 32 bytes of k), 4-stage smem ring of 48 KB,
// two 256-column TMEM accumulators so the epilogue of tile t overlaps the MMAs of tile t + 1.
#include "igemm.h"
#include <algorithm>
#include <cstdlib>

namespace traj {
namespace {

// IGEMM_BK: bytes of k per pipeline stage (128: 128B-swizzled rows, 4 stages; 64: 64B-swizzled rows,
// 8 stages of half the size -- finer refill granularity for the same bytes in flight)
#ifndef IGEMM_BK
#define IGEMM_BK 128
#endif
constexpr int IBM = 128, IBN = 256, IBK = IGEMM_BK, ISTAGES = 4 * 128 / IGEMM_BK;
constexpr int SW_ROW = IGEMM_BK;                       // swizzle span = one row of a stage
constexpr uint32_t SW_LAYOUT = IGEMM_BK == 128 ? 2 : 4;  // SWIZZLE_128B / SWIZZLE_64B descriptor codes
constexpr int IA_BYTES = IBM * IBK, IB_BYTES = IBN * IBK, ISTAGE_BYTES = IA_BYTES + IB_BYTES;
constexpr int ITHREADS = 192;
// the unpaired kernel: IEPI epilogue warps, two per TMEM lane quarter, each taking half of the tile's
// 256 accumulator columns -- the epilogue of a shallow tile (few k-blocks) is a serial chain of TMEM
// loads, reductions and stores that the MMAs of the next tile no longer hide with one warp per quarter
#ifndef IGEMM_EPI_WARPS
#define IGEMM_EPI_WARPS 8
#endif
constexpr int IEPI = IGEMM_EPI_WARPS;
constexpr int IMAIN_THREADS = 64 + 32 * IEPI;
constexpr int ISMEM = ISTAGES * ISTAGE_BYTES + 1024 + 256;
// raster: tiles are taken in groups of `gm` m-blocks (m fastest) so that a wave of CTAs shares A and B
// slabs through L2 (TRAJ_IGEMM_GM overrides the default for experiments)
constexpr int IGM = 16;

// K-major operand, 128-byte rows, 128B swizzle (8-row atoms of 1 KB): SBO = 1024 B, version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)((8 * SW_ROW) >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)SW_LAYOUT << 61);
}

// instruction descriptor: D s32, A s8, B s8, both K-major, N >> 3 at bit 17, M >> 4 at bit 24
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct KArgs {
  int M, N, K;
  int tiles_m, tiles_n;
  long long tiles;       // batch * tiles_m * tiles_n
  int a_div, b_div, a_batched, b_batched;
  void* C;
  long long ldc, strideC;
  int out;
  const int* moduli;
  int nmod;
  int flags;
  int gm;
  int oz_s, oz_T, oz_a_traj, oz_b_traj;
  int oz_pa[3], oz_pb[3];
  const int32_t* gate;
  const int32_t* kdev;
  const int32_t* ndev;
  int ksplit, kcb;   // k chunks, k-blocks per chunk
  int barrett_kb;    // tiles of at most this many k-blocks reduce mod m in integer arithmetic (ModRed)
};

// batch entry z -> (A entry, B entry, modulus index)
__device__ __forceinline__ void zmap(const KArgs& a, int z, int& za, int& zb, int& q) {
  if (a.oz_s) {
    const int t = z % a.oz_T, pq = z / a.oz_T;
    const int p = pq / a.oz_s;
    q = pq - p * a.oz_s;
    za = a.oz_a_traj ? (a.oz_pa[p] * a.oz_s + q) * a.oz_T + t : a.oz_pa[p] * a.oz_s + q;
    zb = a.oz_b_traj ? (a.oz_pb[p] * a.oz_s + q) * a.oz_T + t : a.oz_pb[p] * a.oz_s + q;
  } else {
    za = a.a_batched ? z / a.a_div : 0;
    zb = a.b_batched ? z / a.b_div : 0;
    q = z % a.nmod;
  }
}

struct Tile {
  int z, kc, mb, nb;
};

__device__ __forceinline__ Tile tile_of(const KArgs& a, long long t) {
  const long long per = (long long)a.tiles_m * a.tiles_n;
  Tile r;
  const long long zk = t / per;
  r.z = (int)(zk / a.ksplit);
  r.kc = (int)(zk - (long long)r.z * a.ksplit);
  const int rem = (int)(t - zk * per);
  const int gsz = a.gm * a.tiles_n;
  const int g = rem / gsz, first = g * a.gm;
  const int h = min(a.gm, a.tiles_m - first), w = rem - g * gsz;
  r.mb = first + w % h;
  r.nb = w / h;
  return r;
}

__device__ __forceinline__ int traj_of(const KArgs& a, int z) { return a.oz_s ? z % a.oz_T : z; }

__device__ __forceinline__ bool tile_live(const KArgs& a, const Tile& t) {
  if ((a.flags & IG_UPPER) && (t.nb + 1) * IBN - 1 < t.mb * IBM) return false;
  if (a.ndev && t.nb * IBN >= a.ndev[traj_of(a, t.z)]) return false;
  return true;
}

// the tile's k-blocks [kb0, kb0 + count)
__device__ __forceinline__ int tile_kblocks(const KArgs& a, const Tile& t, int* kb0 = nullptr) {
  int kend = a.K;
  if (a.flags & IG_TRI_B) kend = min(kend, (t.nb + 1) * IBN);
  if (a.kdev) kend = min(kend, a.kdev[traj_of(a, t.z)]);
  const int nkb = (kend + IBK - 1) / IBK;
  const int b0 = t.kc * a.kcb;
  if (kb0) *kb0 = b0;
  return max(0, min(nkb, b0 + a.kcb) - b0);
}

// x mod m (m <= 256) of an exact int32 accumulator (|x| <= K 2^14 < 2^30 for K <= 65536) by Barrett
// reduction on u = x + k0 (k0 the least multiple of m >= 2^30, so 0 <= u < 2^32): q = hi32(u floor(2^32 / m))
// is floor(u / m) or one less, r = u - q m in [0, 2m), one conditional subtract (as min(r, r - m) in
// unsigned arithmetic).  Integer multiply-adds only: the FP64 floor it replaces ran three conversions
// per value, which bounded the epilogue of short-K tiles.
// The FP64 form (x - m floor(x / m)) is kept for deep tiles (more than barrett_kb k-blocks, e.g. the
// K U product), whose epilogue hides under the MMAs anyway: measured, the integer form there costs
// ~3% of the INT8 rate (c3 K U 59.5 -> 61.7 ms), the power of the extra ALU work under a power-limited
// tensor pipe.
struct ModRed {
  uint32_t m = 1, magic = 0, k0 = 0;
  double inv = 0.0;
  bool barrett = true;
  __device__ __forceinline__ void set(int mod, bool use_barrett) {
    m = (uint32_t)mod;
    magic = (uint32_t)(0x100000000ull / (unsigned long long)mod);
    k0 = m * ((0x40000000u + m - 1) / m);
    barrett = use_barrett;
    if (!barrett) inv = 1.0 / (double)mod;
  }
  __device__ __forceinline__ uint32_t operator()(int x) const {
    const uint32_t u = (uint32_t)x + k0;
    const uint32_t r = u - __umulhi(u, magic) * m;
    return min(r, r - m);
  }
  // 32 accumulators -> 32 residue bytes packed four per word
  __device__ __forceinline__ void pack32(const uint32_t* v, uint32_t* w) const {
    if (barrett) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t packed = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) packed |= (*this)((int)v[4 * j + b]) << (8 * b);
        w[j] = packed;
      }
    } else {
      const int mi = (int)m;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t packed = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int x = (int)v[4 * j + b];
          int r = x - mi * (int)floor((double)x * inv);
          r += (r < 0) ? mi : 0;
          r -= (r >= mi) ? mi : 0;
          packed |= (uint32_t)r << (8 * b);
        }
        w[j] = packed;
      }
    }
  }
};

__global__ void __launch_bounds__(IMAIN_THREADS, 1)
    igemm_i8_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, const KArgs a) {
  if (a.gate && *a.gate == 0) return;   // uniform over the grid: no TMEM allocated, no barrier used
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + ISTAGES * ISTAGE_BYTES);
  uint64_t* empty = full + ISTAGES;
  uint64_t* tfull = empty + ISTAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ISTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], IEPI);
    }
    fence_mbar_init();
    prefetch_tmap(&ta);
    prefetch_tmap(&tb);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (long long t = blockIdx.x; t < a.tiles; t += gridDim.x) {
        const Tile tl = tile_of(a, t);
        if (!tile_live(a, tl)) continue;
        int kb0;
        const int nk = tile_kblocks(a, tl, &kb0);
        int za, zb, q;
        zmap(a, tl.z, za, zb, q);
        for (int kb = kb0; kb < kb0 + nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = base + stage * ISTAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], ISTAGE_BYTES);
          tma_load_3d(sa, &ta, kb * IBK, tl.mb * IBM, za, &full[stage]);
          tma_load_3d(sa + IA_BYTES, &tb, kb * IBK, tl.nb * IBN, zb, &full[stage]);
          if (++stage == ISTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {   // ---------------- MMA issuer
    constexpr uint32_t idesc = idesc_i8(IBM, IBN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (long long t = blockIdx.x; t < a.tiles; t += gridDim.x) {
      const Tile tl = tile_of(a, t);
      if (!tile_live(a, tl)) continue;
      const int nk = tile_kblocks(a, tl);
      const int buf = it & 1;
      const uint32_t use = (uint32_t)(it >> 1);
      mbar_wait(&tempty[buf], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t dt = tmem + buf * IBN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = base_u32 + stage * ISTAGE_BYTES, sb = sa + IA_BYTES;
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sb);
#pragma unroll
          for (int k = 0; k < IBK / 32; ++k)   // +32 bytes of k = +2 in the descriptor's address field
            mma_i8(dt, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == ISTAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) mma_commit(&tfull[buf]);
      __syncwarp();
      ++it;
    }
  } else {   // ---------------- epilogue: warps 2 .. 2 + IEPI - 1
    const int q = warp & 3;
    constexpr int CPW = (IBN / 32) * 4 / IEPI;   // 32-column chunks per warp
    const int c_lo = ((warp - 2) >> 2) * CPW;
    int it = 0;
    for (long long t = blockIdx.x; t < a.tiles; t += gridDim.x) {
      const Tile tl = tile_of(a, t);
      if (!tile_live(a, tl)) continue;
      const int buf = it & 1;
      const uint32_t use = (uint32_t)(it >> 1);
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const int row = tl.mb * IBM + q * 32 + lane;
      const bool row_ok = row < a.M;
      const bool kzero = tile_kblocks(a, tl) == 0;   // empty contraction: the accumulator was never written
      const uint32_t taddr = tmem + buf * IBN + ((uint32_t)(q * 32) << 16);
      int mod = 0;
      ModRed red;
      if (a.out != IG_OUT_I32) {
        int za, zb, q;
        zmap(a, tl.z, za, zb, q);
        mod = a.moduli[q];
        red.set(mod, tile_kblocks(a, tl) <= a.barrett_kb);
      }
#pragma unroll 1
      for (int c = c_lo; c < c_lo + CPW; ++c) {
        uint32_t v[32];
        __syncwarp();
        tmem_ld32(taddr + c * 32, v);
        if (kzero) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0;
        }
        const int col = tl.nb * IBN + c * 32;
        if (!row_ok || col >= a.N) {
        } else if (a.out == IG_OUT_I32) {
          int* p = reinterpret_cast<int*>(a.C) + ((long long)tl.z * a.ksplit + tl.kc) * a.strideC +
                   (long long)row * a.ldc + col;
          if (col + 32 <= a.N) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<int4*>(p)[j] = make_int4((int)v[4 * j], (int)v[4 * j + 1], (int)v[4 * j + 2], (int)v[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < a.N) p[j] = (int)v[j];
          }
        } else {
          uint32_t w[8];
          red.pack32(v, w);
          uint8_t* p = reinterpret_cast<uint8_t*>(a.C) + ((long long)tl.z * a.ksplit + tl.kc) * a.strideC +
                       (long long)row * a.ldc + col;
          if (a.out == IG_OUT_MOD_ACC) {   // add the residues already there (< m each), reduce once more
            uint32_t old[8];
            if (col + 32 <= a.N) {
              const uint4 o0 = reinterpret_cast<const uint4*>(p)[0], o1 = reinterpret_cast<const uint4*>(p)[1];
              old[0] = o0.x; old[1] = o0.y; old[2] = o0.z; old[3] = o0.w;
              old[4] = o1.x; old[5] = o1.y; old[6] = o1.z; old[7] = o1.w;
            } else {
              for (int jj = 0; jj < 8; ++jj) old[jj] = 0;
#pragma unroll
              for (int jj = 0; jj < 32; ++jj)
                if (col + jj < a.N) old[jj >> 2] |= (uint32_t)p[jj] << (8 * (jj & 3));
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              uint32_t packed = 0;
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                uint32_t r = ((w[j] >> (8 * b)) & 0xff) + ((old[j] >> (8 * b)) & 0xff);
                r -= r >= (uint32_t)mod ? (uint32_t)mod : 0u;
                packed |= r << (8 * b);
              }
              w[j] = packed;
            }
          }
          if (col + 32 <= a.N) {
            reinterpret_cast<uint4*>(p)[0] = make_uint4(w[0], w[1], w[2], w[3]);
            reinterpret_cast<uint4*>(p)[1] = make_uint4(w[4], w[5], w[6], w[7]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < a.N) p[j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2): a cluster of two CTAs computes 256 x 256 tiles; each CTA
// stages its 128 rows of A and its 128 rows (n) of B per 128-k block, the leader's elected lane
// issues 256 x 256 x 32 MMAs that read both CTAs' shared memory, and each CTA's TMEM holds its 128
// accumulator rows x 256 columns.  A stage is 32 KB per SM (against 48 KB unpaired), so six stages
// hold 1.5x the k-depth of the unpaired ring and each SM reads a third fewer operand bytes per MAC.
constexpr int PBM = 256, PBN = 256, PSTAGES = 6 * 128 / IGEMM_BK;
constexpr int PA_BYTES = 128 * IBK, PB_BYTES = 128 * IBK, PSTAGE_BYTES = PA_BYTES + PB_BYTES;
constexpr int PSMEM = PSTAGES * PSTAGE_BYTES + 1024 + 256;
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;   // clears the CTA-rank bit of a shared::cluster address

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar) & PEER_MASK)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {   // arrives at this offset in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {   // the rank-0 CTA's copy of this barrier
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ra) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ Tile pair_tile_of(const KArgs& a, long long t, int tiles_m2) {
  const long long per = (long long)tiles_m2 * a.tiles_n;
  Tile r;
  const long long zk = t / per;
  r.z = (int)(zk / a.ksplit);
  r.kc = (int)(zk - (long long)r.z * a.ksplit);
  const int rem = (int)(t - zk * per);
  const int gm = max(1, a.gm / 2);
  const int gsz = gm * a.tiles_n;
  const int g = rem / gsz, first = g * gm;
  const int h = min(gm, tiles_m2 - first), w = rem - g * gsz;
  r.mb = first + w % h;   // in units of 256 rows
  r.nb = w / h;
  return r;
}
__device__ __forceinline__ bool pair_tile_live(const KArgs& a, const Tile& t) {
  if ((a.flags & IG_UPPER) && (t.nb + 1) * PBN - 1 < t.mb * PBM) return false;
  if (a.ndev && t.nb * PBN >= a.ndev[traj_of(a, t.z)]) return false;
  return true;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ITHREADS, 1)
    igemm_i8_pair_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, const KArgs a,
                         const int tiles_m2, const long long ptiles) {
  if (a.gate && *a.gate == 0) return;   // uniform over the grid (both CTAs of every pair)
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + PSTAGES * PSTAGE_BYTES);
  uint64_t* empty = full + PSTAGES;
  uint64_t* tfull = empty + PSTAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < PSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);   // four epilogue warps in each CTA of the pair (used in the leader)
    }
    fence_mbar_init();
    prefetch_tmap(&ta);
    prefetch_tmap(&tb);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer (both CTAs; bytes land on the leader's barrier)
      int stage = 0;
      uint32_t phase = 0;
      for (long long t = pair; t < ptiles; t += npairs) {
        const Tile tl = pair_tile_of(a, t, tiles_m2);
        if (!pair_tile_live(a, tl)) continue;
        int kb0;
        const int nk = tile_kblocks(a, tl, &kb0);
        int za, zb, q;
        zmap(a, tl.z, za, zb, q);
        for (int kb = kb0; kb < kb0 + nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = base + stage * PSTAGE_BYTES;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * PSTAGE_BYTES);
          tma_load_3d_pair(sa, &ta, kb * IBK, tl.mb * PBM + (int)rank * 128, za, &full[stage]);
          tma_load_3d_pair(sa + PA_BYTES, &tb, kb * IBK, tl.nb * PBN + (int)rank * 128, zb, &full[stage]);
          if (++stage == PSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {   // ---------------- MMA issuer (leader CTA only)
      constexpr uint32_t idesc = idesc_i8(PBM, PBN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (long long t = pair; t < ptiles; t += npairs) {
        const Tile tl = pair_tile_of(a, t, tiles_m2);
        if (!pair_tile_live(a, tl)) continue;
        const int nk = tile_kblocks(a, tl);
        const int buf = it & 1;
        const uint32_t use = (uint32_t)(it >> 1);
        mbar_wait_cluster(&tempty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem + buf * PBN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = base_u32 + stage * PSTAGE_BYTES, sb = sa + PA_BYTES;
            const uint64_t da = sw128_desc(sa), db = sw128_desc(sb);
#pragma unroll
            for (int k = 0; k < IBK / 32; ++k) mma_i8_pair(dt, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
            mma_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == PSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) mma_commit_pair(&tfull[buf]);
        __syncwarp();
        ++it;
      }
    }
  } else {   // ---------------- epilogue: warps 2..5 of each CTA, its 128 rows
    const int q = warp & 3;
    int it = 0;
    for (long long t = pair; t < ptiles; t += npairs) {
      const Tile tl = pair_tile_of(a, t, tiles_m2);
      if (!pair_tile_live(a, tl)) continue;
      const int buf = it & 1;
      const uint32_t use = (uint32_t)(it >> 1);
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const int row = tl.mb * PBM + (int)rank * 128 + q * 32 + lane;
      const bool row_ok = row < a.M;
      const bool kzero = tile_kblocks(a, tl) == 0;
      const uint32_t taddr = tmem + buf * PBN + ((uint32_t)(q * 32) << 16);
      int mod = 0;
      ModRed red;
      if (a.out == IG_OUT_MOD) {
        int za, zb, qq;
        zmap(a, tl.z, za, zb, qq);
        mod = a.moduli[qq];
        red.set(mod, tile_kblocks(a, tl) <= a.barrett_kb);
      }
#pragma unroll 1
      for (int c = 0; c < PBN / 32; ++c) {
        uint32_t v[32];
        __syncwarp();
        tmem_ld32(taddr + c * 32, v);
        if (kzero) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0;
        }
        const int col = tl.nb * PBN + c * 32;
        if (!row_ok || col >= a.N) {
        } else if (a.out == IG_OUT_I32) {
          int* p = reinterpret_cast<int*>(a.C) + ((long long)tl.z * a.ksplit + tl.kc) * a.strideC +
                   (long long)row * a.ldc + col;
          if (col + 32 <= a.N) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<int4*>(p)[j] = make_int4((int)v[4 * j], (int)v[4 * j + 1], (int)v[4 * j + 2], (int)v[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < a.N) p[j] = (int)v[j];
          }
        } else {
          uint32_t w[8];
          red.pack32(v, w);
          uint8_t* p = reinterpret_cast<uint8_t*>(a.C) + ((long long)tl.z * a.ksplit + tl.kc) * a.strideC +
                       (long long)row * a.ldc + col;
          if (col + 32 <= a.N) {
            reinterpret_cast<uint4*>(p)[0] = make_uint4(w[0], w[1], w[2], w[3]);
            reinterpret_cast<uint4*>(p)[1] = make_uint4(w[4], w[5], w[6], w[7]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < a.N) p[j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[buf]);
      ++it;
    }
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------------------------
// B-multicast variant: a cluster of two CTAs on adjacent m-blocks of the same n-block; each CTA loads
// its own A tile and half of the shared B tile, multicast into both CTAs' shared memory (each CTA's
// L2 reads per stage 32 KB instead of 48 KB).  MMAs, TMEM and the epilogue stay per CTA (cta_group::1);
// a stage is refilled only when both CTAs' MMAs have consumed it (commits multicast to both empties).
__device__ __forceinline__ void tma_load_3d_mc(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2,
                                               uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar) {   // arrives at this offset in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ITHREADS, 1)
    igemm_i8_mc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, const KArgs a,
                       const int tiles_m2, const long long ptiles) {
  if (a.gate && *a.gate == 0) return;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + ISTAGES * ISTAGE_BYTES);
  uint64_t* empty = full + ISTAGES;
  uint64_t* tfull = empty + ISTAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_rank();
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ISTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);   // both CTAs' MMAs
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_mbar_init();
    prefetch_tmap(&ta);
    prefetch_tmap(&tb);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // this CTA's tile of the pair tile: m-block 2 mb2 + rank (the pair is live when either tile is)
  auto my_tile = [&](long long t, bool& live, bool& mine) {
    Tile tl = pair_tile_of(a, t, tiles_m2);
    Tile t0 = tl, t1 = tl;
    t0.mb = 2 * tl.mb;
    t1.mb = 2 * tl.mb + 1;
    const bool l0 = tile_live(a, t0), l1 = t1.mb < a.tiles_m && tile_live(a, t1);
    live = l0 || l1;
    mine = rank ? l1 : l0;
    return rank ? t1 : t0;
  };
  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (long long t = pair; t < ptiles; t += npairs) {
        bool live, mine;
        const Tile tl = my_tile(t, live, mine);
        if (!live) continue;
        int kb0;
        const int nk = tile_kblocks(a, tl, &kb0);
        int za, zb, q;
        zmap(a, tl.z, za, zb, q);
        for (int kb = kb0; kb < kb0 + nk; ++kb) {
          mbar_wait_cluster(&empty[stage], phase ^ 1);
          uint8_t* sa = base + stage * ISTAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], ISTAGE_BYTES);
          tma_load_3d(sa, &ta, kb * IBK, tl.mb * IBM, za, &full[stage]);
          tma_load_3d_mc(sa + IA_BYTES + rank * (IB_BYTES / 2), &tb, kb * IBK, tl.nb * IBN + rank * (IBN / 2), zb,
                         &full[stage], (uint16_t)3);
          if (++stage == ISTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {   // ---------------- MMA issuer
    constexpr uint32_t idesc = idesc_i8(IBM, IBN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (long long t = pair; t < ptiles; t += npairs) {
      bool live, mine;
      const Tile tl = my_tile(t, live, mine);
      if (!live) continue;
      const int nk = tile_kblocks(a, tl);
      const int buf = it & 1;
      const uint32_t use = (uint32_t)(it >> 1);
      mbar_wait(&tempty[buf], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t dt = tmem + buf * IBN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = base_u32 + stage * ISTAGE_BYTES, sb = sa + IA_BYTES;
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sb);
#pragma unroll
          for (int k = 0; k < IBK / 32; ++k) mma_i8(dt, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          mma_commit_mc(&empty[stage]);
        }
        __syncwarp();
        if (++stage == ISTAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) mma_commit(&tfull[buf]);
      __syncwarp();
      ++it;
    }
  } else {   // ---------------- epilogue: warps 2..5
    const int q = warp & 3;
    int it = 0;
    for (long long t = pair; t < ptiles; t += npairs) {
      bool live, mine;
      const Tile tl = my_tile(t, live, mine);
      if (!live) continue;
      const int buf = it & 1;
      const uint32_t use = (uint32_t)(it >> 1);
      mbar_wait(&tfull[buf], use & 1);
      tc_fence_after();
      const int row = tl.mb * IBM + q * 32 + lane;
      const bool row_ok = mine && row < a.M;
      const bool kzero = tile_kblocks(a, tl) == 0;
      const uint32_t taddr = tmem + buf * IBN + ((uint32_t)(q * 32) << 16);
      int mod = 0;
      ModRed red;
      if (a.out == IG_OUT_MOD) {
        int za, zb, qq;
        zmap(a, tl.z, za, zb, qq);
        mod = a.moduli[qq];
        red.set(mod, tile_kblocks(a, tl) <= a.barrett_kb);
      }
#pragma unroll 1
      for (int c = 0; c < IBN / 32; ++c) {
        uint32_t v[32];
        __syncwarp();
        tmem_ld32(taddr + c * 32, v);
        if (kzero) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0;
        }
        const int col = tl.nb * IBN + c * 32;
        if (!row_ok || col >= a.N) {
        } else if (a.out == IG_OUT_I32) {
          int* p = reinterpret_cast<int*>(a.C) + ((long long)tl.z * a.ksplit + tl.kc) * a.strideC +
                   (long long)row * a.ldc + col;
          if (col + 32 <= a.N) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<int4*>(p)[j] = make_int4((int)v[4 * j], (int)v[4 * j + 1], (int)v[4 * j + 2], (int)v[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < a.N) p[j] = (int)v[j];
          }
        } else {
          uint32_t w[8];
          red.pack32(v, w);
          uint8_t* p = reinterpret_cast<uint8_t*>(a.C) + ((long long)tl.z * a.ksplit + tl.kc) * a.strideC +
                       (long long)row * a.ldc + col;
          if (col + 32 <= a.N) {
            reinterpret_cast<uint4*>(p)[0] = make_uint4(w[0], w[1], w[2], w[3]);
            reinterpret_cast<uint4*>(p)[1] = make_uint4(w[4], w[5], w[6], w[7]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < a.N) p[j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      ++it;
    }
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

typedef CUresult (*PFN_encode_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encode_t encode_i8() {
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

bool map_i8(PFN_encode_t enc, CUtensorMap* m, const int8_t* p, long long K, long long rows, long long ld, long long nb,
            long long stride, int box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)nb};
  cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)(nb > 1 ? stride : ld * rows)};
  cuuint32_t box[3] = {IBK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, IGEMM_BK == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

int igemm(cudaStream_t st, const IgemmArgs& g, std::string* err) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return 0;
  if (g.K <= 0 || g.K >= (1 << 17) || g.M >= (1LL << 31) || g.N >= (1LL << 31) || (g.lda & 15) || (g.ldb & 15) ||
      g.lda < g.K || g.ldb < g.K || (g.ldc & 15) || g.ldc < g.N || g.a_div < 1 || g.b_div < 1 ||
      g.batch % g.a_div || g.batch % g.b_div || (reinterpret_cast<uintptr_t>(g.A) & 15) ||
      (reinterpret_cast<uintptr_t>(g.B) & 15) || (reinterpret_cast<uintptr_t>(g.C) & 15) ||
      (g.out != IG_OUT_I32 && g.out != IG_OUT_MOD && g.out != IG_OUT_MOD_ACC) ||
      (g.out != IG_OUT_I32 && (!g.moduli || g.nmod < 1))) {
    if (err) *err = "igemm: needs 0 < K < 2^17, lda/ldb multiples of 16 >= K, ldc a multiple of 16 >= N, 16-B alignment";
    return 1;
  }
  PFN_encode_t enc = encode_i8();
  if (!enc) {
    if (err) *err = "igemm: cuTensorMapEncodeTiled unavailable";
    return 4;
  }
  const long long na = g.oz_s ? g.oz_na : g.batch / g.a_div, nb = g.oz_s ? g.oz_nb : g.batch / g.b_div;
  const bool ab = g.strideA != 0 && na > 1, bb = g.strideB != 0 && nb > 1;
  if (g.oz_s && (g.oz_np < 1 || g.oz_np > 3 || g.batch != (long long)g.oz_np * g.oz_s * g.oz_T || g.oz_T < 1 || !g.moduli || g.out == IG_OUT_I32)) {
    if (err) *err = "igemm: modular batch map needs batch = np s T (np <= 3) and the modular epilogue";
    return 1;
  }
  // the CTA-pair kernel from 256 rows on.  Default (TRAJ_IGEMM_PAIR unset): paired for the triangular
  // products (IG_UPPER Grams, IG_TRI_B TRMMs: c3 Gram launch 17.2 -> 15.2 ms, TRMM 9.7 -> 8.1 ms), unpaired
  // for the dense ones -- on K U the pair kernel's wave misses L2 far more often (420 vs 98 GB of DRAM,
  // profiles/r02/igemm_pair_vs_single.txt; 56.0 -> 58.3 ms).  TRAJ_IGEMM_PAIR=1 / 0: always / never.
  static int pair_env = -2;
  if (pair_env == -2) {
    const char* v = getenv("TRAJ_IGEMM_PAIR");
    pair_env = !v || !v[0] ? -1 : (v[0] == '1' ? 1 : 0);
  }
  const bool pair_wanted = pair_env == 1 || (pair_env == -1 && (g.flags & (IG_UPPER | IG_TRI_B)) != 0);
  const bool use_pair = pair_wanted && g.M >= 256 && num_sms() >= 2 && g.out != IG_OUT_MOD_ACC;
  static int mc_env = -1;
  if (mc_env < 0) {
    const char* v = getenv("TRAJ_IGEMM_MC");
    mc_env = (v && v[0] == '1') ? 1 : 0;
  }
  const bool use_mc = !use_pair && mc_env && g.M >= 256 && num_sms() >= 2 && g.out != IG_OUT_MOD_ACC;
  CUtensorMap ma, mb;
  if (!map_i8(enc, &ma, g.A, g.K, g.M, g.lda, ab ? na : 1, g.strideA, IBM) ||
      !map_i8(enc, &mb, g.B, g.K, g.N, g.ldb, bb ? nb : 1, g.strideB, (use_pair || use_mc) ? 128 : IBN)) {
    if (err) *err = "igemm: tensor map";
    return 4;
  }
  KArgs a;
  a.M = (int)g.M;
  a.N = (int)g.N;
  a.K = (int)g.K;
  a.tiles_m = (int)ceil_div(g.M, IBM);
  a.tiles_n = (int)ceil_div(g.N, IBN);
  a.ksplit = std::max(1, g.ksplit);
  {
    const int nkb = (int)ceil_div(g.K, IBK);
    a.kcb = (int)ceil_div(nkb, a.ksplit);
  }
  a.tiles = g.batch * a.ksplit * a.tiles_m * a.tiles_n;
  a.a_div = g.a_div;
  a.b_div = g.b_div;
  a.a_batched = ab;
  a.b_batched = bb;
  a.C = g.C;
  a.ldc = g.ldc;
  a.strideC = g.strideC;
  a.out = g.out;
  a.moduli = g.moduli;
  a.nmod = g.nmod;
  a.flags = g.flags;
  {
    static int gm_env = -1;
    if (gm_env < 0) {
      const char* v = getenv("TRAJ_IGEMM_GM");
      gm_env = v ? std::max(1, atoi(v)) : 0;
    }
    // the upper-triangular (Gram) products: one group, column-major over all M-tiles (measured c3
    // Gram 19.3 -> 17.4 ms; the K U product keeps groups of IGM: 58.3 vs 62.0 ms with one group)
    a.gm = gm_env ? gm_env : ((g.flags & IG_UPPER) ? std::max(1, a.tiles_m) : IGM);
    static int bk_env = -2;
    if (bk_env == -2) {
      const char* v = getenv("TRAJ_IGEMM_BARRETT_KB");
      bk_env = v ? atoi(v) : -1;
    }
    a.barrett_kb = bk_env >= 0 ? bk_env : 64;
  }
  a.oz_s = g.oz_s;
  a.oz_T = g.oz_T;
  a.oz_a_traj = g.oz_a_traj;
  a.oz_b_traj = g.oz_b_traj;
  a.gate = g.gate;
  a.kdev = g.kdev;
  a.ndev = g.ndev;
  for (int i = 0; i < 3; ++i) {
    a.oz_pa[i] = g.oz_pa[i];
    a.oz_pb[i] = g.oz_pb[i];
  }
  if (use_pair) {
    const int tiles_m2 = (int)ceil_div(g.M, PBM);
    const long long ptiles = g.batch * a.ksplit * (long long)tiles_m2 * a.tiles_n;
    if (ensure_smem((const void*)igemm_i8_pair_kernel, PSMEM) != cudaSuccess) {
      if (err) *err = "igemm: shared memory attribute (pair)";
      return 4;
    }
    const long long npairs = std::min<long long>(ptiles, num_sms() / 2);
    igemm_i8_pair_kernel<<<(unsigned)(2 * npairs), ITHREADS, PSMEM, st>>>(ma, mb, a, tiles_m2, ptiles);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      if (err) *err = std::string("igemm (pair): ") + cudaGetErrorString(e);
      return 4;
    }
    return 0;
  }
  if (use_mc) {
    const int tiles_m2 = (int)ceil_div(a.tiles_m, 2);
    const long long ptiles = g.batch * a.ksplit * (long long)tiles_m2 * a.tiles_n;
    if (ensure_smem((const void*)igemm_i8_mc_kernel, ISMEM) != cudaSuccess) {
      if (err) *err = "igemm: shared memory attribute (multicast)";
      return 4;
    }
    const long long npairs = std::min<long long>(ptiles, num_sms() / 2);
    igemm_i8_mc_kernel<<<(unsigned)(2 * npairs), ITHREADS, ISMEM, st>>>(ma, mb, a, tiles_m2, ptiles);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      if (err) *err = std::string("igemm (multicast): ") + cudaGetErrorString(e);
      return 4;
    }
    return 0;
  }
  if (ensure_smem((const void*)igemm_i8_kernel, ISMEM) != cudaSuccess) {
    if (err) *err = "igemm: shared memory attribute";
    return 4;
  }
  const long long grid = std::min<long long>(a.tiles, num_sms());
  igemm_i8_kernel<<<(unsigned)grid, IMAIN_THREADS, ISMEM, st>>>(ma, mb, a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (err) *err = std::string("igemm: ") + cudaGetErrorString(e);
    return 4;
  }
  return 0;
}

}  // namespace traj
