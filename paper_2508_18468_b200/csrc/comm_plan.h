// Point-to-point schedules of the row-sharded step, as plain host data.
//
// The NCCL executor in shard.cu walks exactly these lists, and traj_comm_plan (traj.h) exports
// them so that the pairing can be checked without GPUs: tests/test_comm_plan.py matches every
// rank's list under NCCL's rule (operations between one pair of ranks pair up in issue order)
// and runs them with torch.distributed send/recv on gloo, world sizes 2 and 4.
//
// Host code only; no CUDA, no NCCL.
#pragma once
#include <algorithm>
#include <cmath>
#include <vector>

namespace traj {

enum { COMM_SEND = 0, COMM_RECV = 1 };

struct CommOp {
  int group;   // ops of one group are issued between one ncclGroupStart / ncclGroupEnd
  int kind;    // COMM_SEND / COMM_RECV
  int peer;    // the other rank
  int slot;    // which local buffer: propagate -- 0 = own U block (send) or Ufull block `block` (recv);
               // halo -- 0 = low edge / low halo, 1 = high edge / high halo
  int block;   // global identity of the data moved (what the receiver must end up holding)
};

// a1 with the exchange fused into the chunked K_g U (shard.cu propagate_dense): for ring distance
// d = 1 .. P-1 (group d - 1), rank g sends its own U block (identity g) to g + d and receives block
// g - d from g - d; the K-chunk product of distance d waits only for group d - 1.
inline std::vector<CommOp> ring_plan(int P, int g) {
  std::vector<CommOp> ops;
  for (int d = 1; d < P; ++d) {
    const int to = (g + d) % P, from = (g - d + P) % P;
    ops.push_back({d - 1, COMM_SEND, to, 0, g});
    ops.push_back({d - 1, COMM_RECV, from, 0, from});
  }
  return ops;
}

// NEXT-1 banded propagator with sharding: the W-row halos from the two ring neighbours, one group.
// Edge identities: low edge of rank r = 2r, high edge = 2r + 1.  The low halo of g is the high
// edge of g - 1, its high halo the low edge of g + 1.  Sends go (high edge -> right, low edge ->
// left) and receives (low halo <- left, high halo <- right): with P <= 2 left == right, and this
// order makes the first message each way the high edge, the second the low edge, on both sides.
inline std::vector<CommOp> halo_plan(int P, int g) {
  const int left = (g + P - 1) % P, right = (g + 1) % P;
  return {{0, COMM_SEND, right, 1, 2 * g + 1},
          {0, COMM_SEND, left, 0, 2 * g},
          {0, COMM_RECV, left, 0, 2 * left + 1},
          {0, COMM_RECV, right, 1, 2 * right}};
}


// Row slices [b[i], b[i+1]) of M rows over P ranks, 128-aligned; tri: equal area of an upper
// triangle (the Hermitian update).  Used by the distributed Cholesky (cholinv.cu dist_gemm): rank i
// computes slice i, then one broadcast per non-empty slice (root i) re-replicates the block.
inline std::vector<long long> row_slices(long long M, int P, bool tri) {
  std::vector<long long> b(P + 1, 0);
  for (int i = 1; i < P; ++i) {
    const double f = (double)i / P;
    const double x = tri ? M * (1.0 - std::sqrt(1.0 - f)) : M * f;
    b[i] = std::min(M, std::max(b[i - 1], (long long)(x / 128.0 + 0.5) * 128));
  }
  b[P] = M;
  return b;
}

// Leaf size and split point of the Cholesky recursion (cholinv.cu): h = 64 ceil(ceil(n / 64) / 2).
constexpr int CHOL_NB = 64;
inline long long chol_split(long long n) {
  const long long nb = (n + CHOL_NB - 1) / CHOL_NB;
  return CHOL_NB * ((nb + 1) / 2);
}

// The broadcasts the distributed Cholesky of an n x n Gram issues on every rank, in order: one
// entry (root, rows, cols) per non-empty slice of each of the four split GEMMs of every recursion
// level with size >= min_n (rec() in cholinv.cu: level (o, n) -> A = (o, h), then the products
// R_B^dag [r x h], C -= R_B^dag R_B [r x r, triangle], then C = (o + h, r), then R_B X_C [h x r],
// X_B [h x r]).  NCCL requires the same sequence on every rank.
struct BcastOp {
  int root;
  long long rows, cols;
};
inline void dist_chol_plan_rec(long long n, int P, long long min_n, std::vector<BcastOp>* out) {
  if (n <= CHOL_NB) return;
  const long long h = chol_split(n), r = n - h;
  dist_chol_plan_rec(h, P, min_n, out);
  if (P > 1 && n >= min_n) {
    auto share = [&](long long M, long long cols, bool tri) {
      const std::vector<long long> b = row_slices(M, P, tri);
      for (int i = 0; i < P; ++i)
        if (b[i + 1] > b[i]) out->push_back({i, b[i + 1] - b[i], cols});
    };
    share(r, h, false);
    share(r, r, true);
    dist_chol_plan_rec(r, P, min_n, out);
    share(h, r, false);
    share(h, r, false);
    return;
  }
  dist_chol_plan_rec(r, P, min_n, out);
}

}  // namespace traj
