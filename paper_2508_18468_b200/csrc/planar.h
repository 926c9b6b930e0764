// Internal interface of the planar 3M propagator (planar.cu): K and U as (re, im, re + im) planes,
// three real GEMMs (dgemm.cu), then (P1 - P2) + i (P3 - P1 - P2).
#pragma once
#include <algorithm>
#include <string>
#include "common.cuh"

namespace traj {

// Kp planes [3][nrows][ld] (plane stride ps) of rows [row0, row0 + nrows) of K = kx (x) ky (Lx*Ly
// sites, row-major site = y Lx + x); nrows < 0: all L rows
int build_k_planar(cudaStream_t st, double* Kp, long long ld, long long ps, int Lx, int Ly, const cplx* kx,
                   const cplx* ky, std::string* err, long long row0 = 0, long long nrows = -1);
// Pl[t][p][row][col] (plane stride ps, trajectory stride ts) = (re, im, re + im)[p] of U[t][row][col]
int split_planes(cudaStream_t st, const cplx* U, long long ldu, long long sU, int L, int N, int T, double* Pl,
                 long long ldp, long long ps, long long ts, std::string* err);
// U[t][row][col] = (P1 - P2) + i (P3 - P1 - P2) from Pl[t][0..2]
int combine_planes(cudaStream_t st, const double* Pl, long long ldp, long long ps, long long ts, int L, int N, int T,
                   cplx* U, long long ldu, long long sU, std::string* err);

// Pl[t][0..5] = (re, im, re - im, re, im, re + im) of U[t]
int split6_planes(cudaStream_t st, const cplx* U, long long ldu, long long sU, int L, int N, int T, double* Pl,
                  long long ldp, long long ps, long long ts, std::string* err);
// upper triangle of G[t] (n x n) = (P1 + Q2) + i (P3 - P1 + Q2) from Pl[t][0..2]
int combine_gram(cudaStream_t st, const double* Pl, long long ldp, long long ps, long long ts, int n, int T, cplx* G,
                 long long ldg, long long sG, std::string* err);

// products per plane x 3 planes for `levels` Strassen levels
inline int strassen_products(int levels) { return 3 * (levels >= 3 ? 343 : (levels == 2 ? 49 : 7)); }

// Strassen on each planar product, `levels` = 1, 2 or 3 (planar.cu), leaf grid h = L / 2^levels,
// nh = N / 2^levels, NS = 7^levels products per plane: Ks [3][NS][h][ldks] = K's operands (once);
// Bc [3][NS][T][h][ldb] = U's operands; U[t] = the recombined product from Mb (Bc's layout).
// K is L x L, U L x N: L and N divisible by 2^levels.
int strassen_k(cudaStream_t st, int levels, const double* Kp, long long ldk, long long pk, int L, double* Ks,
               long long ldks, std::string* err);
int strassen_b(cudaStream_t st, int levels, const cplx* U, long long ldu, long long sU, int L, int N, int T,
               double* Bc, long long ldb, std::string* err);
int strassen_c(cudaStream_t st, int levels, const double* Mb, long long ldb, int L, int N, int T, cplx* U,
               long long ldu, long long sU, std::string* err, int accumulate = 0);   // accumulate: U +=

// the column panel [c0, c1) of the Gram, rows [0, c1), combined from the planes Pl[0..2] into the
// contiguous buf [c1][w] (upper triangle; zeros below the diagonal) for a packed allreduce
int pack_gram_panel(cudaStream_t st, const double* Pl, long long ldp, long long ps, int c0, int c1, cplx* buf, int w,
                    std::string* err);

}  // namespace traj
