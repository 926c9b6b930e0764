// Internal interface of the monitoring kernels and helpers (monitor.cu).
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

// mode 0: n_out[t][i] = sum_k |U_ik|^2; mode 1: also U_i. *= exp(a_i) (homodyne, Eq. A3).
int row_monitor(cudaStream_t st, cplx* U, long long ld, long long sU, int L, int N, int T, int mode, long long step,
                long long traj_base, uint64_t seed, const double* gamma_dev, double dt, double* n_out,
                std::string* err, int site0 = 0);
// flags[t][i] = (u0 of site site0+i < gamma_t dt)
int click_draw(cudaStream_t st, int L, int T, long long step, long long traj_base, uint64_t seed,
               const double* gamma_dev, double dt, int32_t* flags, std::string* err, int site0 = 0);
// The same click decisions on the host (counter-based Philox: the click set is a pure function of
// (seed, step, trajectory, site)): counts[t] = #{i < L : u0(site0 + i) < gamma_t dt}.  Sizes the
// projective launches without reading the device's count back (traj_step stays asynchronous).
void host_click_counts(int L, int T, long long step, long long traj_base, uint64_t seed, const double* gamma,
                       double dt, int32_t* counts, int site0 = 0);
// list[t] = site0 + (ascending flagged indices), count[t]
int compact(cudaStream_t st, const int32_t* flags, int L, int T, int32_t* list, int cap, int32_t* count,
            std::string* err, int site0 = 0);
// dst[t][r] = src[t][idx[t][r] - row_offset] for r < count[t] (or rows if count_dev is null)
int gather_rows(cudaStream_t st, const cplx* src, long long lds, long long sS, const int32_t* idx, long long sIdx,
                const int32_t* count_dev, int rows, int T, cplx* dst, long long ldd, long long sD, int ncols,
                std::string* err, int row_offset = 0, int zero_fill = 0);
// batched helpers of the projective rank-k update (k_dev: per-trajectory counts, padded to kmax)
int gather_sub_batched(cudaStream_t st, const cplx* D0, long long ld0, long long s0, const int32_t* pos, int cap,
                       const int32_t* k_dev, int kmax, int T, cplx* D11, long long ld1, long long s1,
                       std::string* err);
int sub_identity_batched(cudaStream_t st, cplx* T, long long ld, long long sT, const int32_t* S1, int cap,
                         const int32_t* k_dev, int kmax, int nT, std::string* err);
int zero_rows_batched(cudaStream_t st, cplx* U, long long ld, long long sU, const int32_t* rows, int cap,
                      const int32_t* k_dev, int kmax, int T, int ncols, std::string* err);
// Blocked conditional Born sampling of every trajectory's click list on C_SS (D0, kept);
// pos0 (optional): positions within S of the empty outcomes;
// Dw: work copy; Linv/DLinv: [T][64][64]; Ybuf/Zbuf: [T][64][ldy] with ldy >= maxc.
int sample_outcomes(cudaStream_t st, const cplx* D0, cplx* Dw, long long ldd, long long sD, const int32_t* S, int cap,
                    const int32_t* count, int maxc, int T, long long step, long long traj_base, uint64_t seed,
                    int32_t* occ, cplx* Linv, cplx* DLinv, cplx* Ybuf, cplx* Zbuf, long long ldy, int32_t* pos1,
                    int32_t* S1, int32_t* S0, int32_t* k1, int32_t* k0, std::string* err, int32_t* pos0 = nullptr);
int gather_sub(cudaStream_t st, const cplx* D0, long long ld0, const int32_t* pos, int k, cplx* D11, long long ld1,
               std::string* err);
// T[S1[c] - row0][c] -= 1 for the S1 entries c < k (and c < *k_dev when given) inside [row0, row0 + nrows)
int sub_identity(cudaStream_t st, cplx* T, long long ld, const int32_t* S1, int k, std::string* err, int row0 = 0,
                 int nrows = 1 << 30, const int32_t* k_dev = nullptr);
// zero the rows (global ids; the first nrows, and < *k_dev when given) inside [row0, row0 + nlocal) of U
int zero_rows(cudaStream_t st, cplx* U, long long ld, const int32_t* rows, int nrows, int ncols, std::string* err,
              int row0 = 0, int nlocal = 1 << 30, const int32_t* k_dev = nullptr);
// out[0] = in[0] + ... + in[n-1] (device)
int sum_i32(cudaStream_t st, const int32_t* in, int n, int32_t* out, std::string* err);
int entropy_reduce(cudaStream_t st, const double* lam, int n, double* S_out, int32_t* bad, std::string* err);
// rows [row0, row0+nrows) of K (nrows < 0: all L rows)
int build_k(cudaStream_t st, cplx* K, long long ld, int Lx, int Ly, const cplx* kx, const cplx* ky, std::string* err,
            long long row0 = 0, long long nrows = -1);
// bins[r] += sum_i |C[i][row0+i+r]|^2 over the R rows of the block C (rows row0.. of U U^dag)
int bin_abs2(cudaStream_t st, const cplx* C, long long ld, int R, int row0, int L, double* bins, std::string* err);
// out[0] += sum_{i<R, mask[j]} |C[i][j]|^2 (part: >= 1024 doubles of scratch)
int masked_abs2(cudaStream_t st, const cplx* C, long long ld, int R, int ncols, const int32_t* mask, double* part,
                double* out, std::string* err);
// X = a X + b I (full n x n batch entries)
int axpby_identity(cudaStream_t st, cplx* X, long long ld, long long sX, int n, int T, double a, double b,
                   std::string* err);
// upper triangle of every n x n batch entry := identity
int set_identity(cudaStream_t st, cplx* G, long long ld, long long sG, int n, int T, std::string* err);
// out[i] += in[i]
int add_inplace(cudaStream_t st, double* out, const double* in, long long n, std::string* err);
// out[t] = max_{i<=j} |G_ij - delta_ij| (as the bit pattern of a non-negative double)
int gram_deviation(cudaStream_t st, const cplx* G, long long ld, long long sG, int n, int T, unsigned long long* out,
                   std::string* err);
// CholeskyQR2's second-pass decision on the device: gate[0] = 1 if some trajectory's dev (bit pattern of
// max|G2 - I| from gram_deviation) exceeds thr (then the full factorisation runs), and fallbacks[0]++
int cqr2_decide(cudaStream_t st, const unsigned long long* dev, int T, double thr, int32_t* gate,
                unsigned long long* fallbacks, std::string* err);
// X = I - triu(E,1) - diag(E)/2 with E = G - I: R^-1 of G = R^dag R to O(|E|^2)
int first_order_inverse(cudaStream_t st, const cplx* G, long long ldg, long long sG, cplx* X, long long ldx,
                        long long sX, int n, int T, std::string* err);
int init_state(cudaStream_t st, cplx* U, long long ld, long long sU, const int32_t* sites, int N, int T,
               std::string* err, int row0 = 0, int nrows = 1 << 30);

}  // namespace traj
