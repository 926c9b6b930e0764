// Internal interface of the exact modular complex-FP64 products (ozaki.cu): the Ozaki-II scheme
// (Ozaki, Uchino, Imamura 2024) on the INT8 tensor cores of sm_100a.
//
// A complex product C = A B (A: M x K, B: K x N, complex128) is computed as follows.
//  1. Each row of A (column of B) is scaled by a power of two 2^e so that the 2-norm of
//     (|re| + |im|) over that row is < 2^beta, and rounded to Gaussian integers (exact for every entry
//     >= 2^(beta - 53) times that norm; the others lose bits below 2^-beta of it).
//  2. The moduli m_q <= 256 are odd, pairwise coprime, and built from primes = 1 (mod 4) only, so each
//     has a j_q with j_q^2 = -1 (mod m_q) and Z[i] / (m_q) = Z_m x Z_m by z -> (z+, z-) = (re + j_q im,
//     re - j_q im): a complex product mod m_q is TWO independent real products (the 3M scheme over the
//     integers needs three, the plain one four).  The two planes z+-, mod each of the s moduli, are
//     stored as int8 residues in [-128, 127]; a conjugated operand just swaps its planes.
//  3. Two products per modulus, P+ = A+ B+ and P- = A- B-, run on the INT8 tensor cores (igemm.cu),
//     exact in int32, reduced mod m_q in the epilogue.
//  4. 2 Re = P+ + P- and 2 Im = -j_q (P+ - P-) mod m_q are exact; the Chinese remainder theorem gives
//     the integers 2X (|2X| < prod m_q / 2 by Cauchy-Schwarz on the scaled norms), and
//     C_ij = X_ij 2^-(eA_i + eB_j) rounded once to FP64.
// The only approximation is step 1's rounding: with s = 16 moduli beta = 57, i.e. every input is
// represented to 2^-58 of its row's (column's) norm (s = 18: beta = 61, the limit of the 62-bit integer
// split); the products themselves are exact (no FP64 rounding error accumulates over k), so the result
// is more accurate than an FP64 GEMM's, whose rounding errors are 2^-53 of the same norms.
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

constexpr int OZ_MAXS = 18;

// the bits per operand side for s moduli (floor(log2(prod m_q) / 2) - 1); 0 if s is not supported
int oz_beta(int s);
int oz_supported(int s);   // s in {4, 6, ..., 18}
// the host constants of s moduli (for tests): the moduli, beta, the pair CRT weights ch / cl (s / 2 each), M
int oz_constants(int s, int* moduli, int* beta, double* ch, double* cl, double* M);
// roots[q]^2 = -1 (mod moduli[q]): the j_q of the plane map
int oz_roots(int s, int* roots);

// Residue layout: R [plane][q][t][rows][ldr] int8 (ldr = round_up(K, 16)), two planes (z+, z-), plane
// stride s*T*rows*ldr.  The nplanes arguments and the OzProduct plane fields below date from the 3M
// scheme (planes re, im, re + im[, re - im]); they are kept so that call sites state which operand is
// conjugated (pa[2] == 3 / pb[2] == 3) and size their scratch generously -- every split writes two planes.
inline long long oz_ld(long long K) { return round_up(K, 16); }

// A operand from the rows of X (T matrices [rows][ldx], stride sX): residue row r = X row r over
// k = X's columns (conj: im -> -im, i.e. the planes swapped); e[t][r] (stride sE) the row exponents.
// cdev (device, per trajectory, optional): columns j >= cdev[t] of X are taken as zero
int oz_split_rows(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T, int conj,
                  int s, int8_t* R, int* e, long long sE, std::string* err, const int32_t* gate = nullptr,
                  const int32_t* cdev = nullptr, int nplanes = 3, const int32_t* rdev = nullptr);

// B operand from the columns of X: residue row j = X column j over k = X's rows;
// part: >= 8 * T * cols doubles of scratch.
// sub_identity: the operand is X - I (square X).  gate (device, optional): skip when *gate == 0.
int oz_split_cols(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T, int nplanes,
                  int s, int8_t* R, int* e, long long sE, double* part, std::string* err, int sub_identity = 0,
                  const int32_t* gate = nullptr, const int32_t* cdev = nullptr, const int32_t* rdev = nullptr);
// (rdev, both splits: rows r >= rdev[t] of X are taken as zero)
// e_in (optional): the columns' exponents given (e.g. global ones over all shards' rows) instead of
// computed from X's own column norms; e is then not written
int oz_split_cols_e(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T,
                    int nplanes, int s, int8_t* R, const int* e_in, long long sE, std::string* err);
// nu2[t][j] (+)= sum over X's rows of (|re| + |im|)^2 of column j (part: >= 8 T cols doubles of scratch);
// sub_identity: of X - I
int oz_colnorm_accumulate(cudaStream_t st, const cplx* X, long long ldx, long long sX, int rows, int cols, int T,
                          double* part, double* nu2, long long sN, int accumulate, std::string* err,
                          int sub_identity = 0);
// the modulus-count tier of a gated product from its operand's squared column norms nu2[0..n):
// gate[1] = !gate[0] && max nu2 <= thr2 (the low count suffices), gate[2] = !gate[0] && !gate[1]
int oz_tier_decide(cudaStream_t st, const double* nu2, long long n, double thr2, int32_t* gate, std::string* err);
// e[t][j] = the column exponents for s moduli from the squared norms nu2
int oz_exponents(cudaStream_t st, const double* nu2, long long sN, int cols, int T, int s, int* e, long long sE,
                 std::string* err);

enum OzFlags {
  OZ_UPPER = 1,       // C upper triangular (only j >= i computed and written)
  OZ_TRI_B = 2,       // B upper triangular (k > j skipped)
  OZ_NEG_P2 = 4,      // (3M scheme: one operand conjugated; ignored, the plane swap carries it)
  OZ_ACCUMULATE = 8,  // C += A B instead of C = A B
  OZ_NEGATE = 16,     // -A B (with base / OZ_ACCUMULATE: C = base - A B)
};

struct OzProduct {
  int M = 0, N = 0, K = 0, T = 1, s = 16;
  const int8_t* RA = nullptr;   // [planes][s][Ta][M][oz_ld(K)], Ta = T if a_traj else 1
  int a_traj = 1;
  long long a_planes = 3;       // (unused)
  int pa[3] = {0, 1, 2};        // pa[2] == 3: A is conjugated
  const int* eA = nullptr;      // [Ta][M] (stride sEA)
  long long sEA = 0;
  const int8_t* RB = nullptr;   // [planes][s][T][N][oz_ld(K)]
  long long b_planes = 3;
  int pb[3] = {0, 1, 2};        // pb[2] == 3: B is conjugated
  const int* eB = nullptr;      // [T][N]
  long long sEB = 0;
  uint8_t* RC = nullptr;        // scratch [2][s][T][ksplit][M][oz_ld(N)]
  cplx* C = nullptr;
  long long ldc = 0, sC = 0;
  int flags = 0;
  const cplx* base = nullptr;   // C = base + A B (same layout as C; may alias it)
  const int32_t* gate = nullptr;   // device flag: every launch does nothing when *gate == 0
  const int32_t* kdev = nullptr;   // per trajectory: the contraction runs over k < kdev[t] (operands zero past it)
  const int32_t* ndev = nullptr;   // per trajectory: only columns j < ndev[t] of C are computed and written
  int ksplit = 1;                  // split-K chunks of the INT8 launch (RC holds ksplit x the residue products)
  long long lda_override = 0;      // RA's row length in bytes when it is a k-range of wider residue rows
  int mma_accumulate = 0;          // oz_product_mma: add the residues to RC's (k-chunks summed) instead of writing
};

// The residue scratch of one handle's modular products (the caller sizes it for its shapes): operand
// residues RU / RX, products RC, exponents eU / eU2 (stride sEU per trajectory) and eX (stride sEX)
struct OzWork {
  int s = 16;
  int8_t* RU = nullptr;
  int8_t* RX = nullptr;
  uint8_t* RC = nullptr;
  size_t RC_bytes = 0;
  int* eU = nullptr;
  int* eU2 = nullptr;
  int* eX = nullptr;
  long long sEU = 0, sEX = 0;
  double* part = nullptr;
};

// the products (one batched INT8 launch) and the CRT combine into C
int oz_product(cudaStream_t st, const OzProduct& p, std::string* err);
// the same in two calls (the caller times the INT8 launch alone)
int oz_product_mma(cudaStream_t st, const OzProduct& p, std::string* err);
int oz_product_combine(cudaStream_t st, const OzProduct& p, std::string* err);

// bytes of the scratch buffers for a product of this shape
inline long long oz_residue_bytes(long long planes, int s, long long T, long long rows, long long K) {
  return planes * s * T * rows * oz_ld(K);
}

}  // namespace traj
