/*
 * traj.h -- C-ABI of libtraj.so: the quantum-trajectory time step of a monitored
 * U(1) Gaussian (Slater-determinant) state on B200 (sm_100a).
 *
 * Paper: B. Fan, C. Yin, A. M. Garcia-Garcia, "Entanglement dynamics of monitored
 * non-interacting fermions on GPUs", arXiv 2508.18468.  "P:NNN" cites a line of
 * that paper's LaTeX source together with the section / equation.
 * Q-numbers are the readings of ambiguous passages listed in DESIGN.md.
 *
 * State of one trajectory (App. A): |psi> = prod_k [sum_j U_jk c_j^dag] |vac>,
 * U an L x N complex matrix with U^dag U = 1, N = L/2 (half filling).
 * One step (north star; P:203-209 QSD, P:171-196 PM):
 *   (a) U <- K U with K = exp(-i H~ dt), H~_ij = J delta_{i+-1,j}, dense;
 *   (b) n_i = sum_k |U_ik|^2, then the monitor: homodyne Eq. (A3) in split form, or
 *       projective clicks with Born outcomes, Eq. (A1)/(A2) (sign-corrected A2, Q15);
 *   (c) CholeskyQR2: G = U^dag U, R^dag R = G, U <- U R^-1, twice ("QR ... after each step").
 * At sampled times: C_A = U_A U_A^dag, S_A = -sum[l ln l + (1-l) ln(1-l)],
 * I_2 = S_A + S_B - S_{AuB}.
 *
 * Conventions (all calls):
 *   - Every call returns a traj_status; nothing aborts.  After TRAJ_EINVAL,
 *     TRAJ_ECONFIG or TRAJ_EDOMAIN the handle stays usable.
 *   - Calls are ordered on cfg.stream and asynchronous, except those returning host
 *     values (traj_entropy, traj_mutual_info, traj_failed, traj_get_step), which
 *     synchronise the stream.
 *   - Complex numbers are complex128 stored as interleaved (re, im) doubles; matrices
 *     are row-major.  The library copies traj_config; the caller owns every pointer it
 *     passes and the workspace, which must outlive the handle.
 *   - The library owns its cuSOLVER handle and events and frees them in traj_destroy.
 *   - There is no CPU fallback: without a CUDA device, traj_init returns TRAJ_ECUDA.
 *   - One handle per host thread.
 */
#ifndef TRAJ_H
#define TRAJ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct traj_ctx* traj_handle;      /* opaque; owned by the library */

typedef enum {
  TRAJ_OK = 0,
  TRAJ_EINVAL = 1,    /* bad argument to a call (null pointer, out-of-range index)        */
  TRAJ_ECONFIG = 2,   /* invalid traj_config (mirrors SPEC's "config error = 2")           */
  TRAJ_ENUMERIC = 3,  /* Cholesky breakdown / spectrum outside [-1e-8, 1+1e-8]; the
                         trajectory is marked failed and excluded (never reseeded)        */
  TRAJ_ECUDA = 4,     /* CUDA / cuSOLVER error, or no device                              */
  TRAJ_ENCCL = 5,     /* NCCL error (row-sharded mode)                                     */
  TRAJ_EDOMAIN = 6    /* overlapping regions, site index outside the lattice              */
} traj_status;

/* Protocols.  TRAJ_HOMODYNE: Eq. (A3) in exact split form (K, then the diagonal factor).
 * TRAJ_HOMODYNE_RK4: the paper-literal integrator of P:209 -- classical RK4 on
 * dU/dt = M U, M = -i H~ + diag(dW/dt) + gamma diag(2 <n>_t - 1) held fixed over the step
 * (dW and <n>_t at time t), H~ applied as a nearest-neighbour stencil, then CholeskyQR2. */
/* TRAJ_PROJECTIVE_EVENTS: the paper-literal event-driven PM of P:173-195 --
 * Poisson waiting times -ln(eta)/(gamma N), one uniformly chosen site per event, Born outcome
 * against p_c, the exact rank-1 update of Eq. (A1)/(A2) in orbital form; traj_step advances the
 * time by dt per step, processing every event inside the window, then CholeskyQR2.  Event e of
 * trajectory tau draws Philox counters (e_lo, e_hi, tau, 1) and (e_lo, e_hi, tau, 2).
 * traj_last_clicks reports the events of the last window and how many were "occupied". */
enum { TRAJ_PROJECTIVE = 0, TRAJ_HOMODYNE = 1, TRAJ_HOMODYNE_RK4 = 2, TRAJ_PROJECTIVE_EVENTS = 3 };
/* Initial state (Q1, Q2): sites with (x + y) even occupied.  TRAJ_INIT_NEEL: the Neel state
 * |1010...> of P:173/P:198 (0-based even sites) in 1d -- and, for compatibility, the same (x + y)
 * even rule in 2d; TRAJ_INIT_CHECKERBOARD: the 2d checkerboard (dim = 2 only, TRAJ_ECONFIG in 1d). */
enum { TRAJ_INIT_NEEL = 0, TRAJ_INIT_CHECKERBOARD = 1 };

typedef struct {
  int32_t dim;              /* 1 or 2 (P:42 ring; P:123 square torus)                         */
  int64_t Lx, Ly;           /* extents; Ly = 1 in 1d; L = Lx*Ly even (then exactly L/2 sites
                               have x+y even); 2d needs Lx, Ly >= 3; site = y*Lx + x (Q2)     */
  int64_t N;                /* particle number, must equal L/2                         */
  double J, dt;             /* hopping J (J = 1) and time step dt > 0 (0.05)     */
  int32_t protocol;         /* TRAJ_PROJECTIVE, TRAJ_HOMODYNE or TRAJ_HOMODYNE_RK4
                                                                                  */
  int32_t init;             /* TRAJ_INIT_NEEL (1d or 2d) or TRAJ_INIT_CHECKERBOARD (2d)          */
  uint64_t seed;            /* Philox4x32-10 key (lo, hi words), Q9                            */
  int64_t n_traj;           /* trajectories held by this handle, >= 1                          */
  int64_t traj_base;        /* global id of the first one (Philox counter word 2)              */
  const double* gamma;      /* host[n_traj]: per-site monitoring rate, gamma >= 0 (Q11);
                               projective needs gamma*dt <= 1 (Q10)                            */
  /* Row sharding of K and U, n_traj must be 1 and L % shard_size == 0.
   * shard_size = 1, nccl_id = NULL: no sharding.
   * nccl_id != NULL: this handle is rank shard_rank of shard_size processes (one per GPU);
   *   nccl_id is a 128-byte ncclUniqueId (traj_nccl_unique_id on rank 0, broadcast by the
   *   caller, e.g. over torch.distributed).  Rank r owns rows [r L/P, (r+1) L/P).
   * nccl_id = NULL, shard_size = P > 1, shard_rank = 0: single-GPU emulation -- the handle
   *   holds all P shards and performs the collectives as device copies / sums.          */
  int32_t shard_rank;
  int32_t shard_size;
  const void* nccl_id;
  void* stream;             /* cudaStream_t the handle runs on (e.g. torch's current stream)   */
  void* workspace;          /* device memory, >= traj_workspace_bytes, 256-byte aligned        */
  size_t workspace_bytes;
  int32_t propagator;       /* TRAJ_PROP_DENSE (the north star's dense K U) or TRAJ_PROP_BANDED */
  int32_t orthonormalizer;  /* TRAJ_ORTH_CQR2 (default) or TRAJ_ORTH_LOWRANK (projective only)   */
} traj_config;

/* Orthonormalisation of the projective step.  CQR2: CholeskyQR2 (its first Gram formed from the
 * rows zeroed by the empty outcomes).  LOWRANK ("orthonormalise the projective
 * step at low rank"): U is orthonormal before k0 rows V are zeroed, so U' (I + V^dag F V) with
 * F = Z^2 (Z + I)^-1, Z = (I - V V^dag)^(-1/2) (coupled Newton-Schulz on the k0 x k0 block) is
 * orthonormal -- two O(L N k0) GEMMs instead of pass 1's Cholesky and triangular multiply; the
 * second CholeskyQR pass (measured Gram) follows.  Falls back to CQR2 if the iteration does not
 * converge in 100 steps. */
enum { TRAJ_ORTH_CQR2 = 0, TRAJ_ORTH_LOWRANK = 1 };

/* Propagator of step (a).  DENSE: U <- K U with the dense L x L K on the FP64 tensor pipe
 * (8 L^2 N flops).  BANDED: K is a circulant per lattice axis whose
 * coefficients fall below 1e-18 after a few neighbours (Bessel tail); U <- K U becomes one
 * (1d) or two (2d, K = K_y (x) K_x) banded stencil passes of half-width W (W chosen so the
 * dropped tail is < 1e-18; the dense path is used if 2W+1 exceeds an extent).  No L x L
 * matrix is stored.  With row sharding the U allgather is replaced by a halo exchange of W rows
 * (1d) or W*Lx rows (2d, whole lattice rows per shard required) with the neighbouring shards. */
enum { TRAJ_PROP_DENSE = 0, TRAJ_PROP_BANDED = 1 };

/* Device bytes the handle needs for cfg (the caller allocates them, e.g. with torch).
 * Validates cfg; TRAJ_ECONFIG if invalid.  Needs a CUDA device (cuSOLVER query). */
int traj_workspace_bytes(const traj_config* cfg, size_t* out);

/* Validate cfg, build K = exp(-i H~ dt) on the device (1d: Bessel series of the
 * circulant; 2d: K_y (x) K_x), set U0 = Neel / checkerboard for every trajectory,
 * step counter = 0.  *out receives the handle. */
int traj_init(const traj_config* cfg, traj_handle* out);

/* Advance every trajectory by n_steps >= 0 steps (P:203-209 / P:171-196).  Step s
 * draws Philox counters (site, s, traj_base + t, 0).  Asynchronous (stream-ordered, no host
 * round trip) for TRAJ_HOMODYNE, TRAJ_HOMODYNE_RK4 and TRAJ_PROJECTIVE with CholeskyQR2, sharded or
 * not: the projective launches are sized by click counts the host computes from the same
 * counter-based draws (the device's own draws decide the clicks), the occupied / empty counts of
 * the Born sampling stay on the device (launches bounded there), and CholeskyQR2's second-pass
 * fallback is decided on the device.  TRAJ_PROJECTIVE_EVENTS (host-drawn event times and staged
 * stencil taps) and TRAJ_ORTH_LOWRANK (its k0 x k0 iteration checks convergence on the host)
 * synchronise within the step.  A trajectory whose Cholesky breaks down is marked failed
 * (traj_failed).
 * Small lattices (dense K, projective or homodyne, unsharded, U and the step's scratch
 * within one CTA's shared memory: L up to ~110) run all n_steps in one asynchronous launch
 * of the fused step (one CTA per trajectory); there a failed trajectory stops evolving.
 * TRAJ_SMALL_STEP=0 in the environment at traj_init selects the general path. */
int traj_step(traj_handle h, int64_t n_steps);

/* Re-orthonormalise every trajectory with CholeskyQR2 (step (c) alone). */
int traj_orthonormalize(traj_handle h);

/* Entanglement entropy of region A (host array of nA distinct site indices in
 * [0, L)) for every trajectory: S_out = host[n_traj].  eigvalsh of
 * C_A = U_A U_A^dag (or U_A^dag U_A when nA > N) by cuSOLVER.  Returns TRAJ_ENUMERIC
 * if some eigenvalue is outside [-1e-8, 1+1e-8] (that trajectory's S_out is NaN and
 * it is marked failed); failed trajectories give NaN. */
int traj_entropy(traj_handle h, const int64_t* A, int64_t nA, double* S_out);

/* I_2 = S_A + S_B - S_{AuB} for every trajectory; A and B must be disjoint
 * (TRAJ_EDOMAIN otherwise). */
int traj_mutual_info(traj_handle h, const int64_t* A, int64_t nA,
                     const int64_t* B, int64_t nB, double* I_out);

/* Density correlator of Eq. (2) for the 1d chain: C_out = host[L],
 * C_out[r] = mean over the L - r pairs i < j = i + r of C_ij = -D_ij D_ji = -|(U U^dag)_ij|^2,
 * r = 1..L-1 (C_out[0] = NaN).  Rows of U U^dag are formed in blocks on the DMMA GEMM and
 * binned by a deterministic kernel (8 L^2 N flops).  TRAJ_EDOMAIN in 2d. */
int traj_density_correlation(traj_handle h, int64_t traj, double* C_out);

/* Particle-number covariance of Eq. (5) between disjoint regions A and B:
 * G_out = host[n_traj], G_AB = -sum_{i in A, j in B} C_ij = sum |(U U^dag)_ij|^2 >= 0.
 * The paper compares I_2 with (2 pi^2 / 3) G_AB. */
int traj_particle_covariance(traj_handle h, const int64_t* A, int64_t nA, const int64_t* B, int64_t nB,
                             double* G_out);

/* n_out = device[n_traj][L] doubles: n_i = sum_k |U_ik|^2 of the current state
 * (row-sharded: the rows this handle holds, see traj_shard_info). */
int traj_occupations(traj_handle h, double* n_out);

/* Rows [row0, row0+nrows) of C = U U^dag for trajectory traj into C_out =
 * device complex128 [nrows][L]. */
int traj_correlation_rows(traj_handle h, int64_t traj, int64_t row0, int64_t nrows, void* C_out);

/* Copy U (L x N, complex128 row-major, ld = N) of trajectory traj out of / into the
 * handle (row-sharded: the rows this handle holds).  The pointer may be host or device
 * (UVA copy).  traj_set_state does not orthonormalise: call traj_orthonormalize (or
 * traj_step) afterwards. */
int traj_get_state(traj_handle h, int64_t traj, void* U_out);
int traj_set_state(traj_handle h, int64_t traj, const void* U_in);

/* Step counter (the Philox step word of the next step); set for checkpoint/resume.  For
 * TRAJ_PROJECTIVE_EVENTS traj_set_step also rebuilds the event clock at time step * dt (events
 * before it counted, the next event's time) from the Philox waiting times, so (state, step) is a
 * complete checkpoint for every protocol. */
int traj_get_step(traj_handle h, int64_t* step);
int traj_set_step(traj_handle h, int64_t step);

/* *flag = 1 if trajectory traj failed (Cholesky breakdown or bad spectrum). */
int traj_failed(traj_handle h, int64_t traj, int32_t* flag);

/* Clicks of the last projective step of trajectory traj: |S| and the number of
 * "occupied" outcomes. */
int traj_last_clicks(traj_handle h, int64_t traj, int64_t* n_clicks, int64_t* n_occupied);

/* Number of CholeskyQR2 second passes that needed the full Cholesky because
 * N max|G2 - I|^2 >= 1e-18 (otherwise the first-order factor, exact to rounding, is used;
 * environment TRAJ_CQR2_FULL=1 forces the full factorisation every time). */
int traj_cqr2_fallbacks(traj_handle h, int64_t* n);

/* max|G2 - I| over the upper triangle of the Gram matrix G2 = U'^dag U' that the most recent
 * CholeskyQR2 second pass measured (App. A: the QR step that keeps U orthonormal; SURVEY §8(a)
 * a3), one double per trajectory of the handle (host array, n_traj entries; 1 for a row-sharded
 * handle): the orthonormality left by the first pass, the quantity the first-order / full
 * factorisation decision and the modulus count of the modular correction are keyed on.  0 before the
 * first second pass.  Synchronises the handle's stream.  TRAJ_EINVAL for the fused small-lattice step. */
int traj_gram_deviation(traj_handle h, double* out);

/* Counters of the low-rank projective orthonormaliser (TRAJ_ORTH_LOWRANK, NEXT-1 option; SURVEY
 * §8(f) 1 "orthonormalise the projective step at low rank"), cumulative since traj_init:
 *   newton_iters  coupled Newton-Schulz iterations for (I - V V^dag)^(-1/2);
 *   fallbacks     steps where the iteration did not converge and CholeskyQR2 ran instead;
 *   probes        orthonormality certificates: ||U^dag U - I||_F estimated with 4 unit-modulus
 *                 random probes (Hutchinson) after a low-rank step, two HBM passes over U;
 *   refinements   probes above the tolerance (environment TRAJ_LOWRANK_TOL, default 5e-13;
 *                 0 = refine every step), each followed by one measured CholeskyQR pass.
 * Any pointer may be NULL.  TRAJ_EINVAL on a NULL handle.  Zeros for other orthonormalisers. */
int traj_lowrank_stats(traj_handle h, int64_t* newton_iters, int64_t* fallbacks, int64_t* probes,
                       int64_t* refinements);

/* The orthonormality certificate used by the low-rank orthonormaliser, on the current state:
 * est_out[t] (host, n_traj doubles) = sqrt((1/4) sum_j ||U_t^dag (U_t x_j) - x_j||^2), an unbiased
 * (in the square) estimate of ||U_t^dag U_t - I||_F from 4 probes x_j with entries (+-1 +- i)/sqrt 2
 * drawn by Philox (k, step, traj, 3).  Synchronises the stream.  TRAJ_EINVAL with row sharding. */
int traj_probe_orthonormality(traj_handle h, double* est_out);

/* Per-phase device timing with CUDA events on the handle's stream.  enable != 0
 * starts recording (and zeroes the totals).  traj_phase_times fills ms[TRAJ_NPHASES]
 * with accumulated milliseconds and launches[TRAJ_NPHASES] with kernel-launch counts
 * (synchronises).  Phases: */
enum { TRAJ_PH_PROPAGATE = 0,  /* U <- K U                                   */
       TRAJ_PH_MONITOR = 1,    /* occupations + homodyne factor / click draw */
       TRAJ_PH_PROJECT = 2,    /* click list, D_SS, sampling, rank-k update  */
       TRAJ_PH_GRAM = 3,       /* G = U^dag U (both CQR passes)              */
       TRAJ_PH_CHOL = 4,       /* Cholesky + triangular inverse of G         */
       TRAJ_PH_TRMM = 5,       /* U <- U R^-1                                */
       TRAJ_PH_FUSED = 6,      /* the fused small-lattice step (all rows)    */
       /* nested (not additive): the INT8 tensor-core launch of the modular products inside the
        * propagate, Gram and TRMM phases (traj_ozaki_info) */
       TRAJ_PH_KU_MMA = 7, TRAJ_PH_GRAM_MMA = 8, TRAJ_PH_TRMM_MMA = 9,
       /* nested in chol: the structured pass 1's factor chain (on the stream it runs on; not recorded
        * when factor and solve are interleaved on the DMMA path) */
       TRAJ_PH_STRUCT_FACTOR = 10,
       TRAJ_NPHASES = 11 };
int traj_profile(traj_handle h, int enable);
/* Which contractions of this handle run as exact modular products on the INT8 tensor cores
 * (csrc/ozaki.h; environment TRAJ_OZAKI=0 selects the FP64 DMMA kernels instead):
 * out[0] = the dense K U, out[1] = the CholeskyQR Grams and TRMMs, out[2] = the modulus count
 * (16: every operand row / column to 2^-58 of its 2-norm).  Row-sharded handles: out[0] = out[1] =
 * the chunked K_g U (its residues accumulated over the P chunks at U's global column exponents) and
 * the local Grams / TRMMs; the projective rank-k products and the structured pass stay on DMMA. */
int traj_ozaki_info(traj_handle h, int32_t* out3);
int traj_phase_times(traj_handle h, double* ms, int64_t* launches);

/* Row sharding: *shard_size = P, *local_shards = shards held by this handle (1, or P in
 * the single-GPU emulation), rows [*row0, *row0 + *rows) of U / n are held here. */
int traj_shard_info(traj_handle h, int32_t* shard_size, int32_t* local_shards, int64_t* row0, int64_t* rows);

/* The communication schedule of the row-sharded step for rank `rank` of P, as plain
 * host data (no GPU, no NCCL): the NCCL executor issues exactly these operations, in this order.
 *   kind 0: the U exchange fused into the chunked K_g U (dense propagator): for ring distance
 *           d = 1..P-1 one group {send own block to rank+d, receive block rank-d};
 *   kind 1: the halo exchange of the banded propagator: one group of two sends and two receives;
 *           entries are 5 int64: (group, op 0 = send / 1 = recv, peer, slot, block) -- slot is the local
 *           buffer (kind 0: 0 = own block / the received block's row range of U_full; kind 1: 0 = low
 *           edge / low halo, 1 = high edge / high halo), block the global identity of the data (kind 0:
 *           the row block's owner; kind 1: 2r = low edge of rank r, 2r + 1 = its high edge);
 *   kind 2: the broadcasts of the distributed Cholesky of an n x n Gram (levels >= TRAJ_DIST_CHOL_MIN,
 *           default 2048), in issue order: 3 int64 (root, rows, cols) per broadcast.
 * NCCL pairs the operations between two ranks in issue order; tests/test_comm_plan.py checks that every
 * receive meets the send of the block it names, for P = 2..8, and runs the schedules over gloo.
 * Writes min(count, max_entries) entries to out (host) and returns the entry count, or -TRAJ_EINVAL. */
int64_t traj_comm_plan(int kind, int P, int rank, int64_t n, int64_t* out, int64_t max_entries);

/* out128 <- a fresh ncclUniqueId (128 bytes) for traj_config.nccl_id. */
int traj_nccl_unique_id(void* out128);

/* Kernels launched by the library in this process so far (every launch site counts). */
long long traj_kernel_launches(void);

int traj_destroy(traj_handle h);
/* Message of the last failure on h (h = NULL: the last failure of a handle-less call
 * on this thread, e.g. traj_init). */
const char* traj_last_error(traj_handle h);
const char* traj_strerror(int status);

/* ---------------------------------------------------------------------------
 * Building blocks, exported for kernel-level tests.  Device pointers; all
 * matrices complex128 row-major with leading dimension ld (in complex elements,
 * ld >= columns, ld*16 a multiple of 16 bytes).
 *
 * traj_zgemm: C_b = alpha * op(A_b) op(B_b) + beta * C_b for b in [0, batch),
 *   op(X) = X (op = 0) or X^dag (op = 1); op(A) is M x K, op(B) is K x N.
 *   X_b = X + b*strideX (strideX in complex elements; 0 shares X across the batch).
 *   flags: TRAJ_TRI_* declare a triangular operand whose other triangle is
 *   stored as zeros (k-blocks that are all zero are skipped); TRAJ_C_UPPER writes
 *   only entries with row <= col (and skips tiles below the diagonal).
 *   The FP64 tensor pipe (DMMA) does the arithmetic; 8mnk flops. */
enum { TRAJ_TRI_A_UPPER = 1, TRAJ_TRI_A_LOWER = 2, TRAJ_TRI_B_UPPER = 4,
       TRAJ_TRI_B_LOWER = 8, TRAJ_C_UPPER = 16 };
int traj_zgemm(void* stream, int opA, int opB, int64_t M, int64_t N, int64_t K,
               double alpha_re, double alpha_im,
               const void* A, int64_t lda, int64_t strideA,
               const void* B, int64_t ldb, int64_t strideB,
               double beta, void* C, int64_t ldc, int64_t strideC,
               int64_t batch, int flags);

/* Complex multiplication scheme of every contraction (process-wide): 1 = 3M (Gauss, the
 * default): A_r B_r, A_i B_i and (A_r + A_i)(B_r + B_i) as three real DMMA products, 6mnk
 * tensor-pipe flops per 8mnk algorithmic, FP64 throughout, the usual ZGEMM3M error bound for
 * the imaginary part; 0 = 4M: two real DMMA products over an interleaved (re, im) k axis,
 * 8mnk tensor flops.  Initial value from the environment: TRAJ_ZGEMM_3M=0 selects 4M. */
/* Real FP64 GEMM on the DMMA pipe, C_z = alpha A_z B_z + beta C_z (row-major, no transposes), the
 * building block of the planar 3M complex product (three real products, one accumulator set per
 * warp).  Device pointers; stream = cudaStream_t.  Needs K > 0, even lda and ldc, ldb a multiple of
 * 16 with ldb >= N rounded up to 16, 16-byte alignment; TRAJ_EINVAL otherwise. */
int traj_dgemm(void* stream, int64_t M, int64_t N, int64_t K, double alpha, const void* A, int64_t lda,
               int64_t strideA, const void* B, int64_t ldb, int64_t strideB, double beta, void* C, int64_t ldc,
               int64_t strideC, int64_t batch);

int traj_set_zgemm_algorithm(int algo);
int traj_get_zgemm_algorithm(void);

/* traj_igemm: C_z = A_z B_z^T for z < batch on the INT8 tensor cores (tcgen05.mma kind::i8 with TMEM
 * accumulators, operands staged by TMA; csrc/igemm.cu).  A_z: int8 M x K (row-major, lda bytes,
 * A_z = A + z*strideA), B_z: int8 N x K (ldb, strideB), C_z: the exact int32 sums (ldc elements,
 * strideC) -- or, with moduli != NULL (device int32[nmod], each in [2, 256]), those sums mod
 * moduli[z % nmod] in [0, m) as uint8.  flags: 1 = only the 128 x 256 tiles that meet the upper
 * triangle are computed, 2 = B_z[n][k] = 0 for k > n is assumed (those k-blocks are skipped).
 * Needs 0 < K < 2^17 (so |sum| <= K 128^2 < 2^31), lda and ldb multiples of 16 >= K, ldc a multiple
 * of 16 >= N, 16-byte aligned pointers; TRAJ_EINVAL otherwise.  Stream-ordered, asynchronous. */
int traj_igemm(void* stream, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int64_t strideA,
               const void* B, int64_t ldb, int64_t strideB, void* C, int64_t ldc, int64_t strideC, int64_t batch,
               const int32_t* moduli, int nmod, int flags);

/* traj_zgemm_ozaki: C = op(A) B in complex128 (row-major, ld in complex elements), computed by the
 * exact modular scheme on the INT8 tensor cores (csrc/ozaki.h: Ozaki-II; the contraction the paper
 * states as a complex-FP64 matrix product).  opA = 0: A is M x K; opA = 1: A is stored
 * K x M and op(A) = A^dag (the Gram form U^dag U).  B is K x N.  nmod in {4, 6, ..., 18} pairwise
 * coprime moduli, each with a square root of -1 (so a complex product mod m is two real ones): every
 * row of op(A) and column of B is represented to 2^-(beta+1) of its 2-norm, beta = 57 for 16 and 61
 * for 18, and the products are exact (an FP64 GEMM's rounding errors are 2^-53 of the same norms).  flags: TRAJ_C_UPPER (only j >= i written), TRAJ_TRI_B_UPPER (B upper triangular).  The
 * residue scratch is allocated and freed on the stream (cudaMallocAsync); TRAJ_EINVAL on a bad
 * shape. */
int traj_zgemm_ozaki(void* stream, int opA, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                     const void* B, int64_t ldb, void* C, int64_t ldc, int nmod, int flags);

/* The host-side constants of the modular scheme for nmod moduli (no device needed; for tests):
 * moduli[nmod] (odd, pairwise coprime, <= 256, prime factors = 1 mod 4), *beta (operand bits: every
 * row / column is scaled below 2^beta), ch[nmod/2], cl[nmod/2] (the CRT weights of the moduli pairs:
 * X / M = frac(sum_p r_p (ch_p + cl_p)), ch_p a multiple of 2^-36), *M (prod m as a double).
 * TRAJ_EINVAL for an unsupported nmod. */
int traj_ozaki_constants(int nmod, int32_t* moduli, int32_t* beta, double* ch, double* cl, double* M);
/* roots[q]^2 = -1 (mod moduli[q]): the image j_q of the imaginary unit in Z_m, which splits a complex
 * residue into the two real planes re +- j_q im (csrc/ozaki.h). */
int traj_ozaki_roots(int nmod, int32_t* roots);

/* traj_chol_inverse: for each b, G_b (n x n Hermitian positive definite; only the
 * upper triangle is read) = R^dag R with R upper triangular; writes X_b = R^-1
 * (upper triangle; the strict lower triangle is set to zero).  G_b's strict lower
 * triangle is used as scratch.  scratch: device, >= traj_chol_scratch_bytes(n, batch).
 * failed: device int32[batch]; set to 1 where a pivot is not positive/finite. */
size_t traj_chol_scratch_bytes(int64_t n, int64_t batch);
int traj_chol_inverse(void* stream, int64_t n, void* G, int64_t ldg, int64_t strideG,
                      void* X, int64_t ldx, int64_t strideX, int64_t batch,
                      void* scratch, int32_t* failed);

#ifdef __cplusplus
}
#endif
#endif /* TRAJ_H */
