// Row-sharded trajectory step: K and U split by rows across P shards.
#pragma once
#include <complex>
#include <string>
#include <vector>

#include "../../include/traj.h"
#include "common.cuh"
#include "profiler.h"
#include "cholinv.h"
#include "watchdog.h"
#include "structchol.h"

typedef struct ncclComm* ncclComm_t;
typedef struct cusolverDnContext* cusolverDnHandle_t;

namespace traj {

// Collectives over the P shards.  NCCL mode: one shard per process (rank = shard_rank).
// Emulation mode (nccl_id == NULL): all P shards live in this handle on one GPU and the
// collectives are device copies / sums in rank order -- the same data movement, used to
// validate the sharded algorithm on a single GPU.
struct ShardComm {
  int P = 1, P_local = 1, rank0 = 0;
  ncclComm_t comm = nullptr;
  Watchdog wd;             // NCCL mode: async-error / deadline polling, abort (watchdog.h)
  // every NCCL call site: begin() returns TRAJ_ENCCL once the communicator was aborted, else
  // takes the watchdog's lock; end(st) releases it and hands the watchdog a completion mark on st
  int begin(std::string* err);
  void end(cudaStream_t st);
  int allgather(cudaStream_t st, void* const* send, void* recv, size_t bytes, std::string* err);
  int allreduce(cudaStream_t st, double* const* part, double* out, size_t n, std::string* err);
  // halo exchange on the ring of shards: recv_lo[s] <- send_hi of shard g-1, recv_hi[s] <- send_lo of g+1
  int halo(cudaStream_t st, void* const* send_lo, void* const* send_hi, void* const* recv_lo, void* const* recv_hi,
           size_t bytes, std::string* err);
};

struct ShardLocal {
  int g = 0, row0 = 0;
  cplx* K = nullptr;       // Lp x ldL: rows [row0, row0 + Lp) of K
  cplx* U[2] = {nullptr, nullptr};   // Lp x ldN
  cplx* Gpart = nullptr;   // N x ldN partial Gram (aliases G in NCCL mode)
  int32_t* flags = nullptr;
  int32_t* Sloc = nullptr;
  int32_t* cnt = nullptr;
  cplx* USloc = nullptr;   // capr x ldN
  cplx* Tm = nullptr;      // Lp x ldcap
  cplx* Uext = nullptr;    // banded: (H + Lp + H) x ldN, halo rows around the local block
  // planar 3M (dense K): K_g's planes [3][Lp][ldKs], product planes [3][Lp][ldPs], U's six planes
  double *Kp = nullptr, *Pp = nullptr, *Up6 = nullptr;
  double* Ks = nullptr;    // Strassen: the operands of every K chunk K_g[:, s], [P][3 7^lv][Lp/2^lv][ldS]
  // modular engine (ozaki.h): K_g's row residues [3][s][Lp][oz_ld(L)] over the full row, its row exponents
  int8_t* RK = nullptr;
  int* eK = nullptr;
};

struct ShardedCtx {
  ShardComm comm;
  int L = 0, N = 0, Lx = 0, Ly = 0, P = 1, Lp = 0, capr = 0, cap = 0, lwork = 0;
  long long ldN = 0, ldL = 0, ldcap = 0;
  int protocol = 0;
  bool banded = false;     // NEXT-1 with sharding: halo exchange instead of the allgather
  int Wx = 0, Wy = 0, H = 0;
  cplx* bcoef = nullptr;
  std::vector<cplx> band_host;   // host copy of the stencil taps (launch parameters)
  double dt = 0, J = 0, gamma = 0;
  uint64_t seed = 0;
  long long traj_base = 0;
  std::vector<ShardLocal> loc;
  int cur = 0;
  cplx *Ufull = nullptr, *G = nullptr, *X = nullptr;
  void* chol_scratch = nullptr;
  int32_t *Srecv = nullptr, *cntrecv = nullptr, *S = nullptr, *count = nullptr;
  cplx *USrecv = nullptr, *US = nullptr;
  cplx *D0 = nullptr, *Dw = nullptr, *Linv = nullptr, *DLinv = nullptr, *Ybuf = nullptr, *Zbuf = nullptr;
  int32_t *occ = nullptr, *pos1 = nullptr, *S1 = nullptr, *S0 = nullptr, *k1 = nullptr, *k0 = nullptr;
  cplx *D11 = nullptr, *X11 = nullptr, *W = nullptr;
  void* chol_scratch_small = nullptr;
  double* gamma_dev = nullptr;
  int32_t* failed_dev = nullptr;
  double* eig_w = nullptr;
  cplx* eig_work = nullptr;
  int* eig_info = nullptr;
  double* S_dev = nullptr;
  int32_t* bad_dev = nullptr;
  unsigned long long* gdev = nullptr;
  int32_t* region = nullptr;
  cplx* kcoef = nullptr;
  int32_t* sites = nullptr;
  int32_t* h_small = nullptr;
  double* h_dev = nullptr;
  long long last_nS = 0, last_n1 = 0, cqr2_fallbacks = 0;
  unsigned long long* fb_dev = nullptr;   // second passes that took the full factorisation (device count)
  int32_t* gate = nullptr;                // this step's second-pass decision (device)
  CholFallbackGraph fbg;                  // the decision + the conditional factorisation as one graph
  int fbg_state = 0;                      // 0: not built yet, 1: built, -1: gated launches
  bool k1_dev = false;                    // the last step's occupied count is in k1 (device)
  std::vector<int32_t> hcnt;              // per-shard click counts of the current step (host Philox)
  // CholeskyQR pass 1 on the structure G = I - V^dag V (structchol.h; TRAJ_STRUCT_CHOL=0: dense):
  // factored once from the gathered V (replicated, no collective), applied to each shard's rows
  bool struct_chol = true, struct_pending = false;
  // NCCL mode, planar Gram: column panels of width gram_pw, each packed (upper part, rows [0, c1))
  // and all-reduced on gst while the next panel's Gram runs (TRAJ_GRAM_PANEL=0: one full allreduce)
  int gram_pw = 0;
  cplx* gpack = nullptr;                  // [2][N][gram_pw]
  cudaStream_t gst = nullptr;
  cudaEvent_t ev_gpacked[2] = {nullptr, nullptr}, ev_gfree[2] = {nullptr, nullptr}, ev_gdone = nullptr;
  StructChol sc;
  bool full_cqr2 = false;
  // pass 1 of CholeskyQR after a projective step: G = I - V^dag V from the zeroed rows V, formed
  // from the gathered (replicated) U_S rows -- no Gram, no allreduce (TRAJ_LOWRANK_GRAM=0: measured)
  bool lowrank_gram = true;
  // CholeskyQR pass 1: factorisation on st_hi, TRMM of each newly final column block on st_lo
  // (TRAJ_CHOL_OVERLAP=0: serial)
  bool chol_overlap = false;
  cudaStream_t st_hi = nullptr, st_lo = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_left = nullptr, ev_lo_done = nullptr, ev_hi_done = nullptr;
  int lr_k0 = -1;          // >= 0: pass 1's G is set (0: no row zeroed, pass 1 has R = I)
  int32_t* pos0 = nullptr;
  cudaStream_t st = nullptr;
  // dense propagate with the allgather overlapped (NCCL mode): per-distance send/recv on cst,
  // chunk d of K_g U_full on st waits only for ev_chunk[d]
  bool overlap = true;
  CholDist cdist;          // the N x N Cholesky's large levels split over the ranks
  // planar 3M for K_g U and the local Gram / TRMM (TRAJ_PLANAR_KU / TRAJ_PLANAR_CQR, N >= TRAJ_PLANAR_MIN_N)
  bool planar = false;
  long long ldKs = 0, ldPs = 0;
  // Strassen (slv levels) on each K-chunk product K_g[:, s] U_s (TRAJ_STRASSEN=0: off): U_s's operands
  // Sb and the leaf products Sm [3 7^lv][Lp/2^lv][ldSM], shared by the chunks
  int slv = 0;
  long long ldS = 0, ldSM = 0;
  double *Sb = nullptr, *Sm = nullptr;
  double *Cp = nullptr, *Gp = nullptr, *Xp = nullptr;   // chunk planes [3][Lp], Gram / X planes [3][N]
  // modular engine (TRAJ_OZAKI, N >= TRAJ_PLANAR_MIN_N): K_g U as P chunk products K_g[:, s] U_s whose
  // residues accumulate in RC (U_s split with the GLOBAL column exponents eG of U, from the column norms
  // summed over the shards), one CRT combine; the local Grams and TRMMs as in the unsharded step
  bool oz = false;
  // TRAJ_SHARD_OZ_CHUNKS=1: K_g U as the P ring-ordered chunk products (residues accumulated in the
  // epilogue, the NCCL exchange under them); default: the gathered U, one product of depth L
  bool oz_chunked = false;
  int oz_s = 16, oz_s_corr = 10;
  int8_t *RU = nullptr, *RX = nullptr;
  uint8_t* RC = nullptr;
  size_t RC_bytes = 0;
  int *eU = nullptr, *eU2 = nullptr, *eX = nullptr, *eG = nullptr;
  double *oz_part = nullptr, *nu2 = nullptr;
  int oz_proj_min = 1024;   // click count from which the projective rank-k products and the structured
                            // pass 1's solve go modular (TRAJ_OZAKI_PROJ_MIN)
  bool struct_serial = false;           // TRAJ_STRUCT_PIPELINE=0: structured factor and solve on one stream
  std::vector<cudaEvent_t> sc_ev;       // per-block events of the pipelined structured pass 1
  cplx* dist_scratch = nullptr;
  size_t dist_scratch_bytes = 0;
  cudaStream_t cst = nullptr;
  cudaEvent_t ev_start = nullptr;
  std::vector<cudaEvent_t> ev_chunk;
  cusolverDnHandle_t solver = nullptr;
  Profiler* prof = nullptr;
  bool test_stall = false;       // TRAJ_WATCHDOG_TEST_STALL=1 (NCCL mode): watchdog test hook
  double *obs_bins = nullptr, *obs_part = nullptr, *obs_out = nullptr;
  int32_t* obs_mask = nullptr;
};

// Validates the sharding fields; fills the geometry of sh.
int shard_validate(const traj_config* c, std::string* why);
// banded: the compiled half-widths (Wx, Wy) of the banded propagator, or false for the dense K
size_t shard_carve(ShardedCtx* sh, const traj_config* c, char* base, int lwork, bool banded = false, int Wx = 0,
                   int Wy = 0);
// halo rows of the banded sharded propagator and whether they fit the shard geometry
bool shard_banded_fits(const traj_config* c, int Wx, int Wy, std::string* why);
int shard_init(ShardedCtx* sh, const traj_config* c, std::string* err);
int shard_build(ShardedCtx* sh, const std::vector<std::complex<double>>& kc, const std::vector<int32_t>& sites,
                std::string* err, const std::vector<std::complex<double>>* band = nullptr);
int shard_step(ShardedCtx* sh, long long* step, std::string* err);
int shard_step_impl(ShardedCtx* sh, long long* step, std::string* err);
int shard_orthonormalize(ShardedCtx* sh, std::string* err);
int shard_entropy(ShardedCtx* sh, const int64_t* A, int64_t nA, double* S_out, std::string* err);
int shard_occupations(ShardedCtx* sh, double* n_out, long long step, std::string* err);
int shard_correlation_rows(ShardedCtx* sh, int64_t row0, int64_t nrows, void* C_out, std::string* err);
int shard_get_state(ShardedCtx* sh, void* U_out, std::string* err);
int shard_set_state(ShardedCtx* sh, const void* U_in, std::string* err);
int shard_failed(ShardedCtx* sh, int32_t* flag, std::string* err);
// allgather the current U into sh->Ufull (L x ldN, row-major)
int shard_full_state(ShardedCtx* sh, std::string* err);
void shard_destroy(ShardedCtx* sh);
int nccl_unique_id(void* out128, std::string* err);

}  // namespace traj
