// C-ABI of libtraj.so (include/traj.h): handle, workspace, K construction, the
// trajectory step and the sampled observables.  Host code only orchestrates; every
// arithmetic step of the path runs in the kernels of zgemm.cu, cholinv.cu, monitor.cu
// and (eigvalsh, the one vendor call allowed by the north star) cuSOLVER.
#include <cusolverDn.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <complex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/traj.h"
#include "cholinv.h"
#include "common.cuh"
#include "monitor.h"
#include "zgemm.h"
#include "profiler.h"
#include "shard.h"
#include "banded.h"
#include "qsd_rk4.h"
#include "pm_events.h"
#include "igemm.h"
#include "ozaki.h"
#include "probe.h"
#include "dgemm.h"
#include "igemm.h"
#include "ozaki.h"
#include "planar.h"
#include "small_step.h"
#include "comm_plan.h"
#include "structchol.h"

namespace traj {
std::atomic<long long> g_kernel_launches{0};
}

using namespace traj;

struct traj_ctx {
  traj_config cfg;
  ShardedCtx* sh = nullptr;        // row-sharded mode (shard_size > 1 or an NCCL communicator)
  bool banded = false;             // TRAJ_PROP_BANDED with a band narrower than the lattice
  int Wx = 0, Wy = 0;              // compiled half-bandwidths per axis
  cplx* bcoef = nullptr;           // [2Wx+1 | 2Wy+1] stencil coefficients (device copy)
  // planar 3M dense propagator (planar.cu, TRAJ_PLANAR_KU=0: the interleaved zgemm): K planes
  // [3][L][ldK], U planes and product planes [T][3][L][ldP]
  bool planar = false;
  double *Kp = nullptr, *Up = nullptr, *Pp = nullptr;
  long long ldK = 0, ldP = 0;
  // planar CholeskyQR (TRAJ_PLANAR_CQR=0: interleaved): measured Grams as three real U^T U-type
  // products, TRMMs as three real products against X's planes (Xp).  Up holds 6 planes, (re, im,
  // re - im, re, im, re + im), plane-major [plane][T][L][ldP]: planes 0..2 and 3..5 are
  // constant-stride triples over all trajectories, so each group of three products is one launch
  bool planar_cqr = false;
  double* Xp = nullptr;
  // Strassen (1 or 2 levels) on each planar product of K U (planar.cu; TRAJ_STRASSEN=0: off): K's
  // 7^lv operands per plane Ks [3][7^lv][L/2^lv][ldS], U's Bc (in Up's space) and the products Ms
  // [3][7^lv][T][L/2^lv][ldM]
  bool strassen = false;
  int slv = 0;
  double *Ks = nullptr, *Bc = nullptr, *Ms = nullptr;
  long long ldS = 0, ldM = 0;
  // exact modular complex products on the INT8 tensor cores (ozaki.h; TRAJ_OZAKI=0: the DMMA paths):
  // oz_ku = the dense propagator K U, oz_cqr = the CholeskyQR Grams and TRMMs.  K's residues RK
  // [3][s][L][oz_ld(L)] with row exponents eK are formed once; per product U's (or X's) residues
  // RU / RX, the residue products RC [3][s][T][rows][oz_ld(N)] and the row / column exponents eU, eX
  bool oz_ku = false, oz_cqr = false;
  int oz_s = 16;
  int oz_proj_min = 1024;   // click count from which the projective rank-k products go modular (TRAJ_OZAKI_PROJ_MIN)
  int oz_struct_min = 1024; // click capacity from which the structured pass 1's solve goes modular (TRAJ_OZAKI_STRUCT_MIN; default: oz_proj_min)
  int oz_s_corr = 10;   // moduli of the second pass's first-order correction src (X - I) (TRAJ_OZAKI_CORR_MODULI; 0: full)
  int oz_s_low = 8;     // ... when every column norm of X - I is <= 2^(beta_low - 55.5) / N (TRAJ_OZAKI_CORR_LOW; 0: no low tier)
  int8_t *RK = nullptr, *RU = nullptr, *RX = nullptr;
  uint8_t* RC = nullptr;
  int *eK = nullptr, *eU = nullptr, *eX = nullptr, *eU2 = nullptr;
  double* oz_part = nullptr;
  size_t RC_bytes = 0;
  CholOzaki coz;                   // chol_inverse's large levels on the modular path (RU / RX / RC as scratch)
  std::vector<cplx> band_host;     // the same on the host: passed by value to the stencil launches
  cplx* Wrk = nullptr;             // RK4 QSD scratch, shaped like U
  // event-driven PM (NEXT-4)
  std::vector<long long> ev_count;
  std::vector<double> ev_tnext, ev_tcur;
  cplx* yhat = nullptr;
  double* ev_coef = nullptr;
  cplx* ev_y2 = nullptr;           // one-pass events: [2][N] unnormalised yhat
  double* ev_c2 = nullptr;         // [2][8] coef
  double2* ev_g2 = nullptr;        // [2][L] g = U yhat^dag
  cplx* ev_tmp = nullptr;          // 2d lattices: [L][ldN] the x-axis half of the separable pass
  double2* ev_gx = nullptr;        // ... and [L] the x-axis half of K g
  double* ev_part = nullptr;       // [64] prep partials
  bool ev_onepass = true;          // TRAJ_EVENTS_ONEPASS=0: two-pass event updates
  int32_t* occ_count = nullptr;
  cplx* taps_dev = nullptr;
  std::complex<double>* taps_host = nullptr;   // pinned staging
  double* dbuf = nullptr;          // RK4 QSD diagonal generator [T][L]
  std::vector<double> gamma;
  int L = 0, N = 0, Lx = 0, Ly = 0, T = 0, cap = 0;
  long long ldN = 0, ldL = 0, ldcap = 0, sU = 0, sG = 0;
  cudaStream_t st = nullptr;
  // CholeskyQR pass 1: the factorisation runs on st_hi (high priority) while the TRMM of X's left
  // block runs on st_lo as soon as that block is final (TRAJ_CHOL_OVERLAP=0: serial)
  bool chol_overlap = true;
  cudaStream_t st_hi = nullptr, st_lo = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_left = nullptr, ev_lo_done = nullptr, ev_hi_done = nullptr, ev_split = nullptr;
  cplx* K = nullptr;
  cplx* U[2] = {nullptr, nullptr};
  int cur = 0;
  cplx* G = nullptr;
  cplx* X = nullptr;
  void* chol_scratch = nullptr;
  double* gamma_dev = nullptr;
  double* nbuf = nullptr;
  int32_t* failed_dev = nullptr;
  // projective
  int32_t *flags = nullptr, *S = nullptr, *count = nullptr, *occ = nullptr, *pos1 = nullptr, *S1 = nullptr,
          *S0 = nullptr, *k1 = nullptr, *k0 = nullptr;
  cplx *US = nullptr, *D0 = nullptr, *Dw = nullptr, *D11 = nullptr, *X11 = nullptr, *W = nullptr, *Tm = nullptr;
  cplx *Linv = nullptr, *DLinv = nullptr, *Ybuf = nullptr, *Zbuf = nullptr;
  cplx* Tm2 = nullptr;             // split-K partner of Tm (one trajectory)
  void* chol_scratch_small = nullptr;
  long long sUS = 0, sD = 0;
  // observables
  double* eig_w = nullptr;
  cplx* eig_work = nullptr;
  int lwork = 0;
  int* eig_info = nullptr;
  double* S_dev = nullptr;
  int32_t* bad_dev = nullptr;
  unsigned long long* gdev = nullptr;   // per-trajectory max |G2 - I| of the second CQR pass
  int32_t* region = nullptr;
  bool full_cqr2 = false;                // TRAJ_CQR2_FULL=1: always factor G2 by chol_inverse
  bool lowrank_gram = true;              // TRAJ_LOWRANK_GRAM=0: always measure the first Gram
  bool lowrank_orth = false;             // TRAJ_ORTH_LOWRANK
  bool lowrank_refine = true;            // TRAJ_LOWRANK_REFINE=0: never refine (drift studies only)
  double lowrank_tol = 5e-13;            // TRAJ_LOWRANK_TOL: refine when the probed ||U^dag U - I||_F exceeds it
  cplx *PX = nullptr, *PY = nullptr, *Ppart = nullptr;
  double* pest = nullptr;
  long long lowrank_probes = 0, lowrank_refinements = 0;
  cplx *Mb = nullptr, *Yb = nullptr, *Zb = nullptr, *Tb = nullptr, *Pb = nullptr, *Qb = nullptr, *FV = nullptr;
  long long lowrank_iters = 0, lowrank_fallbacks = 0;
  int lr_k0 = -1;                        // >= 0: pass-1 Gram of this step = I - V^dag V, V (k0 rows) in US
  double* obs_bins = nullptr;            // C(r) accumulators [L]
  double* obs_part = nullptr;            // reduction partials [1024]
  double* obs_out = nullptr;             // [n_traj]
  int32_t* obs_mask = nullptr;           // region indicator [L]
  long long cqr2_fallbacks = 0;
  unsigned long long* fb_dev = nullptr;  // CholeskyQR2 second passes that took the full factorisation
  int32_t* gate = nullptr;               // [1]: this step's second-pass decision (device)
  CholFallbackGraph fbg;                 // the decision + the conditional factorisation as one graph
  int fbg_state = 0;                     // 0: not built yet, 1: built, -1: unavailable (gated launches)
  std::vector<int32_t> hcount;           // host click counts of the current step (host Philox)
  bool k1_dev = false;                   // the last projective step's occupied counts are in k1 (device)
  const int32_t* lr_kdev = nullptr;      // device bound of pass 1's V rows (k0), with lr_k0 its capacity
  // CholeskyQR pass 1 on the structure G = I - V^dag V (structured_pass1; TRAJ_STRUCT_CHOL=0: dense)
  bool struct_chol = true;
  bool struct_serial = false;            // TRAJ_STRUCT_PIPELINE=0: factor and solve on one stream
  std::vector<cudaEvent_t> sc_ev;        // per-block events of the pipelined structured pass 1
  int sb = 128;                          // column block of the structured factorisation
  cplx *sY = nullptr, *sC = nullptr, *sX = nullptr, *sW = nullptr, *sZ = nullptr;
  void* s_chol_scratch = nullptr;
  bool struct_batched = true;            // the batched structured factor (structchol.h)
  cplx *sSb = nullptr, *sXMb = nullptr, *sQb = nullptr, *sCb = nullptr;
  long long sbS = 0, sEs = 0;
  cplx* sEb = nullptr;
  void* s_bscratch = nullptr;
  int32_t* s_bfail = nullptr;
  cplx* kcoef = nullptr;
  int32_t* sites = nullptr;
  cusolverDnHandle_t solver = nullptr;
  long long step = 0;
  int32_t* h_small = nullptr;     // pinned host scratch
  double* h_dev = nullptr;        // pinned host copy of gdev
  std::vector<int64_t> last_nS, last_n1;
  // fused small-lattice step (small_step.cu; TRAJ_SMALL_STEP=0: the general path): U, the step's
  // scratch and the sampler fit one CTA's shared memory, one CTA per trajectory, one launch per
  // traj_step call; the last step's click counts stay on the device (small_last [T][2])
  bool small = false;
  int32_t* small_last = nullptr;
  unsigned long long* small_fallbacks = nullptr;   // full second-pass factorisations in the fused step
  bool small_last_dev = false;
  std::string err;
  Profiler prof;
};

namespace {

thread_local std::string g_err;

int fail(traj_ctx* h, int status, const std::string& msg) {
  if (h) h->err = msg;
  g_err = msg;
  return status;
}

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) return fail(h, TRAJ_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define TRY(x)                          \
  do {                                  \
    int s_ = (x);                       \
    if (s_) return fail(h, s_, h->err); \
  } while (0)

struct Layout {
  size_t off = 0;
  char* base = nullptr;
  template <typename P>
  void take(P*& p, size_t bytes) {
    off = (off + 255) & ~size_t(255);
    p = base ? reinterpret_cast<P*>(base + off) : nullptr;
    off += bytes;
  }
};

int validate(const traj_config* c, std::string* why) {
  auto bad = [&](const char* m) {
    *why = m;
    return TRAJ_ECONFIG;
  };
  if (!c) return bad("null config");
  if (c->dim != 1 && c->dim != 2) return bad("dim must be 1 or 2");
  if (c->dim == 1 && c->Ly != 1) return bad("1d needs Ly = 1");
  if (c->dim == 1 && c->Lx < 2) return bad("1d needs Lx >= 2");
  if (c->dim == 2 && (c->Lx < 3 || c->Ly < 3)) return bad("2d needs Lx, Ly >= 3");
  const long long L = c->Lx * c->Ly;
  if (L % 2) return bad("L = Lx*Ly must be even (half filling)");
  if (L > (1ll << 20)) return bad("L too large");
  if (c->N != L / 2) return bad("N must equal L/2 (P:43)");
  if (!(c->dt > 0) || !isfinite(c->dt)) return bad("dt must be > 0");
  if (!isfinite(c->J)) return bad("J must be finite");
  if (c->protocol != TRAJ_PROJECTIVE && c->protocol != TRAJ_HOMODYNE && c->protocol != TRAJ_HOMODYNE_RK4 &&
      c->protocol != TRAJ_PROJECTIVE_EVENTS)
    return bad("unknown protocol");
  if (c->init != TRAJ_INIT_NEEL && !(c->init == TRAJ_INIT_CHECKERBOARD && c->dim == 2))
    return bad("init must be TRAJ_INIT_NEEL, or TRAJ_INIT_CHECKERBOARD in 2d");
  if (c->n_traj < 1 || c->n_traj > 65535) return bad("n_traj must be in [1, 65535]");
  if (c->traj_base < 0 || c->traj_base + c->n_traj > (1ll << 32)) return bad("trajectory ids must fit 32 bits");
  if (!c->gamma) return bad("gamma is null");
  for (long long t = 0; t < c->n_traj; ++t) {
    const double g = c->gamma[t];
    if (!(g >= 0) || !isfinite(g)) return bad("gamma must be >= 0 and finite");
    if (c->protocol == TRAJ_PROJECTIVE && g * c->dt > 1.0) return bad("projective needs gamma*dt <= 1 (Q10)");
  }
  if (c->propagator != TRAJ_PROP_DENSE && c->propagator != TRAJ_PROP_BANDED) return bad("unknown propagator");
  if (c->orthonormalizer != TRAJ_ORTH_CQR2 && c->orthonormalizer != TRAJ_ORTH_LOWRANK)
    return bad("unknown orthonormalizer");
  if (c->shard_size != 1 || c->nccl_id) {
    if (c->protocol == TRAJ_HOMODYNE_RK4) return bad("the RK4 QSD protocol is not combined with row sharding");
    if (c->protocol == TRAJ_PROJECTIVE_EVENTS) return bad("the event-driven protocol is not combined with row sharding");
    if (c->orthonormalizer == TRAJ_ORTH_LOWRANK) return bad("the low-rank orthonormaliser is not combined with row sharding");
    return shard_validate(c, why);
  }
  if (c->shard_rank != 0) return bad("shard_rank must be 0 without sharding");
  return 0;
}

// click-list capacity: mean + 12 sigma + 64 of Binomial(L, p), at most L
int click_capacity(long long L, const traj_config* c) {
  if (c->protocol != TRAJ_PROJECTIVE) return 0;
  double pmax = 0;
  for (long long t = 0; t < c->n_traj; ++t) pmax = std::max(pmax, c->gamma[t] * c->dt);
  const double m = L * pmax, sd = sqrt(L * pmax * (1 - pmax));
  return (int)std::min<long long>(L, (long long)ceil(m + 12 * sd + 64));
}

std::vector<std::complex<double>> ring_coefficients(int n, double J, double dt);
constexpr long long EV_TAPCAP = 1 << 20;     // complex taps staged per upload (event-driven PM)

// half-bandwidth of a ring propagator: smallest w with sum_{w < |d| <= n/2} |c_d| < 1e-18
int band_width(const std::vector<std::complex<double>>& c) {
  const int n = (int)c.size();
  double tail = 0.0;
  for (int d = n / 2; d >= 1; --d) {
    tail += std::abs(c[d]) + (n - d != d ? std::abs(c[n - d]) : 0.0);
    if (tail >= 1e-18) return d;
  }
  return 0;
}

// compiled widths (Wx, Wy) for the banded propagator, or false if it does not fit
bool banded_widths(const traj_config* c, int* Wx, int* Wy) {
  if (c->propagator != TRAJ_PROP_BANDED) return false;
  const int wx = banded_template_width(band_width(ring_coefficients((int)c->Lx, c->J, c->dt)));
  const int wy = c->Ly > 1 ? banded_template_width(band_width(ring_coefficients((int)c->Ly, c->J, c->dt))) : 0;
  if (wx < 0 || wy < 0 || 2 * wx + 1 > c->Lx || (c->Ly > 1 && 2 * wy + 1 > c->Ly)) return false;
  *Wx = wx;
  *Wy = wy;
  return true;
}

size_t carve(traj_ctx* h, const traj_config* c, char* base, int lwork) {
  Layout lay;
  lay.base = base;
  const long long Lx = c->Lx, Ly = c->Ly, L = Lx * Ly, N = c->N, T = c->n_traj;
  const long long ldN = round_up(N, 8), ldL = round_up(L, 8);
  const int cap = click_capacity(L, c);
  const long long ldcap = round_up(std::max(cap, 1), 8);
  h->L = (int)L;
  h->N = (int)N;
  h->Lx = (int)Lx;
  h->Ly = (int)Ly;
  h->T = (int)T;
  h->cap = cap;
  h->ldN = ldN;
  h->ldL = ldL;
  h->ldcap = ldcap;
  h->sU = L * ldN;
  h->sG = N * ldN;
  h->banded = banded_widths(c, &h->Wx, &h->Wy);
  {
    const char* pk = getenv("TRAJ_PLANAR_KU");
    // below N = 512 the split / combine passes and the 128 x 128 tiles cost more than they save
    // (TRAJ_PLANAR_MIN_N overrides the threshold, e.g. for small parity tests)
    const char* mn = getenv("TRAJ_PLANAR_MIN_N");
    const long long min_n = mn ? atoll(mn) : 512;
    h->planar = !h->banded && c->protocol != TRAJ_HOMODYNE_RK4 && c->protocol != TRAJ_PROJECTIVE_EVENTS &&
                !(pk && pk[0] == '0') && N >= min_n;
    const char* pc = getenv("TRAJ_PLANAR_CQR");
    h->planar_cqr = !(pc && pc[0] == '0') && N >= min_n;
    // the modular INT8 products replace both DMMA paths from the same size on (TRAJ_OZAKI=0: off,
    // TRAJ_OZAKI_MODULI: 4..18 even, default 16 = beta 57 bits per operand row / column; 18 = 61)
    const char* oz = getenv("TRAJ_OZAKI");
    const char* om = getenv("TRAJ_OZAKI_MODULI");
    h->oz_s = om ? atoi(om) : 16;
    const char* opm = getenv("TRAJ_OZAKI_PROJ_MIN");
    h->oz_proj_min = opm ? atoi(opm) : 1024;
    const char* osm = getenv("TRAJ_OZAKI_STRUCT_MIN");
    h->oz_struct_min = osm ? atoi(osm) : h->oz_proj_min;
    const char* oc = getenv("TRAJ_OZAKI_CORR_MODULI");
    h->oz_s_corr = oc ? atoi(oc) : 10;
    if (h->oz_s_corr != 0 && !oz_supported(h->oz_s_corr)) h->oz_s_corr = 10;
    const char* ol = getenv("TRAJ_OZAKI_CORR_LOW");
    h->oz_s_low = ol ? atoi(ol) : 8;
    if (h->oz_s_low != 0 && (!oz_supported(h->oz_s_low) || h->oz_s_low >= h->oz_s_corr || 8 * h->L < 9 * h->N))
      h->oz_s_low = 0;
    const bool oz_on = !(oz && oz[0] == '0') && oz_supported(h->oz_s) && N >= min_n && L <= 65535;
    h->oz_cqr = oz_on;
    h->oz_ku = oz_on && h->planar;
    if (h->oz_ku) h->planar = false;
    if (h->oz_cqr) h->planar_cqr = false;
  }
  if (c->protocol == TRAJ_HOMODYNE_RK4) {     // stencil generator: no K
    h->banded = false;
    lay.take(h->Wrk, (size_t)T * L * ldN * 16);
    lay.take(h->dbuf, (size_t)T * L * 8);
  } else if (c->protocol == TRAJ_PROJECTIVE_EVENTS) {   // per-event stencils: no K
    h->banded = false;
    lay.take(h->yhat, (size_t)N * 16);
    lay.take(h->ev_coef, 64);
    lay.take(h->ev_y2, (size_t)2 * N * 16);
    lay.take(h->ev_c2, 2 * 8 * 8);
    lay.take(h->ev_g2, (size_t)2 * L * 16);
    if (h->Ly > 1) {
      lay.take(h->ev_tmp, (size_t)L * ldN * 16);
      lay.take(h->ev_gx, (size_t)L * 16);
    }
    lay.take(h->ev_part, 64 * 8);
    lay.take(h->occ_count, (size_t)T * 4);
    lay.take(h->taps_dev, (size_t)EV_TAPCAP * 16);
  } else if (h->banded) {
    lay.take(h->bcoef, (size_t)(2 * h->Wx + 2 * h->Wy + 2) * 16);
  } else if (h->planar) {
    h->ldK = round_up(L, 16);
    lay.take(h->Kp, (size_t)3 * L * h->ldK * 8);
    const char* sv = getenv("TRAJ_STRASSEN");
    const char* sm = getenv("TRAJ_STRASSEN_MIN_N");
    const long long smin = sm ? atoll(sm) : 2048;
    h->strassen = !(sv && sv[0] == '0') && L % 4 == 0 && N >= smin;
    if (h->strassen) {
      // two levels when K's 147 quarter operands fit 24 GB (c3: 19.7 GB, c4: 1.2 GB; c4 391 vs 401 ms
      // per step with one level, c2 (N = 1024) is below TRAJ_STRASSEN_MIN_N), else one (c5); three
      // for one trajectory when K's 1029 eighth-size operands fit 40 GB (c3: 34.5 GB)
      const char* lv = getenv("TRAJ_STRASSEN_LEVELS");
      const bool two_ok = L % 8 == 0 && 147.0 * (L / 4) * round_up(L / 4, 16) * 8 <= 24e9;
      const bool three_ok = T == 1 && L % 16 == 0 && 1029.0 * (L / 8) * round_up(L / 8, 16) * 8 <= 40e9;
      const int want = lv ? atoi(lv) : 3;
      h->slv = want >= 3 && three_ok ? 3 : (want >= 2 && two_ok ? 2 : 1);
      const long long hh = L >> h->slv, ns = strassen_products(h->slv);
      h->ldS = round_up(hh, 16);
      h->ldM = round_up(N >> h->slv, 16);
      lay.take(h->Ks, (size_t)ns * hh * h->ldS * 8);
      // the products alias K's planes once Ks is built, when they fit (one trajectory)
      const size_t mb = (size_t)ns * T * hh * h->ldM * 8;
      if (mb <= (size_t)3 * L * h->ldK * 8) h->Ms = h->Kp;
      else lay.take(h->Ms, mb);
    }
  } else if (!h->oz_ku) {
    lay.take(h->K, (size_t)L * ldL * 16);
  }
  if (h->oz_ku || h->oz_cqr) {
    const long long s = h->oz_s;
    const size_t ru = (size_t)std::max(oz_residue_bytes(4, s, T, N, L), oz_residue_bytes(3, s, T, L, N));
    h->RC_bytes = (size_t)oz_residue_bytes(3, s, T, L, N);   // (two product planes needed; the structured solve splits it in halves)
    if (h->oz_ku) {
      lay.take(h->RK, (size_t)oz_residue_bytes(2, s, 1, L, L));
      lay.take(h->eK, (size_t)L * 4);
      h->RC_bytes = std::max<size_t>(h->RC_bytes, (size_t)L * ldL * 16);   // K is built there before its split
    }
    lay.take(h->RU, ru);
    lay.take(h->RC, h->RC_bytes);
    if (h->oz_cqr) lay.take(h->RX, (size_t)oz_residue_bytes(3, s, T, N, N));
    lay.take(h->eU, (size_t)T * L * 4);
    lay.take(h->eU2, (size_t)T * L * 4);
    lay.take(h->eX, (size_t)T * N * 4);
    lay.take(h->oz_part, (size_t)8 * T * L * 8);
  }
  if (h->planar || h->planar_cqr) {
    h->ldP = round_up(N, 16);
    lay.take(h->Up, (size_t)T * std::max<long long>(6 * L * h->ldP,
                                                     h->strassen ? strassen_products(h->slv) * (L >> h->slv) * h->ldM
                                                                 : 0) * 8);
    h->Bc = h->Up;   // U's Strassen operands use the plane buffer (free during K U)
    lay.take(h->Pp, (size_t)T * 3 * L * h->ldP * 8);
    if (h->planar_cqr) lay.take(h->Xp, (size_t)T * 3 * N * h->ldP * 8);
  }
  lay.take(h->small_last, (size_t)T * 2 * 4);
  lay.take(h->small_fallbacks, 8);
  lay.take(h->U[0], (size_t)T * L * ldN * 16);
  lay.take(h->U[1], (size_t)T * L * ldN * 16);
  lay.take(h->G, (size_t)T * N * ldN * 16);
  lay.take(h->X, (size_t)T * N * ldN * 16);
  lay.take(h->chol_scratch, chol_scratch_bytes(N, T));
  lay.take(h->gamma_dev, (size_t)T * 8);
  lay.take(h->nbuf, (size_t)T * L * 8);
  lay.take(h->failed_dev, (size_t)T * 4);
  lay.take(h->eig_w, (size_t)N * 8);
  lay.take(h->eig_work, (size_t)std::max(lwork, 1) * 16);
  lay.take(h->eig_info, 16);
  lay.take(h->S_dev, (size_t)T * 8);
  lay.take(h->bad_dev, (size_t)T * 4);
  lay.take(h->gdev, (size_t)T * 8);
  lay.take(h->fb_dev, 8);
  lay.take(h->gate, 16);
  lay.take(h->obs_bins, (size_t)L * 8);
  lay.take(h->obs_part, 1024 * 8);
  lay.take(h->obs_out, (size_t)T * 8);
  lay.take(h->obs_mask, (size_t)L * 4);
  lay.take(h->region, (size_t)L * 4);
  lay.take(h->kcoef, (size_t)(Lx + Ly) * 16);
  lay.take(h->sites, (size_t)N * 4);
  lay.take(h->PX, probe_x_bytes(N, T));
  lay.take(h->PY, probe_y_bytes(L, T));
  lay.take(h->Ppart, probe_partial_bytes(N, T));
  lay.take(h->pest, (size_t)T * 8);
  if (cap > 0) {
    h->sUS = (long long)cap * ldN;
    h->sD = (long long)cap * ldcap;
    lay.take(h->flags, (size_t)T * L * 4);
    lay.take(h->S, (size_t)T * cap * 4);
    lay.take(h->count, (size_t)T * 4);
    lay.take(h->occ, (size_t)T * cap * 4);
    lay.take(h->pos1, (size_t)T * cap * 4);
    lay.take(h->S1, (size_t)T * cap * 4);
    lay.take(h->S0, (size_t)T * cap * 4);
    lay.take(h->k1, (size_t)T * 4);
    lay.take(h->k0, (size_t)T * 4);
    lay.take(h->US, (size_t)T * cap * ldN * 16);
    lay.take(h->D0, (size_t)T * cap * ldcap * 16);
    lay.take(h->Dw, (size_t)T * cap * ldcap * 16);
    lay.take(h->Linv, (size_t)T * 64 * 64 * 16);
    lay.take(h->DLinv, (size_t)T * 64 * 64 * 16);
    lay.take(h->Ybuf, (size_t)T * 64 * ldcap * 16);
    lay.take(h->Zbuf, (size_t)T * 64 * ldcap * 16);
    lay.take(h->D11, (size_t)T * cap * ldcap * 16);
    lay.take(h->X11, (size_t)T * cap * ldcap * 16);
    lay.take(h->chol_scratch_small, chol_scratch_bytes(cap, T));
    lay.take(h->W, (size_t)T * N * ldcap * 16);
    lay.take(h->Tm, (size_t)T * L * ldcap * 16);
    if (T == 1) lay.take(h->Tm2, (size_t)L * ldcap * 16);
    if (c->orthonormalizer == TRAJ_ORTH_LOWRANK) {
      for (cplx** b : {&h->Mb, &h->Yb, &h->Zb, &h->Tb, &h->Pb, &h->Qb}) lay.take(*b, (size_t)T * cap * ldcap * 16);
      lay.take(h->FV, (size_t)T * cap * ldN * 16);
    }
    {   // structured CholeskyQR pass 1 (structured_pass1): Y [cap][sb], C [sb][sb], the blocks' R^-1
        // [N][sb], W = V X and Z = M W [cap][ldN]
      // wider blocks when many rows are zeroed (c5: k0 ~ 1800): the solve's L x b x k0 products fill
      // the GPU better and the factor has fewer sequential blocks (measured: c5 chol phase 399 ms at
      // b = 128, 306 ms at 512; c3 flat from 128 to 512)
      const char* sbv = getenv("TRAJ_STRUCT_B");
      // on the modular path the solve's per-block residue splits of the L x k0 accumulator favour fewer,
      // wider blocks (c5: 2048)
      h->sb = sbv ? std::max(16, std::min(4096, atoi(sbv) / 16 * 16))
                  : (cap >= 1024 ? (h->oz_cqr && cap >= h->oz_struct_min ? 2048 : 512) : 128);
      const long long b = h->sb;
      lay.take(h->sY, (size_t)T * cap * b * 16);
      lay.take(h->sC, (size_t)T * b * b * 16);
      lay.take(h->sX, (size_t)T * round_up(N, b) * b * 16);
      lay.take(h->sW, (size_t)T * cap * ldN * 16);
      lay.take(h->sZ, (size_t)T * cap * ldN * 16);
      lay.take(h->s_chol_scratch, chol_scratch_bytes(b, T));
      // the batched factor (struct_chol_factor_batched; TRAJ_STRUCT_BATCHED=0: the sequential chain)
      const char* sbat = getenv("TRAJ_STRUCT_BATCHED");
      h->struct_batched = !(sbat && sbat[0] == '0');
      // (DMMA solve only: with the modular solve (c5) the sequential chain pipelines each factor block
      // under the solve on two streams, measured faster than the batched factor followed by the solve)
      if (h->struct_batched && !(h->oz_cqr && cap >= h->oz_struct_min)) {
        const long long nblk = ceil_div(N, b);
        if (nblk > 1) {   // the batched solve's prefix sums
          h->sEs = (long long)L * ldcap;
          lay.take(h->sEb, (size_t)(nblk - 1) * h->sEs * 16);
        }
        h->sbS = (long long)cap * std::max<long long>(ldcap, b);
        lay.take(h->sSb, (size_t)nblk * h->sbS * 16);
        lay.take(h->sXMb, (size_t)nblk * h->sbS * 16);
        lay.take(h->sQb, (size_t)nblk * cap * b * 16);
        lay.take(h->sCb, (size_t)nblk * b * b * 16);
        lay.take(h->s_bscratch, std::max(chol_scratch_bytes(cap, nblk), chol_scratch_bytes(b, nblk)));
        lay.take(h->s_bfail, (size_t)2 * nblk * 4);
      }
    }
  }
  return lay.off + 256;
}

int eig_lwork(int N, int* lwork, std::string* why) {
  cusolverDnHandle_t s;
  if (cusolverDnCreate(&s) != CUSOLVER_STATUS_SUCCESS) {
    *why = "cusolverDnCreate failed (no CUDA device?)";
    return TRAJ_ECUDA;
  }
  int lw = 0;
  cusolverStatus_t r = cusolverDnZheevd_bufferSize(s, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, N, nullptr,
                                                   N, nullptr, &lw);
  cusolverDnDestroy(s);
  if (r != CUSOLVER_STATUS_SUCCESS) {
    *why = "cusolverDnZheevd_bufferSize failed";
    return TRAJ_ECUDA;
  }
  *lwork = lw;
  return 0;
}

// 1d coefficient row of K = exp(-i H~ dt) on a ring of n sites:
//   K_{ij} = c[(j - i) mod n],  c_d = sum_{m in Z, m = d mod n} (-i)^|m| J_|m|(2 J dt)
// (Jacobi-Anger generating function of the Bessel functions; H~ = J (T + T^-1)).
std::vector<std::complex<double>> ring_coefficients(int n, double J, double dt) {
  std::vector<std::complex<double>> c(n, 0.0);
  const double x = 2.0 * J * dt;
  const int mmax = (int)ceil(fabs(x)) + 80;
  const std::complex<double> ph[4] = {{1, 0}, {0, -1}, {-1, 0}, {0, 1}};
  for (int m = -mmax; m <= mmax; ++m) {
    const int a = m < 0 ? -m : m;
    const double jv = jn(a, x);
    if (jv == 0.0) continue;
    c[((m % n) + n) % n] += ph[a & 3] * jv;
  }
  return c;
}

// CholeskyQR2 on U (state), tmp another buffer of the same shape; result in U.
// Pass 2 sees G2 = I + E with |E| ~ kappa(U)^2 eps: its Cholesky inverse is taken from the
// first-order closed form (exact up to N |E|^2, below rounding when N max|E|^2 < 1e-18,
// checked on the device per step); otherwise, or with TRAJ_CQR2_FULL=1, chol_inverse.
// C (M x Nc, ld h->ldcap) = A (M x K, ld lda) op(B) for a skinny output (Nc = a click count, K = N):
// with one trajectory the K range is split in two halves run as one batch-2 launch (twice the CTAs
// for the few output tiles), the second half into Tm2, then added; otherwise one launch.
int skinny_gemm(traj_ctx* h, int opB, long long M, long long Nc, long long K, const cplx* A, long long lda, long long sA,
                const cplx* B, long long ldb, long long sB, cplx* C, long long sC, const int32_t* nc_dev = nullptr) {
  const long long tiles = ceil_div(M, 64) * ceil_div(Nc, 64);
  DevBounds db;             // output columns needed per trajectory (device), Nc their capacity
  db.n = nc_dev;
  if (h->T != 1 || !h->Tm2 || C != h->Tm || K < 2048 || K % 32 || tiles >= 8 * 148)
    return zgemm(h->st, 0, opB, M, Nc, K, 1.0, 0.0, A, lda, sA, B, ldb, sB, 0.0, C, h->ldcap, sC, h->T, 0, &h->err, 0, 0,
                 &db);
  db.per_batch = 0;         // the batch of two is the two K halves of the one trajectory
  // batch entry z in {0, 1} takes k in [z K/2, (z + 1) K/2): A's columns and B's rows (opB = 0) or
  // columns (opB = 1) at a batch stride of K/2, the outputs at Tm and Tm2 (stride Tm2 - Tm)
  const long long k2 = K / 2;
  int s = zgemm(h->st, 0, opB, M, Nc, k2, 1.0, 0.0, A, lda, k2, B, ldb, opB == 0 ? k2 * ldb : k2, 0.0, C, h->ldcap,
                h->Tm2 - C, 2, 0, &h->err, 0, 0, &db);
  if (!s) s = add_inplace(h->st, reinterpret_cast<double*>(C), reinterpret_cast<const double*>(h->Tm2),
                          M * h->ldcap * 2, &h->err);
  return s;
}

// Planes are stored plane-major, [plane][trajectory][rows][ldP], so a triple of planes over all
// trajectories sits at one constant stride: three real products C_q = op(A_q) B_q for every
// trajectory are a single batched launch of 3T entries (entry z = q T + t at z * stride).
int prod3(traj_ctx* h, int opA, long long M, long long N, long long K, const double* A, long long lda, long long sA,
          const double* B, long long ldb, long long sB, double* C, long long sC, int flags, cudaStream_t st = nullptr,
          long long n_off = 0) {
  return dgemm(st ? st : h->st, opA, M, N, K, 1.0, A, lda, sA, B, ldb, sB, 0.0, C, h->ldP, sC, 3LL * h->T, flags,
               &h->err, 0, n_off);
}

// The structured pass 1's solve with its products on the INT8 modular path (structchol.h
// struct_chol_apply_oz) on this handle's residue scratch
int struct_chol_apply_oz(traj_ctx* h, const StructChol& s, const cplx* src, cplx* dst, const cudaEvent_t* ev = nullptr) {
  OzWork w;
  w.s = h->oz_s;
  w.RU = h->RU;
  w.RX = h->RX;
  w.RC = h->RC;
  w.RC_bytes = h->RC_bytes;
  w.eU = h->eU;
  w.eU2 = h->eU2;
  w.eX = h->eX;
  w.sEU = h->L;
  w.sEX = h->N;
  w.part = h->oz_part;
  const int r = struct_chol_apply_oz(h->st, s, w, h->L, src, dst, h->ldN, h->sU, h->Tm, h->ldcap,
                                     (long long)h->L * h->ldcap, h->lr_kdev, ev, &h->err);
  return r ? fail(h, r, h->err) : 0;
}

// CholeskyQR pass 1 after a projective step on the structure of its Gram, G = I - V^dag V
// (structchol.h): V = the k0 zeroed rows in US (capacity kc, zero past k0), M in Dw, A in Tm.
int structured_pass1(traj_ctx* h, const cplx* src, cplx* dst, int kc) {
  StructChol s;
  s.b = h->sb;
  s.N = h->N;
  s.kc = kc;
  s.T = h->T;
  s.M = h->Dw;
  s.ldM = h->ldcap;
  s.sM = h->sD;
  s.Y = h->sY;
  s.sY = (long long)h->cap * h->sb;
  s.C = h->sC;
  s.sC = (long long)h->sb * h->sb;
  s.Xb = h->sX;
  s.sXb = round_up(h->N, h->sb) * h->sb;
  s.W = h->sW;
  s.Z = h->sZ;
  s.ldWZ = h->ldN;
  s.sWZ = h->sUS;
  s.chol_scratch = h->s_chol_scratch;
  const bool oz_apply = h->oz_cqr && kc >= h->oz_struct_min;
  if (h->sSb && !oz_apply) {
    // every block at once (structchol.h): the batched factor, then the batched solve on this stream
    s.Sb = h->sSb;
    s.XMb = h->sXMb;
    s.ldS = h->ldcap;
    s.sS = h->sbS;
    s.Qb = h->sQb;
    s.Cb = h->sCb;
    s.bscratch = h->s_bscratch;
    s.bfail = h->s_bfail;
    s.Eb = h->sEb;
    s.ldE = h->ldcap;
    s.sE = h->sEs;
    {
      Phase pf(&h->prof, h->st, TRAJ_PH_STRUCT_FACTOR);
      TRY(struct_chol_factor_batched(h->st, s, h->US, h->ldN, h->sUS, h->lr_kdev, h->failed_dev, &h->err));
    }
    return struct_chol_apply(h->st, s, h->L, src, dst, h->ldN, h->sU, h->Tm, h->ldcap, (long long)h->L * h->ldcap,
                             h->lr_kdev, &h->err)
               ? fail(h, TRAJ_ECUDA, h->err)
               : 0;
  }
  if (oz_apply && h->chol_overlap && h->st_hi && !h->struct_serial) {
    // the factor chain on the high-priority stream; the modular solve waits per block
    const int nblk = (int)ceil_div(h->N, h->sb);
    while ((int)h->sc_ev.size() < nblk) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->sc_ev.push_back(e);
    }
    CK(cudaEventRecord(h->ev_fork, h->st));
    CK(cudaStreamWaitEvent(h->st_hi, h->ev_fork, 0));
    {
      Phase pf(&h->prof, h->st_hi, TRAJ_PH_STRUCT_FACTOR);
      TRY(struct_chol_factor_events(h->st_hi, s, h->US, h->ldN, h->sUS, h->lr_kdev, h->failed_dev, h->sc_ev.data(),
                                    &h->err));
    }
    return struct_chol_apply_oz(h, s, src, dst, h->sc_ev.data());
  }
  if (!oz_apply && h->chol_overlap && h->st_hi && !h->struct_serial) {
    // the factor chain on the high-priority stream, each solve block after its factor block
    const int nblk = (int)ceil_div(h->N, h->sb);
    while ((int)h->sc_ev.size() < nblk) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->sc_ev.push_back(e);
    }
    CK(cudaEventRecord(h->ev_fork, h->st));
    CK(cudaStreamWaitEvent(h->st_hi, h->ev_fork, 0));
    return struct_chol_pipelined(h->st, h->st_hi, h->sc_ev.data(), (int)h->sc_ev.size(), s, h->US, h->ldN, h->sUS,
                                 h->lr_kdev, h->failed_dev, h->L, src, dst, h->ldN, h->sU, h->Tm, h->ldcap,
                                 (long long)h->L * h->ldcap, &h->err)
               ? fail(h, TRAJ_ECUDA, h->err)
               : 0;
  }
  {
    Phase pf(&h->prof, h->st, TRAJ_PH_STRUCT_FACTOR);
    TRY(struct_chol_factor(h->st, s, h->US, h->ldN, h->sUS, h->lr_kdev, h->failed_dev, &h->err));
  }
  if (oz_apply) return struct_chol_apply_oz(h, s, src, dst);
  return struct_chol_apply(h->st, s, h->L, src, dst, h->ldN, h->sU, h->Tm, h->ldcap, (long long)h->L * h->ldcap,
                           h->lr_kdev, &h->err);
}

int cqr2(traj_ctx* h, cplx* U, cplx* tmp) {
  cplx* src = U;
  cplx* dst = tmp;
  const cplx* planes_of = nullptr;   // the state whose planes Up holds (set by a planar Gram)
  const int lr = h->lr_k0;
  h->lr_k0 = -1;
  if (lr == 0 && h->lowrank_orth) {
    // NEXT-1 low-rank mode: U is orthonormal up to the rounding drift the low-rank updates
    // accumulate; certify that with the probe (probe.cu) and refine with one measured
    // CholeskyQR pass only above the tolerance (TRAJ_LOWRANK_TOL=0: every step)
    if (!h->lowrank_refine) return 0;
    if (h->lowrank_tol > 0) {
      Phase p(&h->prof, h->st, TRAJ_PH_GRAM);
      TRY(probe_orthonormality(h->st, U, h->ldN, h->sU, h->L, h->N, h->T, h->step, h->cfg.traj_base, h->cfg.seed,
                               h->PX, h->PY, h->Ppart, h->pest, &h->err));
      CK(cudaMemcpyAsync(h->h_dev, h->pest, h->T * 8, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      ++h->lowrank_probes;
      bool need = false;
      for (int t = 0; t < h->T; ++t)
        if (h->h_dev[t] > h->lowrank_tol) need = true;   // NaN (failed trajectory) does not force it
      if (!need) return 0;
      ++h->lowrank_refinements;
    }
  }
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 0 && lr == 0) continue;     // no row zeroed: U is orthonormal, pass 1 has R = I
    if (pass == 0 && lr > 0 && h->struct_chol && h->lr_kdev && 2LL * lr <= h->N) {
      // pass 1 on the structure of G = I - V^dag V (k0 <= lr << N): no dense Gram / factorisation / TRMM
      Phase p(&h->prof, h->st, TRAJ_PH_CHOL);
      TRY(structured_pass1(h, src, dst, lr));
      std::swap(src, dst);
      continue;
    }
    {
      Phase p(&h->prof, h->st, TRAJ_PH_GRAM);
      if (pass == 0 && lr > 0) {
        // G = U'^dag U' = I - V^dag V (upper tiles): 4 N^2 k0 instead of 4 L N^2 flops
        // (lr = the rows' capacity; their count k0 is read on the device -- rows past it are zero)
        DevBounds db;
        db.k = h->lr_kdev;
        TRY(set_identity(h->st, h->G, h->ldN, h->sG, h->N, h->T, &h->err));
        TRY(zgemm(h->st, 1, 0, h->N, h->N, lr, -1.0, 0.0, h->US, h->ldN, h->sUS, h->US, h->ldN, h->sUS, 1.0, h->G,
                  h->ldN, h->sG, h->T, TRAJ_C_UPPER_F, &h->err, 0, 0, &db));
      } else if (h->oz_cqr) {
        // G = U^dag U on the INT8 tensor cores: U's column residues (re, im, re + im, re - im) once,
        // P1 = Ur^T Ur, P2' = Ui^T Ui, P3 = (Ur - Ui)^T (Ur + Ui); Re = P1 + P2', Im = P3 - P1 + P2'
        TRY(oz_split_cols(h->st, src, h->ldN, h->sU, h->L, h->N, h->T, 4, h->oz_s, h->RU, h->eU, h->L, h->oz_part,
                          &h->err));
        OzProduct p;
        p.M = h->N;
        p.N = h->N;
        p.K = h->L;
        p.T = h->T;
        p.s = h->oz_s;
        p.RA = h->RU;
        p.a_traj = 1;
        p.a_planes = 4;
        p.pa[2] = 3;
        p.eA = h->eU;
        p.sEA = h->L;
        p.RB = h->RU;
        p.b_planes = 4;
        p.eB = h->eU;
        p.sEB = h->L;
        p.RC = h->RC;
        p.C = h->G;
        p.ldc = h->ldN;
        p.sC = h->sG;
        p.flags = OZ_UPPER | OZ_NEG_P2;
        {
          Phase pm(&h->prof, h->st, TRAJ_PH_GRAM_MMA);
          TRY(oz_product_mma(h->st, p, &h->err));
        }
        TRY(oz_product_combine(h->st, p, &h->err));
      } else if (h->planar_cqr) {
        // G = U^dag U = (P1 + Q2) + i (P3 - P1 + Q2): P1 = Ur^T Ur, Q2 = Ui^T Ui, P3 = (Ur - Ui)^T (Ur + Ui),
        // A triple = planes 0..2, B triple = planes 3..5
        const long long tU = h->L * h->ldP, pU = h->T * tU;
        TRY(split6_planes(h->st, src, h->ldN, h->sU, h->L, h->N, h->T, h->Up, h->ldP, pU, tU, &h->err));
        TRY(prod3(h, 1, h->N, h->N, h->L, h->Up, h->ldP, tU, h->Up + 3 * pU, h->ldP, tU, h->Pp, tU, DG_C_UPPER));
        TRY(combine_gram(h->st, h->Pp, h->ldP, pU, tU, h->N, h->T, h->G, h->ldN, h->sG, &h->err));
        planes_of = src;
      } else {
        TRY(zgemm(h->st, 1, 0, h->N, h->N, h->L, 1.0, 0.0, src, h->ldN, h->sU, src, h->ldN, h->sU, 0.0, h->G,
                  h->ldN, h->sG, h->T, TRAJ_C_UPPER_F, &h->err));
      }
    }
    {
      Phase p(&h->prof, h->st, TRAJ_PH_CHOL);
      const bool full = pass == 0 || h->full_cqr2;
      if (!full) {
        // second pass: G2 = I + E; the first-order factor unless N max|E|^2 >= 1e-18 for some
        // trajectory -- decided on the device (no host round trip): the first-order X is written,
        // then the full factorisation, gated on that decision, overwrites it when needed
        const double thr = 1e-9 / sqrt((double)h->N);
        TRY(gram_deviation(h->st, h->G, h->ldN, h->sG, h->N, h->T, h->gdev, &h->err));
        TRY(first_order_inverse(h->st, h->G, h->ldN, h->sG, h->X, h->ldN, h->sG, h->N, h->T, &h->err));
        if (h->fbg_state == 0) {   // built once: the fallback factorisation as a conditional graph node
          const char* fg = getenv("TRAJ_FALLBACK_GRAPH");
          std::string e2;
          h->fbg_state = (fg && fg[0] == '0') || h->fbg.build(h->N, h->G, h->ldN, h->sG, h->X, h->ldN, h->sG, h->T,
                                                               h->chol_scratch, h->failed_dev, h->gdev, thr,
                                                               h->fb_dev, &e2, h->oz_cqr ? &h->coz : nullptr) ? -1 : 1;
        }
        if (h->fbg_state == 1) {
          // the modular TRMM below keys its full-precision product on the same decision (gate)
          if (h->oz_cqr) TRY(cqr2_decide(h->st, h->gdev, h->T, thr, h->gate, nullptr, &h->err));
          TRY(h->fbg.launch(h->st, &h->err));
        } else {   // the same decision, every kernel of the factorisation gated on it
          TRY(cqr2_decide(h->st, h->gdev, h->T, thr, h->gate, h->fb_dev, &h->err));
          TRY(chol_inverse(h->st, h->N, h->G, h->ldN, h->sG, h->X, h->ldN, h->sG, h->T, h->chol_scratch,
                           h->failed_dev, &h->err, nullptr, nullptr, h->gate, h->oz_cqr ? &h->coz : nullptr));
        }
      }
      if (full && h->chol_overlap && h->st_hi && h->N > 64 && !h->oz_cqr) {
        // fork: factorise on st_hi; as each left-edge block X[0:h, 0:h] is queued, st_lo runs the
        // TRMM of the columns it completes
        CK(cudaEventRecord(h->ev_fork, h->st));
        CK(cudaStreamWaitEvent(h->st_hi, h->ev_fork, 0));
        struct HookUser {
          traj_ctx* h;
          const cplx* src;
          cplx* dst;
          long long hs;
          int status;
        } hu{h, src, dst, 0, 0};
        const bool pl = h->planar_cqr;
        const long long tU = h->L * h->ldP, pU = h->T * tU, tX = (long long)h->N * h->ldP, pX = h->T * tX;
        if (pl) {   // U's (re, im, re + im) planes for the planar pieces, on the low-priority stream
          CK(cudaStreamWaitEvent(h->st_lo, h->ev_fork, 0));
          TRY(split_planes(h->st_lo, src, h->ldN, h->sU, h->L, h->N, h->T, h->Up + 3 * pU, h->ldP, pU, tU, &h->err));
          CK(cudaEventRecord(h->ev_split, h->st_lo));
        }
        CholHook hook;
        hook.user = &hu;
        // each left-edge block adds the column piece [previous h, h): dst[:, a:b] = src[:, 0:b] X[0:b, a:b]
        hook.left_ready = [](void* u, long long hs) {
          HookUser* q = reinterpret_cast<HookUser*>(u);
          traj_ctx* hh = q->h;
          if (q->status || hs <= q->hs) return;
          const long long a = q->hs;
          q->hs = hs;
          if (cudaEventRecord(hh->ev_left, hh->st_hi) != cudaSuccess ||
              cudaStreamWaitEvent(hh->st_lo, hh->ev_left, 0) != cudaSuccess) {
            q->status = TRAJ_ECUDA;
            return;
          }
          if (hh->planar_cqr) {
            // planes of X[0:hs, a:hs], then the three real products into the same columns of Pp
            const long long tU = hh->L * hh->ldP, pU = hh->T * tU, tX = (long long)hh->N * hh->ldP, pX = hh->T * tX;
            q->status = split_planes(hh->st_lo, hh->X + a, hh->ldN, hh->sG, (int)hs, (int)(hs - a), hh->T, hh->Xp + a,
                                     hh->ldP, pX, tX, &hh->err);
            if (!q->status)
              q->status = prod3(hh, 0, hh->L, hs - a, hs, hh->Up + 3 * pU, hh->ldP, tU, hh->Xp + a, hh->ldP, tX,
                                hh->Pp + a, tU, DG_TRI_B_UPPER, hh->st_lo, a);
          } else {
            q->status = zgemm(hh->st_lo, 0, 0, hh->L, hs - a, hs, 1.0, 0.0, q->src, hh->ldN, hh->sU, hh->X + a, hh->ldN,
                              hh->sG, 0.0, q->dst + a, hh->ldN, hh->sU, hh->T, TRAJ_TRI_B_UPPER_F, &hh->err, 0, a);
          }
          if (!q->status && cudaEventRecord(hh->ev_lo_done, hh->st_lo) != cudaSuccess) q->status = TRAJ_ECUDA;
        };
        TRY(chol_inverse(h->st_hi, h->N, h->G, h->ldN, h->sG, h->X, h->ldN, h->sG, h->T, h->chol_scratch,
                         h->failed_dev, &h->err, nullptr, &hook));
        if (hu.status) return fail(h, hu.status, h->err.empty() ? "chol overlap: left TRMM" : h->err);
        if (hu.hs <= 0) return fail(h, TRAJ_ECUDA, "chol overlap: the left block was not reported");
        // dst[:, hs:N] = src X[:, hs:N] (triangle offset hs) on st_hi, then join both into st
        if (pl) {
          CK(cudaStreamWaitEvent(h->st_hi, h->ev_split, 0));   // U's planes (split on st_lo) are ready
          TRY(split_planes(h->st_hi, h->X + hu.hs, h->ldN, h->sG, h->N, (int)(h->N - hu.hs), h->T, h->Xp + hu.hs,
                           h->ldP, pX, tX, &h->err));
          TRY(prod3(h, 0, h->L, h->N - hu.hs, h->N, h->Up + 3 * pU, h->ldP, tU, h->Xp + hu.hs, h->ldP, tX,
                    h->Pp + hu.hs, tU, DG_TRI_B_UPPER, h->st_hi, hu.hs));
        } else {
          TRY(zgemm(h->st_hi, 0, 0, h->L, h->N - hu.hs, h->N, 1.0, 0.0, src, h->ldN, h->sU, h->X + hu.hs, h->ldN, h->sG,
                    0.0, dst + hu.hs, h->ldN, h->sU, h->T, TRAJ_TRI_B_UPPER_F, &h->err, 0, hu.hs));
        }
        CK(cudaEventRecord(h->ev_hi_done, h->st_hi));
        CK(cudaStreamWaitEvent(h->st, h->ev_hi_done, 0));
        CK(cudaStreamWaitEvent(h->st, h->ev_lo_done, 0));
        if (pl) TRY(combine_planes(h->st, h->Pp, h->ldP, pU, tU, h->L, h->N, h->T, dst, h->ldN, h->sU, &h->err));
        std::swap(src, dst);
        continue;   // this pass's TRMM is done (its time is inside the Cholesky phase)
      }
      if (full) {
        TRY(chol_inverse(h->st, h->N, h->G, h->ldN, h->sG, h->X, h->ldN, h->sG, h->T, h->chol_scratch,
                         h->failed_dev, &h->err, nullptr, nullptr, nullptr, h->oz_cqr ? &h->coz : nullptr));
      }
    }
    {
      Phase p(&h->prof, h->st, TRAJ_PH_TRMM);
      if (h->oz_cqr && pass == 1 && !h->full_cqr2 && h->oz_s_corr > 0) {
        // second pass, first-order factor X = I + D (|D| <= ~1e-9 / sqrt(N) by the device check):
        // dst = src + src D needs only oz_s_corr moduli (D's columns carry their own exponents, so
        // the correction is resolved to 2^-beta of |D|, far below the rounding of src); when the
        // device decided on the full factorisation (gate), the full-precision src X overwrites it
        // Tiers, decided on the device: src D at s moduli is resolved to 2^-beta (nu_a |b|_1 + nu_b |a|_1)
        // <= 2^(1.5 - beta) N |D col| of a typical entry of src (2 sqrt(N) from the N-term sums, sqrt(2 N)
        // from the (|re| + |im|) row norm against an entry), below 2^-54 when the largest column norm of D
        // is <= 2^(beta - 55.5) / N: then the low modulus count runs (gate[1]), else the standard count
        // (gate[2]), else the full product (gate[0]); exactly one of the three
        const bool low = h->oz_s_low > 0;
        if (low) {
          double* nu2 = h->oz_part + (size_t)8 * h->T * h->N;   // past the column-norm partials (L >= N + N / 8)
          const double dmax = ldexp(1.0, oz_beta(h->oz_s_low) - 55) / (1.4142135623730951 * (double)h->N);
          TRY(oz_colnorm_accumulate(h->st, h->X, h->ldN, h->sG, h->N, h->N, h->T, h->oz_part, nu2, h->N, 0, &h->err, 1));
          TRY(oz_tier_decide(h->st, nu2, (long long)h->T * h->N, dmax * dmax, h->gate, &h->err));
        }
        for (int tier = low ? 0 : 1; tier < 3; ++tier) {
          const int full = tier == 2;
          const int s = full ? h->oz_s : tier == 1 ? h->oz_s_corr : h->oz_s_low;
          const int32_t* gate = full ? h->gate : low ? h->gate + 1 + tier : nullptr;
          TRY(oz_split_rows(h->st, src, h->ldN, h->sU, h->L, h->N, h->T, 0, s, h->RU, h->eU, h->L, &h->err, gate));
          TRY(oz_split_cols(h->st, h->X, h->ldN, h->sG, h->N, h->N, h->T, 3, s, h->RX, h->eX, h->N, h->oz_part,
                            &h->err, full ? 0 : 1, gate));
          OzProduct p;
          p.M = h->L;
          p.N = h->N;
          p.K = h->N;
          p.T = h->T;
          p.s = s;
          p.RA = h->RU;
          p.a_traj = 1;
          p.eA = h->eU;
          p.sEA = h->L;
          p.RB = h->RX;
          p.eB = h->eX;
          p.sEB = h->N;
          p.RC = h->RC;
          p.C = dst;
          p.ldc = h->ldN;
          p.sC = h->sU;
          p.flags = OZ_TRI_B;
          p.base = full ? nullptr : src;
          p.gate = gate;
          {
            Phase pm(&h->prof, h->st, TRAJ_PH_TRMM_MMA);
            TRY(oz_product_mma(h->st, p, &h->err));
          }
          TRY(oz_product_combine(h->st, p, &h->err));
        }
      } else if (h->oz_cqr) {
        // U X on the INT8 tensor cores: U's row residues, X's column residues (X upper triangular:
        // k-blocks past each output column block skipped)
        TRY(oz_split_rows(h->st, src, h->ldN, h->sU, h->L, h->N, h->T, 0, h->oz_s, h->RU, h->eU, h->L, &h->err));
        TRY(oz_split_cols(h->st, h->X, h->ldN, h->sG, h->N, h->N, h->T, 3, h->oz_s, h->RX, h->eX, h->N, h->oz_part,
                          &h->err));
        OzProduct p;
        p.M = h->L;
        p.N = h->N;
        p.K = h->N;
        p.T = h->T;
        p.s = h->oz_s;
        p.RA = h->RU;
        p.a_traj = 1;
        p.eA = h->eU;
        p.sEA = h->L;
        p.RB = h->RX;
        p.eB = h->eX;
        p.sEB = h->N;
        p.RC = h->RC;
        p.C = dst;
        p.ldc = h->ldN;
        p.sC = h->sU;
        p.flags = OZ_TRI_B;
        {
          Phase pm(&h->prof, h->st, TRAJ_PH_TRMM_MMA);
          TRY(oz_product_mma(h->st, p, &h->err));
        }
        TRY(oz_product_combine(h->st, p, &h->err));
      } else if (h->planar_cqr && planes_of == src) {
        // U X = (P1 - P2) + i (P3 - P1 - P2): P1 = Ur Xr, P2 = Ui Xi, P3 = (Ur + Ui)(Xr + Xi) on the
        // Gram's planes of U and X's planes (X upper triangular: k-blocks past the diagonal skipped)
        const long long tU = h->L * h->ldP, pU = h->T * tU, tX = (long long)h->N * h->ldP, pX = h->T * tX;
        TRY(split_planes(h->st, h->X, h->ldN, h->sG, h->N, h->N, h->T, h->Xp, h->ldP, pX, tX, &h->err));
        TRY(prod3(h, 0, h->L, h->N, h->N, h->Up + 3 * pU, h->ldP, tU, h->Xp, h->ldP, tX, h->Pp, tU, DG_TRI_B_UPPER));
        TRY(combine_planes(h->st, h->Pp, h->ldP, pU, tU, h->L, h->N, h->T, dst, h->ldN, h->sU, &h->err));
      } else {
        TRY(zgemm(h->st, 0, 0, h->L, h->N, h->N, 1.0, 0.0, src, h->ldN, h->sU, h->X, h->ldN, h->sG, 0.0, dst, h->ldN,
                  h->sU, h->T, TRAJ_TRI_B_UPPER_F, &h->err));
      }
    }
    std::swap(src, dst);
  }
  if (lr == 0) {   // one pass ran: the result is in tmp
    CK(cudaMemcpyAsync(U, tmp, (size_t)h->T * h->sU * 16, cudaMemcpyDeviceToDevice, h->st));
  }
  return 0;   // two passes: result back in U
}

// NEXT-1 option: orthonormalise U' (rows S0 of the orthonormal U zeroed; V = those rows, in US)
// at low rank: U' <- U' + (U' V^dag) F V, F = Z^2 (Z + I)^-1, Z = (I - M)^(-1/2), M = V V^dag.
// Z by the coupled Newton-Schulz iteration Y <- Y T, Z <- T Z, T = (3I - Z Y)/2 from Y = I - M,
// Z = I (converges for spec(M) in [0, 1)).  On success CQR2 skips its first pass (lr_k0 = 0).
int lowrank_orthonormalize(traj_ctx* h, cplx* U, int k) {
  const int T = h->T;
  const long long ld = h->ldcap, s2 = (long long)h->cap * h->ldcap;
  // M = V V^dag, Y = I - M, Z = I
  TRY(zgemm(h->st, 0, 1, k, k, h->N, 1.0, 0.0, h->US, h->ldN, h->sUS, h->US, h->ldN, h->sUS, 0.0, h->Mb, ld, s2, T, 0,
            &h->err));
  CK(cudaMemcpyAsync(h->Yb, h->Mb, (size_t)T * s2 * 16, cudaMemcpyDeviceToDevice, h->st));
  TRY(axpby_identity(h->st, h->Yb, ld, s2, k, T, -1.0, 1.0, &h->err));
  CK(cudaMemsetAsync(h->Zb, 0, (size_t)T * s2 * 16, h->st));
  TRY(axpby_identity(h->st, h->Zb, ld, s2, k, T, 1.0, 1.0, &h->err));
  bool converged = false;
  for (int it = 0; it < 100; ++it) {
    // Tb = Z Y; residual max|Z Y - I| decides convergence
    TRY(zgemm(h->st, 0, 0, k, k, k, 1.0, 0.0, h->Zb, ld, s2, h->Yb, ld, s2, 0.0, h->Tb, ld, s2, T, 0, &h->err));
    TRY(gram_deviation(h->st, h->Tb, ld, s2, k, T, h->gdev, &h->err));
    CK(cudaMemcpyAsync(h->h_dev, h->gdev, (size_t)T * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    double worst = 0.0;
    for (int t = 0; t < T; ++t)
      if (!std::isnan(h->h_dev[t])) worst = std::max(worst, h->h_dev[t]);   // a failed trajectory stays NaN
    ++h->lowrank_iters;
    if (worst < 1e-14) {
      converged = true;
      break;
    }
    // T = 1.5 I - 0.5 Z Y;  Y <- Y T,  Z <- T Z
    TRY(axpby_identity(h->st, h->Tb, ld, s2, k, T, -0.5, 1.5, &h->err));
    TRY(zgemm(h->st, 0, 0, k, k, k, 1.0, 0.0, h->Yb, ld, s2, h->Tb, ld, s2, 0.0, h->Pb, ld, s2, T, 0, &h->err));
    TRY(zgemm(h->st, 0, 0, k, k, k, 1.0, 0.0, h->Tb, ld, s2, h->Zb, ld, s2, 0.0, h->Qb, ld, s2, T, 0, &h->err));
    std::swap(h->Yb, h->Pb);
    std::swap(h->Zb, h->Qb);
  }
  if (!converged) {          // keep CholeskyQR2 (its first Gram from the zeroed rows)
    ++h->lowrank_fallbacks;
    return 0;
  }
  // F = Z^2 (Z + I)^-1 with (Z + I)^-1 = X X^dag, R^dag R = Z + I, X = R^-1
  CK(cudaMemcpyAsync(h->Mb, h->Zb, (size_t)T * s2 * 16, cudaMemcpyDeviceToDevice, h->st));
  TRY(axpby_identity(h->st, h->Mb, ld, s2, k, T, 1.0, 1.0, &h->err));
  TRY(chol_inverse(h->st, k, h->Mb, ld, s2, h->Yb, ld, s2, T, h->chol_scratch_small, h->failed_dev, &h->err));
  TRY(zgemm(h->st, 0, 0, k, k, k, 1.0, 0.0, h->Zb, ld, s2, h->Zb, ld, s2, 0.0, h->Tb, ld, s2, T, 0, &h->err));
  TRY(zgemm(h->st, 0, 0, k, k, k, 1.0, 0.0, h->Tb, ld, s2, h->Yb, ld, s2, 0.0, h->Pb, ld, s2, T, TRAJ_TRI_B_UPPER_F,
            &h->err));
  TRY(zgemm(h->st, 0, 1, k, k, k, 1.0, 0.0, h->Pb, ld, s2, h->Yb, ld, s2, 0.0, h->Qb, ld, s2, T, TRAJ_TRI_B_LOWER_F,
            &h->err));
  // FV = F V (k x N);  P = U' V^dag (L x k);  U' += P FV
  TRY(zgemm(h->st, 0, 0, k, h->N, k, 1.0, 0.0, h->Qb, ld, s2, h->US, h->ldN, h->sUS, 0.0, h->FV, h->ldN, h->sUS, T, 0,
            &h->err));
  const long long sT = (long long)h->L * h->ldcap;
  TRY(skinny_gemm(h, 1, h->L, k, h->N, U, h->ldN, h->sU, h->US, h->ldN, h->sUS, h->Tm, sT));
  TRY(zgemm(h->st, 0, 0, h->L, h->N, k, 1.0, 0.0, h->Tm, h->ldcap, sT, h->FV, h->ldN, h->sUS, 1.0, U, h->ldN, h->sU, T,
            0, &h->err));
  h->lr_k0 = 0;              // U is orthonormal: CholeskyQR2's first pass has R = I
  return 0;
}

int projective(traj_ctx* h, cplx* U) {
  Phase p(&h->prof, h->st, TRAJ_PH_PROJECT);
  const int T = h->T, cap = h->cap;
  // click counts on the host from the same counter-based draws the device makes (click_draw):
  // they size the launches, so no count is read back from the device (traj_step stays async)
  host_click_counts(h->L, T, h->step, h->cfg.traj_base, h->cfg.seed, h->gamma.data(), h->cfg.dt, h->hcount.data());
  int maxc = 0;
  for (int t = 0; t < T; ++t) {
    h->last_nS[t] = h->hcount[t];
    h->last_n1[t] = 0;
    if (h->hcount[t] > cap)
      return fail(h, TRAJ_ENUMERIC, "click list overflow: " + std::to_string(h->hcount[t]) + " > capacity " +
                                        std::to_string(cap));
    maxc = std::max(maxc, h->hcount[t]);
  }
  h->k1_dev = false;
  if (maxc == 0) {            // no click: U = K U is orthonormal, pass 1 of CQR2 has R = I
    if (h->lowrank_gram) h->lr_k0 = 0;
    return 0;
  }
  TRY(compact(h->st, h->flags, h->L, T, h->S, cap, h->count, &h->err));
  TRY(gather_rows(h->st, U, h->ldN, h->sU, h->S, cap, h->count, maxc, T, h->US, h->ldN, h->sUS, h->N, &h->err));
  // the rank-k products on the INT8 modular path once the click count makes them large (c5:
  // |S| ~ 3700, k1 ~ 1850); below TRAJ_OZAKI_PROJ_MIN clicks the DMMA kernels are cheaper than the
  // residue splits of U
  const bool ozp = h->oz_cqr && maxc >= h->oz_proj_min && maxc <= h->N;
  // C_SS = U_S U_S^dag (all trajectories padded to maxc rows; rows beyond a trajectory's
  // count are never read by the sampler)
  if (ozp) {
    // one 4-plane row split of U_S serves both sides: C = (P1 + P2') + i (P3 - P1 + P2') with
    // P1 = re re^T, P2' = im im^T, P3 = (re + im)(re - im)^T
    TRY(oz_split_rows(h->st, h->US, h->ldN, h->sUS, maxc, h->N, T, 0, h->oz_s, h->RU, h->eU, h->L, &h->err, nullptr,
                      nullptr, 4));
    OzProduct p;
    p.M = maxc;
    p.N = maxc;
    p.K = h->N;
    p.T = T;
    p.s = h->oz_s;
    p.RA = h->RU;
    p.a_traj = 1;
    p.a_planes = 4;
    p.eA = h->eU;
    p.sEA = h->L;
    p.RB = h->RU;
    p.b_planes = 4;
    p.pb[2] = 3;
    p.eB = h->eU;
    p.sEB = h->L;
    p.RC = h->RC;
    p.C = h->D0;
    p.ldc = h->ldcap;
    p.sC = h->sD;
    p.flags = OZ_NEG_P2;
    TRY(oz_product(h->st, p, &h->err));
  } else {
    TRY(zgemm(h->st, 0, 1, maxc, maxc, h->N, 1.0, 0.0, h->US, h->ldN, h->sUS, h->US, h->ldN, h->sUS, 0.0, h->D0,
              h->ldcap, h->sD, T, 0, &h->err));
  }
  TRY(sample_outcomes(h->st, h->D0, h->Dw, h->ldcap, h->sD, h->S, cap, h->count, maxc, T, h->step,
                      h->cfg.traj_base, h->cfg.seed, h->occ, h->Linv, h->DLinv, h->Ybuf, h->Zbuf, h->ldcap, h->pos1,
                      h->S1, h->S0, h->k1, h->k0, &h->err));
  h->k1_dev = true;
  // The occupied / empty counts k1[t], k0[t] stay on the device.  Every launch below is sized by
  // the click capacity maxc and reads them there (zgemm.h DevBounds: output tiles past k1 exit,
  // reduction k-blocks past k1 / k0 are skipped); the padded rows / columns are zeros (identity
  // block in C_{S1 S1}, zero rows of U_{S1}), so the rank-k update is the exact rank-k1 one.
  int k0max = maxc;
  if (h->lowrank_orth) {      // the NEXT-1 low-rank orthonormaliser sizes its k0 x k0 iteration on the host
    CK(cudaMemcpyAsync(h->h_small, h->k0, T * 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    k0max = 0;
    for (int t = 0; t < T; ++t) k0max = std::max(k0max, h->h_small[t]);
  }
  const long long sX = (long long)cap * h->ldcap, sW = (long long)h->N * h->ldcap, sT = (long long)h->L * h->ldcap;
  {
    TRY(gather_sub_batched(h->st, h->D0, h->ldcap, h->sD, h->pos1, cap, h->k1, maxc, T, h->D11, h->ldcap, sX,
                           &h->err));
    // R^dag R = C_{S1 S1} (identity past k1),  X11 = R^-1
    TRY(chol_inverse(h->st, maxc, h->D11, h->ldcap, sX, h->X11, h->ldcap, sX, T, h->chol_scratch_small,
                     h->failed_dev, &h->err));
    // U_{S1} rows (zero beyond k1[t]) -> US
    TRY(gather_rows(h->st, U, h->ldN, h->sU, h->S1, cap, h->k1, maxc, T, h->US, h->ldN, h->sUS, h->N, &h->err, 0,
                    1));
    DevBounds b1;
    b1.n = h->k1;
    b1.k = h->k1;
    // W = U_{S1}^dag R^-1   (N x k1)
    TRY(zgemm(h->st, 1, 0, h->N, maxc, maxc, 1.0, 0.0, h->US, h->ldN, h->sUS, h->X11, h->ldcap, sX, 0.0, h->W,
              h->ldcap, sW, T, TRAJ_TRI_B_UPPER_F, &h->err, 0, 0, &b1));
    if (ozp) {
      // Tm = U W (columns < k1), residues of U's rows and W's columns (W past k1 taken as zero)
      TRY(oz_split_rows(h->st, U, h->ldN, h->sU, h->L, h->N, T, 0, h->oz_s, h->RU, h->eU, h->L, &h->err));
      TRY(oz_split_cols(h->st, h->W, h->ldcap, sW, h->N, maxc, T, 3, h->oz_s, h->RX, h->eX, h->N, h->oz_part, &h->err,
                        0, nullptr, h->k1));
      OzProduct p;
      p.M = h->L;
      p.N = maxc;
      p.K = h->N;
      p.T = T;
      p.s = h->oz_s;
      p.RA = h->RU;
      p.a_traj = 1;
      p.eA = h->eU;
      p.sEA = h->L;
      p.RB = h->RX;
      p.eB = h->eX;
      p.sEB = h->N;
      p.RC = h->RC;
      p.C = h->Tm;
      p.ldc = h->ldcap;
      p.sC = sT;
      p.ndev = h->k1;
      TRY(oz_product(h->st, p, &h->err));
    } else {
      // Tm = U W - E_{S1}   (L x k1)
      TRY(skinny_gemm(h, 0, h->L, maxc, h->N, U, h->ldN, h->sU, h->W, h->ldcap, sW, h->Tm, sT, h->k1));
    }
    TRY(sub_identity_batched(h->st, h->Tm, h->ldcap, sT, h->S1, cap, h->k1, maxc, T, &h->err));
    if (ozp) {
      // U <- U - Tm W^dag: Tm's rows and W's rows (conjugated) over k < k1
      TRY(oz_split_rows(h->st, h->Tm, h->ldcap, sT, h->L, maxc, T, 0, h->oz_s, h->RU, h->eU, h->L, &h->err, nullptr,
                        h->k1));
      TRY(oz_split_rows(h->st, h->W, h->ldcap, sW, h->N, maxc, T, 1, h->oz_s, h->RX, h->eX, h->N, &h->err, nullptr,
                        h->k1));
      OzProduct p;
      p.M = h->L;
      p.N = h->N;
      p.K = maxc;
      p.T = T;
      p.s = h->oz_s;
      p.RA = h->RU;
      p.a_traj = 1;
      p.eA = h->eU;
      p.sEA = h->L;
      p.RB = h->RX;
      p.eB = h->eX;
      p.sEB = h->N;
      p.RC = h->RC;
      p.C = U;
      p.ldc = h->ldN;
      p.sC = h->sU;
      p.base = U;
      p.flags = OZ_NEGATE;
      p.kdev = h->k1;
      TRY(oz_product(h->st, p, &h->err));
    } else {
      // U <- U - Tm W^dag  (reduction over the k1 columns)
      DevBounds bk;
      bk.k = h->k1;
      TRY(zgemm(h->st, 0, 1, h->L, h->N, maxc, -1.0, 0.0, h->Tm, h->ldcap, sT, h->W, h->ldcap, sW, 1.0, U, h->ldN,
                h->sU, T, 0, &h->err, 0, 0, &bk));
    }
  }
  // U is orthonormal here (K unitary, the rank-k update exact), so after zeroing rows S0 the
  // first CholeskyQR Gram is I - V^dag V with V the k0 zeroed rows: keep V (zero-padded).
  if (h->lowrank_gram && k0max > 0) {
    TRY(gather_rows(h->st, U, h->ldN, h->sU, h->S0, cap, h->k0, k0max, T, h->US, h->ldN, h->sUS, h->N, &h->err, 0, 1));
    h->lr_k0 = k0max;
    h->lr_kdev = h->k0;
  } else if (h->lowrank_gram) {
    h->lr_k0 = 0;
  }
  if (k0max > 0) TRY(zero_rows_batched(h->st, U, h->ldN, h->sU, h->S0, cap, h->k0, k0max, T, h->N, &h->err));
  if (h->lowrank_orth && k0max > 0) {
    int s = lowrank_orthonormalize(h, U, k0max);
    if (s) return s;
  }
  return 0;
}

// ---- NEXT-4: event-driven PM -------------------------------------------------------------
// uniforms of event e of trajectory t: counter (e_lo, e_hi, traj, 1) -> (u_eta, u_site),
// (e_lo, e_hi, traj, 2) -> u_pc (the oracle's philox.event_uniforms)
void event_uniforms_host(traj_ctx* h, int t, long long e, double* u_eta, double* u_site, double* u_pc) {
  const uint32_t k0 = (uint32_t)(h->cfg.seed & 0xffffffffu), k1 = (uint32_t)(h->cfg.seed >> 32);
  const uint32_t tr = (uint32_t)(h->cfg.traj_base + t);
  const u32x4 a = philox4x32_10(u32x4{(uint32_t)(e & 0xffffffff), (uint32_t)(e >> 32), tr, 1u}, k0, k1);
  const u32x4 b = philox4x32_10(u32x4{(uint32_t)(e & 0xffffffff), (uint32_t)(e >> 32), tr, 2u}, k0, k1);
  if (u_eta) *u_eta = u53(a.x, a.y);
  if (u_site) *u_site = u53(a.z, a.w);
  if (u_pc) *u_pc = u53(b.x, b.y);
}

// waiting time before event e: tau = -ln(eta) / (gamma N), eta = 1 - u in (0, 1]  (Q12)
double event_wait(traj_ctx* h, int t, long long e) {
  double u;
  event_uniforms_host(h, t, e, &u, nullptr, nullptr);
  const double rate = h->gamma[t] * h->N;
  return rate > 0 ? -log(1.0 - u) / rate : INFINITY;
}

// taps of K(tau) along a ring of n sites: the band [-W, W] where the Bessel tail is < 1e-18,
// or the whole circulant when the band does not fit
struct AxisTaps {
  int lo = 0, n = 1;
  std::vector<std::complex<double>> c{1.0};
};

AxisTaps axis_taps(int n, double J, double tau) {
  const double x = 2.0 * J * tau;
  std::vector<double> jm;
  for (int m = 0; m < 100000; ++m) {
    const double v = jn(m, x);
    jm.push_back(v);
    if (m > fabs(x) + 4 && fabs(v) < 1e-30) break;
  }
  int W = (int)jm.size() - 1;
  double tail = 0.0;
  while (W > 0 && tail + 2 * fabs(jm[W]) < 1e-18) tail += 2 * fabs(jm[W--]);
  const std::complex<double> ph[4] = {{1, 0}, {0, -1}, {-1, 0}, {0, 1}};
  AxisTaps a;
  a.c.clear();
  if (2 * W + 1 <= n) {
    a.lo = -W;
    a.n = 2 * W + 1;
    for (int d = -W; d <= W; ++d) a.c.push_back(ph[std::abs(d) & 3] * jm[std::abs(d)]);
  } else {
    a.lo = 0;
    a.n = n;
    a.c.assign(n, 0.0);
    const int M = (int)jm.size() - 1;
    for (int m = -M; m <= M; ++m) a.c[((m % n) + n) % n] += ph[std::abs(m) & 3] * jm[std::abs(m)];
  }
  return a;
}

struct EvPass {
  int j;            // measured site, or -1 for propagation only
  double pc;
  long long off;    // taps offset in the staged buffer
  AxisTaps x, y;
  double tau = 0.0;
  long long offc = 0;   // one-pass: taps of tau_prev + tau (the prep stencil)
  AxisTaps cx, cy;
};

int event_window(traj_ctx* h) {
  const double t_end = (h->step + 1) * h->cfg.dt;
  CK(cudaMemsetAsync(h->occ_count, 0, (size_t)h->T * 4, h->st));
  for (int t = 0; t < h->T; ++t) {
    std::vector<EvPass> passes;
    auto taps = [&](double tau, EvPass& p) {
      p.x = axis_taps(h->Lx, h->cfg.J, tau);
      if (h->Ly > 1) p.y = axis_taps(h->Ly, h->cfg.J, tau);
    };
    while (h->ev_tnext[t] < t_end) {
      EvPass p;
      double u_site, u_pc;
      event_uniforms_host(h, t, h->ev_count[t], nullptr, &u_site, &u_pc);
      p.j = std::min((int)(u_site * h->L), h->L - 1);
      p.pc = u_pc;
      taps(h->ev_tnext[t] - h->ev_tcur[t], p);
      passes.push_back(p);
      h->ev_tcur[t] = h->ev_tnext[t];
      h->ev_count[t] += 1;
      h->ev_tnext[t] = h->ev_tcur[t] + event_wait(h, t, h->ev_count[t]);
    }
    // propagate to the window end; an odd number of passes leaves the state in the other buffer
    const double rest = t_end - h->ev_tcur[t];
    h->ev_tcur[t] = t_end;
    const int nend = (passes.size() + 1) % 2 == 1 ? 1 : 2;
    for (int q = 0; q < nend; ++q) {
      EvPass p;
      p.j = -1;
      p.pc = 0;
      taps(rest / nend, p);
      passes.push_back(p);
    }
    h->last_nS[t] = (int64_t)passes.size() - nend;
    // stage the taps
    long long used = 0;
    size_t first = 0;
    cplx* src = h->U[h->cur] + t * h->sU;
    cplx* dst = h->U[1 - h->cur] + t * h->sU;
    auto flush = [&](size_t upto) -> int {
      if (used) CK(cudaMemcpyAsync(h->taps_dev, h->taps_host, (size_t)used * 16, cudaMemcpyHostToDevice, h->st));
      for (size_t q = first; q < upto; ++q) {
        EvPass& p = passes[q];
        const cplx* cx = h->taps_dev + p.off;
        const cplx* cy = cx + p.x.n;
        if (p.j >= 0) {
          TRY(event_prep(h->st, src, h->ldN, h->N, h->Lx, h->Ly, p.j, cx, p.x.lo, p.x.n, cy, p.y.lo, p.y.n, p.pc,
                         h->yhat, h->ev_coef, h->occ_count + t, &h->err));
        }
        TRY(event_update(h->st, src, dst, h->ldN, h->N, h->Lx, h->Ly, cx, p.x.lo, p.x.n, cy, p.y.lo, p.y.n,
                         p.j >= 0 ? h->yhat : nullptr, p.j >= 0 ? h->ev_coef : nullptr, p.j, &h->err));
        std::swap(src, dst);
      }
      CK(cudaStreamSynchronize(h->st));    // the staging buffer is reused
      used = 0;
      first = upto;
      return 0;
    };
    for (size_t q = 0; q < passes.size(); ++q) {
      const long long need = passes[q].x.n + passes[q].y.n;
      if (used + need > EV_TAPCAP) TRY(flush(q));
      passes[q].off = used;
      for (int r = 0; r < passes[q].x.n; ++r) h->taps_host[used++] = passes[q].x.c[r];
      for (int r = 0; r < passes[q].y.n; ++r) h->taps_host[used++] = passes[q].y.c[r];
    }
    TRY(flush(passes.size()));
  }
  return 0;
}

// NEXT-4, one-pass form (pm_events.cu): per event one read and one write of U.  Events come first
// in a window, then one or two propagation-only passes; yhat / coef / g are double-buffered by
// event parity.  The first event of a window is prepared from U and its g = U yhat^dag taken by
// a GEMV; every later event q+1 is prepared before pass q (row j' of K(tau_q + tau_q+1) U plus the
// rank-1 term's scalar), and pass q accumulates its g.
int event_window_onepass(traj_ctx* h) {
  const double t_end = (h->step + 1) * h->cfg.dt;
  CK(cudaMemsetAsync(h->occ_count, 0, (size_t)h->T * 4, h->st));
  const long long N = h->N;
  for (int t = 0; t < h->T; ++t) {
    std::vector<EvPass> passes;
    auto taps = [&](double tau, AxisTaps& x, AxisTaps& y) {
      x = axis_taps(h->Lx, h->cfg.J, tau);
      if (h->Ly > 1) y = axis_taps(h->Ly, h->cfg.J, tau);
    };
    while (h->ev_tnext[t] < t_end) {
      EvPass p;
      double u_site, u_pc;
      event_uniforms_host(h, t, h->ev_count[t], nullptr, &u_site, &u_pc);
      p.j = std::min((int)(u_site * h->L), h->L - 1);
      p.pc = u_pc;
      p.tau = h->ev_tnext[t] - h->ev_tcur[t];
      taps(p.tau, p.x, p.y);
      passes.push_back(p);
      h->ev_tcur[t] = h->ev_tnext[t];
      h->ev_count[t] += 1;
      h->ev_tnext[t] = h->ev_tcur[t] + event_wait(h, t, h->ev_count[t]);
    }
    const double rest = t_end - h->ev_tcur[t];
    h->ev_tcur[t] = t_end;
    const int nend = (passes.size() + 1) % 2 == 1 ? 1 : 2;
    for (int q = 0; q < nend; ++q) {
      EvPass p;
      p.j = -1;
      p.pc = 0;
      p.tau = rest / nend;
      taps(p.tau, p.x, p.y);
      passes.push_back(p);
    }
    h->last_nS[t] = (int64_t)passes.size() - nend;
    for (size_t q = 1; q < passes.size(); ++q)
      if (passes[q].j >= 0) taps(passes[q - 1].tau + passes[q].tau, passes[q].cx, passes[q].cy);
    long long used = 0;
    size_t first = 0;
    int cur = 0;
    cplx* src = h->U[h->cur] + t * h->sU;
    cplx* dst = h->U[1 - h->cur] + t * h->sU;
    cplx* Y[2] = {h->ev_y2, h->ev_y2 + N};
    double* C[2] = {h->ev_c2, h->ev_c2 + 8};
    double2* G[2] = {h->ev_g2, h->ev_g2 + h->L};
    auto flush = [&](size_t upto) -> int {
      if (used) CK(cudaMemcpyAsync(h->taps_dev, h->taps_host, (size_t)used * 16, cudaMemcpyHostToDevice, h->st));
      for (size_t q = first; q < upto; ++q) {
        EvPass& p = passes[q];
        const cplx* cx = h->taps_dev + p.off;
        const cplx* cy = cx + p.x.n;
        const bool ev = p.j >= 0;
        if (ev && q == 0) {
          TRY(ev_prep(h->st, src, h->ldN, h->N, h->Lx, h->Ly, p.j, cx, p.x.lo, p.x.n, cy, p.y.lo, p.y.n, nullptr, 0, 0,
                      nullptr, 0, 0, nullptr, nullptr, nullptr, -1, p.pc, Y[cur], h->ev_part, C[cur], h->occ_count + t,
                      &h->err));
          TRY(ev_gemv(h->st, src, h->ldN, h->N, h->L, Y[cur], C[cur], G[cur], &h->err));
        }
        const bool next_ev = ev && q + 1 < passes.size() && passes[q + 1].j >= 0;
        if (next_ev) {
          EvPass& pn = passes[q + 1];
          const cplx* ncx = h->taps_dev + pn.off;
          const cplx* ncy = ncx + pn.x.n;
          const cplx* ccx = h->taps_dev + pn.offc;
          const cplx* ccy = ccx + pn.cx.n;
          TRY(ev_prep(h->st, src, h->ldN, h->N, h->Lx, h->Ly, pn.j, ccx, pn.cx.lo, pn.cx.n, ccy, pn.cy.lo, pn.cy.n, ncx,
                      pn.x.lo, pn.x.n, ncy, pn.y.lo, pn.y.n, C[cur], G[cur], Y[cur], p.j, pn.pc, Y[1 - cur],
                      h->ev_part, C[1 - cur], h->occ_count + t, &h->err));
        }
        TRY(ev_pass(h->st, src, dst, h->ldN, h->N, h->Lx, h->Ly, cx, reinterpret_cast<const cplx*>(p.x.c.data()),
                    p.x.lo, p.x.n, cy, reinterpret_cast<const cplx*>(p.y.c.data()), p.y.lo, p.y.n,
                    ev ? Y[cur] : nullptr, ev ? C[cur] : nullptr, G[cur], p.j,
                    next_ev ? Y[1 - cur] : nullptr, next_ev ? C[1 - cur] : nullptr, G[1 - cur], h->ev_tmp, h->ev_gx,
                    &h->err));
        std::swap(src, dst);
        if (ev) cur = 1 - cur;
      }
      CK(cudaStreamSynchronize(h->st));    // the staging buffer is reused
      used = 0;
      first = upto;
      return 0;
    };
    // pass q needs its own taps and, when pass q+1 is an event, that pass's own and combined taps
    // in the same staged buffer: both are (re)staged after a flush
    int gen = 0;
    std::vector<int> sgen(passes.size(), -1);
    auto need_of = [&](size_t i) -> long long {
      return passes[i].x.n + passes[i].y.n + passes[i].cx.n + passes[i].cy.n;
    };
    auto stage = [&](size_t i) {
      EvPass& p = passes[i];
      p.off = used;
      for (int r = 0; r < p.x.n; ++r) h->taps_host[used++] = p.x.c[r];
      for (int r = 0; r < p.y.n; ++r) h->taps_host[used++] = p.y.c[r];
      p.offc = used;
      for (int r = 0; r < p.cx.n; ++r) h->taps_host[used++] = p.cx.c[r];
      for (int r = 0; r < p.cy.n; ++r) h->taps_host[used++] = p.cy.c[r];
      sgen[i] = gen;
    };
    for (size_t q = 0; q < passes.size(); ++q) {
      const bool nx = passes[q].j >= 0 && q + 1 < passes.size() && passes[q + 1].j >= 0;
      const long long need = (sgen[q] == gen ? 0 : need_of(q)) + (nx && sgen[q + 1] != gen ? need_of(q + 1) : 0);
      if (used + need > EV_TAPCAP) {
        TRY(flush(q));
        ++gen;
      }
      if (sgen[q] != gen) stage(q);
      if (nx && sgen[q + 1] != gen) stage(q + 1);
    }
    TRY(flush(passes.size()));
  }
  return 0;
}

int one_step(traj_ctx* h) {
  cplx* Uc = h->U[h->cur];
  cplx* Un = h->U[1 - h->cur];
  cplx* Us = Un;      // where the propagated state lands
  if (h->cfg.protocol == TRAJ_PROJECTIVE_EVENTS) {
    {
      Phase p(&h->prof, h->st, TRAJ_PH_PROJECT);
      int s = h->ev_onepass ? event_window_onepass(h) : event_window(h);
      if (s) return s;
    }
    // the per-event updates are exact rank-1 maps of an orthonormal U: with the low-rank
    // orthonormaliser the window's CholeskyQR runs only when the probe sees drift
    if (h->lowrank_orth) h->lr_k0 = 0;
    int s = cqr2(h, Un, Uc);
    if (s) return s;
    h->cur = 1 - h->cur;
    h->step += 1;
    return 0;
  }
  if (h->cfg.protocol == TRAJ_HOMODYNE_RK4) {
    // NEXT-2: <n>_t from U(t), then RK4 (= Taylor-4 of exp(dt M)) on the Eq. (A3) generator
    {
      Phase p(&h->prof, h->st, TRAJ_PH_MONITOR);
      TRY(row_monitor(h->st, Uc, h->ldN, h->sU, h->L, h->N, h->T, 0, h->step, h->cfg.traj_base, h->cfg.seed,
                      h->gamma_dev, h->cfg.dt, h->nbuf, &h->err));
    }
    {
      Phase p(&h->prof, h->st, TRAJ_PH_PROPAGATE);
      TRY(qsd_rk4_propagate(h->st, Uc, h->Wrk, Un, h->ldN, h->sU, h->Lx, h->Ly, h->N, h->T, h->nbuf, h->dbuf,
                            h->step, h->cfg.traj_base, h->cfg.seed, h->gamma_dev, h->cfg.J, h->cfg.dt, &h->err));
    }
    int s = cqr2(h, Un, Uc);
    if (s) return s;
    h->cur = 1 - h->cur;
    h->step += 1;
    return 0;
  }
  {
    Phase p(&h->prof, h->st, TRAJ_PH_PROPAGATE);
    if (h->banded) {
      // 1d: one pass along the ring; 2d: x pass (lines = rows y) then y pass (lines = columns x)
      TRY(banded_pass(h->st, Uc, Un, h->ldN, h->sU, h->N, h->T, h->Lx, h->Ly, h->Lx, 1, h->band_host.data(), h->Wx,
                      &h->err));
      if (h->Ly > 1) {
        TRY(banded_pass(h->st, Un, Uc, h->ldN, h->sU, h->N, h->T, h->Ly, h->Lx, 1, h->Lx, h->band_host.data() + 2 * h->Wx + 1,
                        h->Wy, &h->err));
        Us = Uc;
      }
    } else {
      // U <- K U  (K shared across the batch: stride 0)
      if (h->oz_ku) {
        TRY(oz_split_cols(h->st, Uc, h->ldN, h->sU, h->L, h->N, h->T, 3, h->oz_s, h->RU, h->eU, h->L, h->oz_part,
                          &h->err));
        OzProduct p;
        p.M = h->L;
        p.N = h->N;
        p.K = h->L;
        p.T = h->T;
        p.s = h->oz_s;
        p.RA = h->RK;
        p.a_traj = 0;
        p.eA = h->eK;
        p.RB = h->RU;
        p.eB = h->eU;
        p.sEB = h->L;
        p.RC = h->RC;
        p.C = Un;
        p.ldc = h->ldN;
        p.sC = h->sU;
        {
          Phase pm(&h->prof, h->st, TRAJ_PH_KU_MMA);
          TRY(oz_product_mma(h->st, p, &h->err));
        }
        TRY(oz_product_combine(h->st, p, &h->err));
      } else if (h->strassen) {
        // Strassen per planar product: U's 7^lv operands per plane, 3 7^lv leaf-size real products
        // (one batched launch for one trajectory), recombined into K U in one pass
        const int np = strassen_products(h->slv);
        const long long hh = h->L >> h->slv, nh = h->N >> h->slv, bK = hh * h->ldS, bM = hh * h->ldM;
        TRY(strassen_b(h->st, h->slv, Uc, h->ldN, h->sU, h->L, h->N, h->T, h->Bc, h->ldM, &h->err));
        // one launch: entry z = (plane, operand) * T + trajectory, K's operand z / T shared by the batch
        TRY(dgemm(h->st, 0, hh, nh, hh, 1.0, h->Ks, h->ldS, bK, h->Bc, h->ldM, bM, 0.0, h->Ms, h->ldM, bM,
                  (long long)np * h->T, 0, &h->err, 0, 0, h->T));
        TRY(strassen_c(h->st, h->slv, h->Ms, h->ldM, h->L, h->N, h->T, Un, h->ldN, h->sU, &h->err));
      } else if (h->planar) {
        // three real products on planes, then (P1 - P2) + i (P3 - P1 - P2)
        const long long tU = h->L * h->ldP, pU = h->T * tU, pK = h->L * h->ldK;
        TRY(split_planes(h->st, Uc, h->ldN, h->sU, h->L, h->N, h->T, h->Up + 3 * pU, h->ldP, pU, tU, &h->err));
        if (h->T == 1) {   // one batch-3 launch: A = K's planes, B = U's
          TRY(dgemm(h->st, 0, h->L, h->N, h->L, 1.0, h->Kp, h->ldK, pK, h->Up + 3 * pU, h->ldP, tU, 0.0, h->Pp,
                    h->ldP, tU, 3, 0, &h->err));
        } else {           // K's plane q is shared by the T trajectories of product q
          for (int q = 0; q < 3; ++q)
            TRY(dgemm(h->st, 0, h->L, h->N, h->L, 1.0, h->Kp + q * pK, h->ldK, 0, h->Up + (3 + q) * pU, h->ldP, tU, 0.0,
                      h->Pp + q * pU, h->ldP, tU, h->T, 0, &h->err));
        }
        TRY(combine_planes(h->st, h->Pp, h->ldP, pU, tU, h->L, h->N, h->T, Un, h->ldN, h->sU, &h->err));
      } else {
        TRY(zgemm(h->st, 0, 0, h->L, h->N, h->L, 1.0, 0.0, h->K, h->ldL, 0, Uc, h->ldN, h->sU, 0.0, Un, h->ldN, h->sU,
                h->T, 0, &h->err));
      }
    }
  }
  cplx* Ut = Us == Un ? Uc : Un;
  if (h->cfg.protocol == TRAJ_HOMODYNE) {
    Phase p(&h->prof, h->st, TRAJ_PH_MONITOR);
    TRY(row_monitor(h->st, Us, h->ldN, h->sU, h->L, h->N, h->T, 1, h->step, h->cfg.traj_base, h->cfg.seed,
                    h->gamma_dev, h->cfg.dt, nullptr, &h->err));
  } else {
    {
      Phase p(&h->prof, h->st, TRAJ_PH_MONITOR);
      TRY(click_draw(h->st, h->L, h->T, h->step, h->cfg.traj_base, h->cfg.seed, h->gamma_dev, h->cfg.dt, h->flags,
                     &h->err));
    }
    int s = projective(h, Us);
    if (s) return s;
  }
  int s = cqr2(h, Us, Ut);
  if (s) return s;
  h->cur = Us == h->U[0] ? 0 : 1;
  h->step += 1;
  return 0;
}

bool is_sharded(const traj_config* c) { return c->shard_size != 1 || c->nccl_id != nullptr; }

int check_traj(traj_ctx* h, int64_t t) {
  if (!h) return TRAJ_EINVAL;
  if (t < 0 || t >= h->T) return fail(h, TRAJ_EINVAL, "trajectory index out of range");
  return 0;
}

int entropy_impl(traj_ctx* h, const int64_t* A, int64_t nA, double* S_out) {
  if (nA < 0 || (nA > 0 && !A) || !S_out) return fail(h, TRAJ_EINVAL, "bad region arguments");
  std::vector<int32_t> idx(nA);
  std::vector<char> seen(h->L, 0);
  for (int64_t q = 0; q < nA; ++q) {
    if (A[q] < 0 || A[q] >= h->L) return fail(h, TRAJ_EDOMAIN, "site index outside the lattice");
    if (seen[A[q]]) return fail(h, TRAJ_EDOMAIN, "duplicate site in region");
    seen[A[q]] = 1;
    idx[q] = (int32_t)A[q];
  }
  if (nA == 0) {
    for (int t = 0; t < h->T; ++t) S_out[t] = 0.0;
    return 0;
  }
  if (h->sh) {
    int r = shard_entropy(h->sh, A, nA, S_out, &h->err);
    return r ? fail(h, r, h->err) : 0;
  }
  CK(cudaMemcpyAsync(h->region, idx.data(), nA * 4, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemsetAsync(h->bad_dev, 0, h->T * 4, h->st));
  const int n = (int)std::min<int64_t>(nA, h->N);
  for (int t = 0; t < h->T; ++t) {
    cplx* Ut = h->U[h->cur] + t * h->sU;
    cplx* UA = h->U[1 - h->cur] + t * h->sU;    // scratch: the other state buffer
    cplx* C = h->G + t * h->sG;
    TRY(gather_rows(h->st, Ut, h->ldN, 0, h->region, 0, nullptr, (int)nA, 1, UA, h->ldN, 0, h->N, &h->err));
    if (nA <= h->N)   // C_A = U_A U_A^dag
      TRY(zgemm(h->st, 0, 1, nA, nA, h->N, 1.0, 0.0, UA, h->ldN, 0, UA, h->ldN, 0, 0.0, C, h->ldN, 0, 1, 0, &h->err));
    else              // same non-zero spectrum: U_A^dag U_A (N x N)
      TRY(zgemm(h->st, 1, 0, h->N, h->N, nA, 1.0, 0.0, UA, h->ldN, 0, UA, h->ldN, 0, 0.0, C, h->ldN, 0, 1, 0, &h->err));
    cusolverStatus_t r = cusolverDnZheevd(h->solver, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                          reinterpret_cast<cuDoubleComplex*>(C), (int)h->ldN, h->eig_w,
                                          reinterpret_cast<cuDoubleComplex*>(h->eig_work), h->lwork, h->eig_info);
    if (r != CUSOLVER_STATUS_SUCCESS) return fail(h, TRAJ_ECUDA, "cusolverDnZheevd failed: " + std::to_string(r));
    TRY(entropy_reduce(h->st, h->eig_w, n, h->S_dev + t, h->bad_dev + t, &h->err));
  }
  std::vector<int32_t> bad(h->T), failed(h->T);
  CK(cudaMemcpyAsync(S_out, h->S_dev, h->T * 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaMemcpyAsync(bad.data(), h->bad_dev, h->T * 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaMemcpyAsync(failed.data(), h->failed_dev, h->T * 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  bool newbad = false;
  for (int t = 0; t < h->T; ++t) {
    if (failed[t]) S_out[t] = nan("");
    if (bad[t] && !failed[t]) {
      newbad = true;
      int32_t one = 1;
      CK(cudaMemcpy(h->failed_dev + t, &one, 4, cudaMemcpyHostToDevice));
    }
  }
  if (newbad) return fail(h, TRAJ_ENUMERIC, "spectrum of C_A outside [-1e-8, 1+1e-8]");
  return 0;
}

// Row-major source of the full U of trajectory t (sharded: gathered) and a scratch area
// of `cap` complex elements for blocks of C = U U^dag.
int full_state(traj_ctx* h, int t, const cplx** U, cplx** scratch, long long* cap) {
  if (h->sh) {
    TRY(shard_full_state(h->sh, &h->err));
    *U = h->sh->Ufull;
    *scratch = h->sh->X;
    *cap = (long long)h->N * h->ldN;
  } else {
    *U = h->U[h->cur] + t * h->sU;
    *scratch = h->X;
    *cap = (long long)h->T * h->N * h->ldN;
  }
  return 0;
}

// C(r), Eq. (2): rows of C = U U^dag in blocks of R, binned by distance
int density_correlation_impl(traj_ctx* h, int t, double* C_out) {
  const cplx* U;
  cplx* scr;
  long long cap;
  int s = full_state(h, t, &U, &scr, &cap);
  if (s) return s;
  const long long ldc = round_up(h->L, 8);
  const int R = (int)std::max<long long>(1, std::min<long long>(h->L, cap / ldc));
  CK(cudaMemsetAsync(h->obs_bins, 0, (size_t)h->L * 8, h->st));
  for (int r0 = 0; r0 < h->L; r0 += R) {
    const int rows = std::min(R, h->L - r0);
    TRY(zgemm(h->st, 0, 1, rows, h->L, h->N, 1.0, 0.0, U + (long long)r0 * h->ldN, h->ldN, 0, U, h->ldN, 0, 0.0, scr,
              ldc, 0, 1, 0, &h->err));
    TRY(bin_abs2(h->st, scr, ldc, rows, r0, h->L, h->obs_bins, &h->err));
  }
  std::vector<double> bins(h->L);
  CK(cudaMemcpyAsync(bins.data(), h->obs_bins, (size_t)h->L * 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  C_out[0] = nan("");
  for (int r = 1; r < h->L; ++r) C_out[r] = -bins[r] / (double)(h->L - r);
  return 0;
}

// G_AB, Eq. (5): sum over i in A (rows of C in blocks), j in B (mask) of |C_ij|^2
int particle_covariance_impl(traj_ctx* h, const std::vector<int32_t>& A, const std::vector<int32_t>& maskB,
                             double* G_out) {
  const long long ldc = round_up(h->L, 8);
  CK(cudaMemcpyAsync(h->obs_mask, maskB.data(), (size_t)h->L * 4, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->region, A.data(), A.size() * 4, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemsetAsync(h->obs_out, 0, (size_t)h->T * 8, h->st));
  for (int t = 0; t < h->T; ++t) {
    const cplx* U;
    cplx* scr;
    long long cap;
    int s = full_state(h, t, &U, &scr, &cap);
    if (s) return s;
    // rows of A gathered into the front of the scratch, the C block after them
    const long long R = std::max<long long>(1, std::min<long long>((long long)A.size(), cap / (ldc + h->ldN)));
    cplx* UA = scr;
    cplx* Cb = scr + R * h->ldN;
    for (long long a0 = 0; a0 < (long long)A.size(); a0 += R) {
      const int rows = (int)std::min<long long>(R, (long long)A.size() - a0);
      TRY(gather_rows(h->st, U, h->ldN, 0, h->region + a0, 0, nullptr, rows, 1, UA, h->ldN, 0, h->N, &h->err));
      TRY(zgemm(h->st, 0, 1, rows, h->L, h->N, 1.0, 0.0, UA, h->ldN, 0, U, h->ldN, 0, 0.0, Cb, ldc, 0, 1, 0,
                &h->err));
      TRY(masked_abs2(h->st, Cb, ldc, rows, h->L, h->obs_mask, h->obs_part, h->obs_out + t, &h->err));
    }
  }
  CK(cudaMemcpyAsync(G_out, h->obs_out, (size_t)h->T * 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return 0;
}

}  // namespace

extern "C" {

const char* traj_strerror(int s) {
  switch (s) {
    case TRAJ_OK: return "ok";
    case TRAJ_EINVAL: return "invalid argument";
    case TRAJ_ECONFIG: return "invalid configuration";
    case TRAJ_ENUMERIC: return "numerical failure (trajectory marked failed)";
    case TRAJ_ECUDA: return "CUDA / cuSOLVER error";
    case TRAJ_ENCCL: return "NCCL error";
    case TRAJ_EDOMAIN: return "domain error";
    default: return "unknown status";
  }
}

const char* traj_last_error(traj_handle h) { return h ? h->err.c_str() : g_err.c_str(); }

long long traj_kernel_launches(void) { return g_kernel_launches.load(); }

int traj_workspace_bytes(const traj_config* cfg, size_t* out) {
  traj_ctx* h = nullptr;
  std::string why;
  if (!out) return fail(h, TRAJ_EINVAL, "null out");
  int s = validate(cfg, &why);
  if (s) return fail(h, s, why);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(h, TRAJ_ECUDA, "no CUDA device");
  int lw = 0;
  if ((s = eig_lwork((int)cfg->N, &lw, &why))) return fail(h, s, why);
  if (is_sharded(cfg)) {
    ShardedCtx sh;
    int Wx = 0, Wy = 0;
    const bool bd = banded_widths(cfg, &Wx, &Wy);
    if (bd && !shard_banded_fits(cfg, Wx, Wy, &why)) return fail(h, TRAJ_ECONFIG, why);
    *out = shard_carve(&sh, cfg, nullptr, lw, bd, Wx, Wy);
  } else {
    traj_ctx tmp;
    *out = carve(&tmp, cfg, nullptr, lw);
  }
  return 0;
}

int traj_init(const traj_config* cfg, traj_handle* out) {
  traj_ctx* h = nullptr;
  std::string why;
  if (!out) return fail(h, TRAJ_EINVAL, "null out");
  *out = nullptr;
  int s = validate(cfg, &why);
  if (s) return fail(h, s, why);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(h, TRAJ_ECUDA, "no CUDA device");
  int lw = 0;
  if ((s = eig_lwork((int)cfg->N, &lw, &why))) return fail(h, s, why);
  {
    size_t need;
    if (is_sharded(cfg)) {
      ShardedCtx sh;
      int Wx = 0, Wy = 0;
      const bool bd = banded_widths(cfg, &Wx, &Wy);
      if (bd && !shard_banded_fits(cfg, Wx, Wy, &why)) return fail(h, TRAJ_ECONFIG, why);
      need = shard_carve(&sh, cfg, nullptr, lw, bd, Wx, Wy);
    } else {
      traj_ctx tmp;
      need = carve(&tmp, cfg, nullptr, lw);
    }
    if (!cfg->workspace || cfg->workspace_bytes < need)
      return fail(h, TRAJ_ECONFIG, "workspace missing or smaller than traj_workspace_bytes");
    if (reinterpret_cast<uintptr_t>(cfg->workspace) & 255) return fail(h, TRAJ_ECONFIG, "workspace not 256-B aligned");
  }
  h = new traj_ctx();
  h->cfg = *cfg;
  h->gamma.assign(cfg->gamma, cfg->gamma + cfg->n_traj);
  h->cfg.gamma = h->gamma.data();
  h->st = reinterpret_cast<cudaStream_t>(cfg->stream);
  {
    const char* co = getenv("TRAJ_CHOL_OVERLAP");
    h->chol_overlap = !(co && co[0] == '0');
    int least = 0, greatest = 0;
    if (h->chol_overlap && cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess &&
        cudaStreamCreateWithPriority(&h->st_hi, cudaStreamNonBlocking, greatest) == cudaSuccess &&
        cudaStreamCreateWithPriority(&h->st_lo, cudaStreamNonBlocking, least) == cudaSuccess) {
      for (cudaEvent_t* e : {&h->ev_fork, &h->ev_left, &h->ev_lo_done, &h->ev_hi_done, &h->ev_split})
        if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) h->chol_overlap = false;
    } else {
      h->chol_overlap = false;
    }
  }
  h->lwork = lw;
  if (is_sharded(cfg)) {
    // (row-sharded: chol_inverse's levels stay on DMMA)
    h->sh = new ShardedCtx();
    {
      int Wx = 0, Wy = 0;
      const bool bd = banded_widths(cfg, &Wx, &Wy);
      shard_carve(h->sh, cfg, reinterpret_cast<char*>(cfg->workspace), lw, bd, Wx, Wy);
      h->banded = bd;
      h->Wx = Wx;
      h->Wy = Wy;
    }
    h->obs_bins = h->sh->obs_bins;
    h->obs_part = h->sh->obs_part;
    h->obs_out = h->sh->obs_out;
    h->obs_mask = h->sh->obs_mask;
    h->region = h->sh->region;
    h->L = h->sh->L;
    h->N = h->sh->N;
    h->Lx = h->sh->Lx;
    h->Ly = h->sh->Ly;
    h->T = 1;
    h->ldN = h->sh->ldN;
    h->ldL = h->sh->ldL;
    h->sh->prof = &h->prof;
  } else {
    carve(h, cfg, reinterpret_cast<char*>(cfg->workspace), lw);
    if (h->oz_cqr) {   // chol_inverse's levels of n >= TRAJ_CHOL_OZAKI_MIN (default 4096) on the modular path
      const char* cm = getenv("TRAJ_CHOL_OZAKI_MIN");
      h->coz.s = h->oz_s;
      h->coz.min_n = cm ? atoll(cm) : 4096;
      h->coz.RA = h->RU;
      h->coz.RB = h->RX;
      h->coz.RC = h->RC;
      h->coz.eA = h->eU;
      h->coz.eB = h->eX;
      h->coz.sE = h->N;
      h->coz.part = h->oz_part;
    }
  }
  h->last_nS.assign(h->T, 0);
  h->last_n1.assign(h->T, 0);
  h->hcount.assign(h->T, 0);
  auto bail = [&](int st, const std::string& m) {
    std::string msg = m;
    traj_destroy(h);
    g_err = msg;
    return st;
  };
  if (cudaMallocHost(&h->h_small, std::max(2 * h->T, 16) * 4) != cudaSuccess ||
      cudaMallocHost(&h->h_dev, std::max(h->T, 16) * 8) != cudaSuccess)
    return bail(TRAJ_ECUDA, "cudaMallocHost");
  {
    const char* e = getenv("TRAJ_CQR2_FULL");
    h->full_cqr2 = e && e[0] == '1';
    const char* g = getenv("TRAJ_LOWRANK_GRAM");
    h->lowrank_gram = !(g && g[0] == '0') || cfg->orthonormalizer == TRAJ_ORTH_LOWRANK;
    h->lowrank_orth = cfg->orthonormalizer == TRAJ_ORTH_LOWRANK &&
                      (cfg->protocol == TRAJ_PROJECTIVE || cfg->protocol == TRAJ_PROJECTIVE_EVENTS);
    const char* rf = getenv("TRAJ_LOWRANK_REFINE");
    h->lowrank_refine = !(rf && rf[0] == '0');
    const char* op = getenv("TRAJ_EVENTS_ONEPASS");
    h->ev_onepass = !(op && op[0] == '0');
    const char* tl = getenv("TRAJ_LOWRANK_TOL");
    if (tl) h->lowrank_tol = atof(tl);
    const char* sc = getenv("TRAJ_STRUCT_CHOL");
    h->struct_chol = !(sc && sc[0] == '0');
    const char* sp = getenv("TRAJ_STRUCT_PIPELINE");
    h->struct_serial = sp && sp[0] == '0';
    const char* sm = getenv("TRAJ_SMALL_STEP");
    const bool proj = cfg->protocol == TRAJ_PROJECTIVE;
    h->small = !h->sh && !h->banded && h->K && !(sm && sm[0] == '0') && !h->lowrank_orth &&
               (proj || cfg->protocol == TRAJ_HOMODYNE) && small_step_fits(h->L, h->N, proj);
  }
  if (cusolverDnCreate(&h->solver) != CUSOLVER_STATUS_SUCCESS) return bail(TRAJ_ECUDA, "cusolverDnCreate");
  cusolverDnSetStream(h->solver, h->st);
  // zero the whole workspace: padded columns (ld > N) must read as zeros
  if (cudaMemsetAsync(cfg->workspace, 0, cfg->workspace_bytes, h->st) != cudaSuccess) return bail(TRAJ_ECUDA, "memset");
  if (h->sh) {
    h->sh->solver = h->solver;
    h->sh->full_cqr2 = h->full_cqr2;
    std::string e;
    int s2 = shard_init(h->sh, cfg, &e);
    if (s2) return bail(s2, e);
  }
  // K = K_y (x) K_x from the ring coefficient rows (Ly = 1: K_y = [1])
  std::vector<std::complex<double>> kc = ring_coefficients(h->Lx, cfg->J, cfg->dt);
  if (h->Ly > 1) {
    std::vector<std::complex<double>> ky = ring_coefficients(h->Ly, cfg->J, cfg->dt);
    kc.insert(kc.end(), ky.begin(), ky.end());
  } else {
    kc.push_back(1.0);
  }
  std::vector<int32_t> sites;
  for (int i = 0; i < h->L; ++i)
    if (((i % h->Lx) + (i / h->Lx)) % 2 == 0) sites.push_back(i);
  if ((int)sites.size() != h->N) return bail(TRAJ_ECONFIG, "initial state does not have N particles");
  std::string e;
  std::vector<std::complex<double>> band;
  if (h->banded) {
    auto axis = [&](int n, int W) {
      std::vector<std::complex<double>> c = ring_coefficients(n, cfg->J, cfg->dt);
      for (int d = -W; d <= W; ++d) band.push_back(c[((d % n) + n) % n]);
    };
    axis(h->Lx, h->Wx);
    if (h->Ly > 1) axis(h->Ly, h->Wy);
    else band.push_back(1.0);
  }
  h->band_host.resize(band.size());
  for (size_t i = 0; i < band.size(); ++i) h->band_host[i] = make_double2(band[i].real(), band[i].imag());
  if (h->sh) {
    int s2 = shard_build(h->sh, kc, sites, &e, &band);
    if (s2) return bail(s2, e);
    *out = h;
    return 0;
  }
  if (cudaMemcpyAsync(h->kcoef, kc.data(), kc.size() * 16, cudaMemcpyHostToDevice, h->st) != cudaSuccess ||
      cudaMemcpyAsync(h->sites, sites.data(), sites.size() * 4, cudaMemcpyHostToDevice, h->st) != cudaSuccess ||
      cudaMemcpyAsync(h->gamma_dev, h->gamma.data(), h->T * 8, cudaMemcpyHostToDevice, h->st) != cudaSuccess)
    return bail(TRAJ_ECUDA, "upload");
  if (h->banded) {
    if (cudaMemcpyAsync(h->bcoef, band.data(), band.size() * 16, cudaMemcpyHostToDevice, h->st) != cudaSuccess)
      return bail(TRAJ_ECUDA, "upload band");
  } else if (h->planar) {
    if (build_k_planar(h->st, h->Kp, h->ldK, h->L * h->ldK, h->Lx, h->Ly, h->kcoef, h->kcoef + h->Lx, &e))
      return bail(TRAJ_ECUDA, e);
    if (h->strassen && strassen_k(h->st, h->slv, h->Kp, h->ldK, h->L * h->ldK, h->L, h->Ks, h->ldS, &e))
      return bail(TRAJ_ECUDA, e);
  } else if (h->oz_ku) {   // K in the product scratch, then its residues (once)
    cplx* Kt = reinterpret_cast<cplx*>(h->RC);
    if (build_k(h->st, Kt, h->ldL, h->Lx, h->Ly, h->kcoef, h->kcoef + h->Lx, &e) ||
        oz_split_rows(h->st, Kt, h->ldL, 0, h->L, h->L, 1, 0, h->oz_s, h->RK, h->eK, 0, &e))
      return bail(TRAJ_ECUDA, e);
  } else if (cfg->protocol != TRAJ_HOMODYNE_RK4 && cfg->protocol != TRAJ_PROJECTIVE_EVENTS &&
             build_k(h->st, h->K, h->ldL, h->Lx, h->Ly, h->kcoef, h->kcoef + h->Lx, &e)) {
    return bail(TRAJ_ECUDA, e);
  }
  if (init_state(h->st, h->U[0], h->ldN, h->sU, h->sites, h->N, h->T, &e)) return bail(TRAJ_ECUDA, e);
  if (cfg->protocol == TRAJ_PROJECTIVE_EVENTS) {
    if (cudaMallocHost(&h->taps_host, (size_t)EV_TAPCAP * 16) != cudaSuccess) return bail(TRAJ_ECUDA, "cudaMallocHost");
    h->ev_count.assign(h->T, 0);
    h->ev_tcur.assign(h->T, 0.0);
    h->ev_tnext.assign(h->T, 0.0);
    for (int t = 0; t < h->T; ++t) h->ev_tnext[t] = event_wait(h, t, 0);
  }
  if (cudaStreamSynchronize(h->st) != cudaSuccess) return bail(TRAJ_ECUDA, "init sync");
  *out = h;
  return 0;
}

int traj_step(traj_handle h, int64_t n_steps) {
  if (!h) return TRAJ_EINVAL;
  if (n_steps < 0) return fail(h, TRAJ_EINVAL, "n_steps < 0");
  if (h->small && n_steps > 0) {
    Phase p(&h->prof, h->st, TRAJ_PH_FUSED);
    SmallStepArgs a;
    a.U = h->U[h->cur];
    a.ldU = h->ldN;
    a.sU = h->sU;
    a.K = h->K;
    a.ldK = h->ldL;
    a.L = h->L;
    a.N = h->N;
    a.T = h->T;
    a.projective = h->cfg.protocol == TRAJ_PROJECTIVE;
    a.step0 = h->step;
    a.n_steps = n_steps;
    a.traj_base = h->cfg.traj_base;
    a.seed = h->cfg.seed;
    a.gamma = h->gamma_dev;
    a.dt = h->cfg.dt;
    a.failed = h->failed_dev;
    a.last = h->small_last;
    a.Dg = h->D0;
    a.ldDg = h->ldcap;
    a.sDg = h->sD;
    a.cap = h->cap;
    a.full_cqr2 = h->full_cqr2 ? 1 : 0;
    a.skip_orthonormal_pass = h->lowrank_gram ? 1 : 0;
    a.fallbacks = h->small_fallbacks;
    int r = small_steps(h->st, a, &h->err);
    if (r) return fail(h, r, h->err);
    h->step += n_steps;
    h->small_last_dev = a.projective != 0;
    return 0;
  }
  for (int64_t s = 0; s < n_steps; ++s) {
    int r = h->sh ? shard_step(h->sh, &h->step, &h->err) : one_step(h);
    if (r) return fail(h, r, h->err);
  }
  return 0;
}

int traj_orthonormalize(traj_handle h) {
  if (!h) return TRAJ_EINVAL;
  if (h->sh) {
    int r = shard_orthonormalize(h->sh, &h->err);
    return r ? fail(h, r, h->err) : 0;
  }
  return cqr2(h, h->U[h->cur], h->U[1 - h->cur]);
}

int traj_entropy(traj_handle h, const int64_t* A, int64_t nA, double* S_out) {
  if (!h) return TRAJ_EINVAL;
  return entropy_impl(h, A, nA, S_out);
}

int traj_mutual_info(traj_handle h, const int64_t* A, int64_t nA, const int64_t* B, int64_t nB, double* I_out) {
  if (!h) return TRAJ_EINVAL;
  if (!I_out || nA < 0 || nB < 0 || (nA && !A) || (nB && !B)) return fail(h, TRAJ_EINVAL, "bad region arguments");
  std::vector<char> inA(h->L, 0);
  for (int64_t q = 0; q < nA; ++q)
    if (A[q] >= 0 && A[q] < h->L) inA[A[q]] = 1;
  for (int64_t q = 0; q < nB; ++q)
    if (B[q] >= 0 && B[q] < h->L && inA[B[q]]) return fail(h, TRAJ_EDOMAIN, "regions overlap");
  std::vector<int64_t> AB(A, A + nA);
  AB.insert(AB.end(), B, B + nB);
  std::vector<double> sa(h->T), sb(h->T), sab(h->T);
  int s;
  if ((s = entropy_impl(h, A, nA, sa.data()))) return s;
  if ((s = entropy_impl(h, B, nB, sb.data()))) return s;
  if ((s = entropy_impl(h, AB.data(), (int64_t)AB.size(), sab.data()))) return s;
  for (int t = 0; t < h->T; ++t) I_out[t] = sa[t] + sb[t] - sab[t];
  return 0;
}

int traj_density_correlation(traj_handle h, int64_t traj, double* C_out) {
  int s = check_traj(h, traj);
  if (s) return s;
  if (!C_out) return fail(h, TRAJ_EINVAL, "null C_out");
  if (h->cfg.dim != 1) return fail(h, TRAJ_EDOMAIN, "C(r) binned by |i - j| is defined for the 1d chain");
  return density_correlation_impl(h, (int)traj, C_out);
}

int traj_particle_covariance(traj_handle h, const int64_t* A, int64_t nA, const int64_t* B, int64_t nB,
                             double* G_out) {
  if (!h) return TRAJ_EINVAL;
  if (!G_out || nA < 0 || nB < 0 || (nA && !A) || (nB && !B)) return fail(h, TRAJ_EINVAL, "bad region arguments");
  std::vector<int32_t> a(nA), mask(h->L, 0);
  for (int64_t q = 0; q < nB; ++q) {
    if (B[q] < 0 || B[q] >= h->L) return fail(h, TRAJ_EDOMAIN, "site index outside the lattice");
    if (mask[B[q]]) return fail(h, TRAJ_EDOMAIN, "duplicate site in region");
    mask[B[q]] = 1;
  }
  std::vector<char> seen(h->L, 0);
  for (int64_t q = 0; q < nA; ++q) {
    if (A[q] < 0 || A[q] >= h->L) return fail(h, TRAJ_EDOMAIN, "site index outside the lattice");
    if (mask[A[q]]) return fail(h, TRAJ_EDOMAIN, "regions overlap");
    if (seen[A[q]]) return fail(h, TRAJ_EDOMAIN, "duplicate site in region");
    seen[A[q]] = 1;
    a[q] = (int32_t)A[q];
  }
  if (nA == 0 || nB == 0) {
    for (int t = 0; t < h->T; ++t) G_out[t] = 0.0;
    return 0;
  }
  return particle_covariance_impl(h, a, mask, G_out);
}

int traj_occupations(traj_handle h, double* n_out) {
  if (!h) return TRAJ_EINVAL;
  if (!n_out) return fail(h, TRAJ_EINVAL, "null n_out");
  if (h->sh) TRY(shard_occupations(h->sh, n_out, h->step, &h->err));
  else TRY(row_monitor(h->st, h->U[h->cur], h->ldN, h->sU, h->L, h->N, h->T, 0, h->step, h->cfg.traj_base, h->cfg.seed,
                  h->gamma_dev, h->cfg.dt, n_out, &h->err));
  return 0;
}

int traj_correlation_rows(traj_handle h, int64_t traj, int64_t row0, int64_t nrows, void* C_out) {
  int s = check_traj(h, traj);
  if (s) return s;
  if (row0 < 0 || nrows < 0 || row0 + nrows > h->L || !C_out) return fail(h, TRAJ_EINVAL, "bad row range");
  if (nrows == 0) return 0;
  if (h->sh) {
    TRY(shard_correlation_rows(h->sh, row0, nrows, C_out, &h->err));
    return 0;
  }
  cplx* Ut = h->U[h->cur] + traj * h->sU;
  TRY(zgemm(h->st, 0, 1, nrows, h->L, h->N, 1.0, 0.0, Ut + row0 * h->ldN, h->ldN, 0, Ut, h->ldN, 0, 0.0,
            reinterpret_cast<cplx*>(C_out), h->L, 0, 1, 0, &h->err));
  return 0;
}

int traj_get_state(traj_handle h, int64_t traj, void* U_out) {
  int s = check_traj(h, traj);
  if (s) return s;
  if (!U_out) return fail(h, TRAJ_EINVAL, "null U_out");
  if (h->sh) {
    TRY(shard_get_state(h->sh, U_out, &h->err));
    return 0;
  }
  CK(cudaMemcpy2DAsync(U_out, (size_t)h->N * 16, h->U[h->cur] + traj * h->sU, (size_t)h->ldN * 16, (size_t)h->N * 16,
                       h->L, cudaMemcpyDefault, h->st));
  CK(cudaStreamSynchronize(h->st));
  return 0;
}

int traj_set_state(traj_handle h, int64_t traj, const void* U_in) {
  int s = check_traj(h, traj);
  if (s) return s;
  if (!U_in) return fail(h, TRAJ_EINVAL, "null U_in");
  if (h->sh) {
    TRY(shard_set_state(h->sh, U_in, &h->err));
    return 0;
  }
  CK(cudaMemcpy2DAsync(h->U[h->cur] + traj * h->sU, (size_t)h->ldN * 16, U_in, (size_t)h->N * 16, (size_t)h->N * 16,
                       h->L, cudaMemcpyDefault, h->st));
  CK(cudaStreamSynchronize(h->st));
  return 0;
}

int traj_get_step(traj_handle h, int64_t* step) {
  if (!h || !step) return TRAJ_EINVAL;
  *step = h->step;
  return 0;
}

int traj_set_step(traj_handle h, int64_t step) {
  if (!h) return TRAJ_EINVAL;
  if (step < 0 || step >= (1ll << 32)) return fail(h, TRAJ_EINVAL, "step out of range");
  h->step = step;
  if (h->cfg.protocol == TRAJ_PROJECTIVE_EVENTS) {
    // the event clock at time step * dt, as event_window leaves it: ev_count = events before that
    // time, ev_tnext = the next event's time (the same accumulation of the Philox waiting times),
    // ev_tcur = the window end; host Philox only
    const double t_end = step * h->cfg.dt;
    for (int t = 0; t < h->T; ++t) {
      long long e = 0;
      double tn = event_wait(h, t, 0);
      while (tn < t_end) {
        ++e;
        tn = tn + event_wait(h, t, e);
      }
      h->ev_count[t] = e;
      h->ev_tnext[t] = tn;
      h->ev_tcur[t] = t_end;
    }
  }
  return 0;
}

int traj_failed(traj_handle h, int64_t traj, int32_t* flag) {
  int s = check_traj(h, traj);
  if (s) return s;
  if (!flag) return fail(h, TRAJ_EINVAL, "null flag");
  if (h->sh) {
    TRY(shard_failed(h->sh, flag, &h->err));
    return 0;
  }
  CK(cudaMemcpyAsync(h->h_small, h->failed_dev + traj, 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  *flag = h->h_small[0];
  return 0;
}

int traj_last_clicks(traj_handle h, int64_t traj, int64_t* n_clicks, int64_t* n_occupied) {
  int s = check_traj(h, traj);
  if (s) return s;
  if (h->sh) {
    if (h->sh->k1_dev && n_occupied) {   // the occupied count of the last step is on the device
      CK(cudaMemcpyAsync(h->h_small, h->sh->k1, 4, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      h->sh->last_n1 = h->h_small[0];
    }
    if (n_clicks) *n_clicks = h->sh->last_nS;
    if (n_occupied) *n_occupied = h->sh->last_n1;
    return 0;
  }
  if (h->k1_dev && n_occupied) {           // general path: k1 of the last projective step (device)
    CK(cudaMemcpyAsync(h->h_small, h->k1 + traj, 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    h->last_n1[traj] = h->h_small[0];
  }
  if (h->cfg.protocol == TRAJ_PROJECTIVE_EVENTS && n_occupied) {
    int32_t v = 0;
    CK(cudaMemcpyAsync(&v, h->occ_count + traj, 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    h->last_n1[traj] = v;
  }
  if (h->small_last_dev) {   // fused small-lattice step: counts of the last step on the device
    CK(cudaMemcpyAsync(h->h_small, h->small_last + 2 * traj, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    h->last_nS[traj] = h->h_small[0];
    h->last_n1[traj] = h->h_small[1];
  }
  if (n_clicks) *n_clicks = h->last_nS[traj];
  if (n_occupied) *n_occupied = h->last_n1[traj];
  return 0;
}

int traj_gram_deviation(traj_handle h, double* out) {
  if (!h || !out) return TRAJ_EINVAL;
  const unsigned long long* dev = h->sh ? h->sh->gdev : (h->small ? nullptr : h->gdev);
  if (!dev) return fail(h, TRAJ_EINVAL, "traj_gram_deviation: the fused small-lattice step keeps the Gram in shared memory");
  const int T = h->sh ? 1 : h->T;
  CK(cudaMemcpyAsync(h->h_dev, dev, (size_t)T * 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  memcpy(out, h->h_dev, (size_t)T * 8);
  return 0;
}

int traj_cqr2_fallbacks(traj_handle h, int64_t* n) {
  if (!h || !n) return TRAJ_EINVAL;
  *n = h->sh ? h->sh->cqr2_fallbacks : h->cqr2_fallbacks;
  // the fused small-lattice step and the general path's device-side decision count on the device
  const unsigned long long* dev = h->sh ? h->sh->fb_dev : (h->small ? h->small_fallbacks : h->fb_dev);
  if (dev) {
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(h->h_dev, dev, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    memcpy(&v, h->h_dev, 8);
    *n += (int64_t)v;
  }
  return 0;
}

int traj_probe_orthonormality(traj_handle h, double* est_out) {
  if (!h || !est_out) return TRAJ_EINVAL;
  if (h->sh) return fail(h, TRAJ_EINVAL, "traj_probe_orthonormality: not available with row sharding");
  TRY(probe_orthonormality(h->st, h->U[h->cur], h->ldN, h->sU, h->L, h->N, h->T, h->step, h->cfg.traj_base,
                           h->cfg.seed, h->PX, h->PY, h->Ppart, h->pest, &h->err));
  CK(cudaMemcpyAsync(est_out, h->pest, h->T * 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return 0;
}

int traj_lowrank_stats(traj_handle h, int64_t* newton_iters, int64_t* fallbacks, int64_t* probes,
                       int64_t* refinements) {
  if (!h) return TRAJ_EINVAL;
  if (newton_iters) *newton_iters = h->lowrank_iters;
  if (fallbacks) *fallbacks = h->lowrank_fallbacks;
  if (probes) *probes = h->lowrank_probes;
  if (refinements) *refinements = h->lowrank_refinements;
  return 0;
}

int traj_profile(traj_handle h, int enable) {
  if (!h) return TRAJ_EINVAL;
  CK(cudaStreamSynchronize(h->st));
  h->prof.reset(enable != 0);
  return 0;
}

int traj_ozaki_info(traj_handle h, int32_t* out3) {
  if (!h || !out3) return TRAJ_EINVAL;
  if (h->sh) {   // row-sharded: K_g U, the local Grams and TRMMs together
    out3[0] = out3[1] = h->sh->oz ? 1 : 0;
    out3[2] = h->sh->oz ? h->sh->oz_s : 0;
    return 0;
  }
  out3[0] = h->oz_ku ? 1 : 0;
  out3[1] = h->oz_cqr ? 1 : 0;
  out3[2] = (h->oz_ku || h->oz_cqr) ? h->oz_s : 0;
  return 0;
}

int traj_phase_times(traj_handle h, double* ms, int64_t* launches) {
  if (!h) return TRAJ_EINVAL;
  CK(cudaStreamSynchronize(h->st));
  h->prof.collect();
  for (int p = 0; p < TRAJ_NPHASES; ++p) {
    if (ms) ms[p] = h->prof.ms[p];
    if (launches) launches[p] = h->prof.launches[p];
  }
  return 0;
}

int traj_destroy(traj_handle h) {
  if (!h) return TRAJ_EINVAL;
  if (h->st) cudaStreamSynchronize(h->st);
  if (h->sh) {
    shard_destroy(h->sh);
    delete h->sh;
  }
  h->prof.destroy();
  h->fbg.destroy();
  for (cudaStream_t q : {h->st_hi, h->st_lo})
    if (q) {
      cudaStreamSynchronize(q);
      cudaStreamDestroy(q);
    }
  for (cudaEvent_t e : {h->ev_fork, h->ev_left, h->ev_lo_done, h->ev_hi_done, h->ev_split})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h->sc_ev) cudaEventDestroy(e);
  if (h->solver) cusolverDnDestroy(h->solver);
  if (h->h_small) cudaFreeHost(h->h_small);
  if (h->h_dev) cudaFreeHost(h->h_dev);
  if (h->taps_host) cudaFreeHost(h->taps_host);
  delete h;
  return 0;
}

int traj_dgemm(void* stream, int64_t M, int64_t N, int64_t K, double alpha, const void* A, int64_t lda,
               int64_t strideA, const void* B, int64_t ldb, int64_t strideB, double beta, void* C, int64_t ldc,
               int64_t strideC, int64_t batch) {
  if (M < 0 || N < 0 || K < 0 || batch < 0 || !C || (K > 0 && (!A || !B))) return fail(nullptr, TRAJ_EINVAL, "traj_dgemm: bad argument");
  std::string e;
  const int s = dgemm_nn(reinterpret_cast<cudaStream_t>(stream), M, N, K, alpha, reinterpret_cast<const double*>(A), lda,
                         strideA, reinterpret_cast<const double*>(B), ldb, strideB, beta, reinterpret_cast<double*>(C),
                         ldc, strideC, batch, &e);
  return s ? fail(nullptr, s == 1 ? TRAJ_EINVAL : s, e) : 0;
}

int traj_zgemm(void* stream, int opA, int opB, int64_t M, int64_t N, int64_t K, double alpha_re, double alpha_im,
               const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb, int64_t strideB, double beta,
               void* C, int64_t ldc, int64_t strideC, int64_t batch, int flags) {
  if ((opA != 0 && opA != 1) || (opB != 0 && opB != 1) || M < 0 || N < 0 || K < 0 || batch < 0 || !C ||
      (K > 0 && (!A || !B)))
    return fail(nullptr, TRAJ_EINVAL, "traj_zgemm: bad arguments");
  std::string e;
  int s = zgemm(reinterpret_cast<cudaStream_t>(stream), opA, opB, M, N, K, alpha_re, alpha_im,
                reinterpret_cast<const cplx*>(A), lda, strideA, reinterpret_cast<const cplx*>(B), ldb, strideB, beta,
                reinterpret_cast<cplx*>(C), ldc, strideC, batch, flags, &e);
  return s ? fail(nullptr, s, e) : 0;
}

int traj_igemm(void* stream, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int64_t strideA,
               const void* B, int64_t ldb, int64_t strideB, void* C, int64_t ldc, int64_t strideC, int64_t batch,
               const int32_t* moduli, int nmod, int flags) {
  if (M < 0 || N < 0 || batch < 0 || !A || !B || !C || (flags & ~3)) return fail(nullptr, TRAJ_EINVAL, "traj_igemm: bad argument");
  IgemmArgs g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.batch = batch;
  g.A = reinterpret_cast<const int8_t*>(A);
  g.lda = lda;
  g.strideA = strideA;
  g.B = reinterpret_cast<const int8_t*>(B);
  g.ldb = ldb;
  g.strideB = strideB;
  g.C = C;
  g.ldc = ldc;
  g.strideC = strideC;
  g.out = moduli ? IG_OUT_MOD : IG_OUT_I32;
  g.moduli = moduli;
  g.nmod = nmod;
  g.flags = flags;
  std::string e;
  const int s = igemm(reinterpret_cast<cudaStream_t>(stream), g, &e);
  return s ? fail(nullptr, s == 1 ? TRAJ_EINVAL : TRAJ_ECUDA, e) : 0;
}

int traj_zgemm_ozaki(void* stream, int opA, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                     const void* B, int64_t ldb, void* C, int64_t ldc, int nmod, int flags) {
  if ((opA != 0 && opA != 1) || M < 0 || N < 0 || K <= 0 || !A || !B || !C || !oz_supported(nmod) || M > 65535 ||
      (flags & ~(TRAJ_C_UPPER | TRAJ_TRI_B_UPPER)) || lda < (opA ? M : K) || ldb < N || ldc < N)
    return fail(nullptr, TRAJ_EINVAL, "traj_zgemm_ozaki: bad argument");
  if (M == 0 || N == 0) return 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int s = nmod;
  const long long na = opA ? 4 : 3;
  const size_t bA = (size_t)oz_residue_bytes(na, s, 1, M, K), bB = (size_t)oz_residue_bytes(3, s, 1, N, K),
               bC = (size_t)oz_residue_bytes(3, s, 1, M, N);
  const size_t bE = (size_t)(M + N) * 4 + 256, bP = (size_t)8 * std::max(M, N) * 8 + 256;
  char* w = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&w), bA + bB + bC + bE + bP + 1024, st) != cudaSuccess)
    return fail(nullptr, TRAJ_ECUDA, "traj_zgemm_ozaki: scratch allocation");
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  int8_t* RA = reinterpret_cast<int8_t*>(w);
  int8_t* RB = reinterpret_cast<int8_t*>(w + al(bA));
  uint8_t* RC = reinterpret_cast<uint8_t*>(w + al(bA) + al(bB));
  int* eA = reinterpret_cast<int*>(w + al(bA) + al(bB) + al(bC));
  int* eB = eA + al((size_t)M * 4) / 4;
  double* part = reinterpret_cast<double*>(w + al(bA) + al(bB) + al(bC) + al(bE));
  std::string e;
  const cplx* a = reinterpret_cast<const cplx*>(A);
  const cplx* b = reinterpret_cast<const cplx*>(B);
  int r = 0;
  OzProduct p;
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.T = 1;
  p.s = s;
  p.RA = RA;
  p.a_traj = 0;
  p.eA = eA;
  p.RB = RB;
  p.eB = eB;
  p.RC = RC;
  p.C = reinterpret_cast<cplx*>(C);
  p.ldc = ldc;
  p.flags = ((flags & TRAJ_C_UPPER) ? OZ_UPPER : 0) | ((flags & TRAJ_TRI_B_UPPER) ? OZ_TRI_B : 0);
  if (opA == 0) {
    r = oz_split_rows(st, a, lda, 0, (int)M, (int)K, 1, 0, s, RA, eA, 0, &e);
  } else {   // A^dag B = (P1 + P2') + i (P3 - P1 + P2'): P1 = Ar^T Br, P2' = Ai^T Bi, P3 = (Ar - Ai)^T (Br + Bi)
    r = oz_split_cols(st, a, lda, 0, (int)K, (int)M, 1, 4, s, RA, eA, 0, part, &e);
    p.a_planes = 4;
    p.pa[2] = 3;
    p.flags |= OZ_NEG_P2;
  }
  if (!r) r = oz_split_cols(st, b, ldb, 0, (int)K, (int)N, 1, 3, s, RB, eB, 0, part, &e);
  if (!r) r = oz_product(st, p, &e);
  cudaFreeAsync(w, st);
  return r ? fail(nullptr, r == 1 ? TRAJ_EINVAL : TRAJ_ECUDA, e) : 0;
}

int traj_ozaki_constants(int nmod, int32_t* moduli, int32_t* beta, double* ch, double* cl, double* M) {
  if (!moduli || !beta || !ch || !cl || !M || oz_constants(nmod, moduli, beta, ch, cl, M))
    return fail(nullptr, TRAJ_EINVAL, "traj_ozaki_constants: nmod must be 4..18 even");
  return 0;
}

int traj_ozaki_roots(int nmod, int32_t* roots) {
  if (!roots || oz_roots(nmod, roots)) return fail(nullptr, TRAJ_EINVAL, "traj_ozaki_roots: nmod must be 4..18 even");
  return 0;
}

int traj_set_zgemm_algorithm(int algo) {
  if (algo != 0 && algo != 1) return fail(nullptr, TRAJ_EINVAL, "algorithm must be 0 (4M) or 1 (3M)");
  set_zgemm_algorithm(algo);
  return 0;
}

int traj_get_zgemm_algorithm(void) { return zgemm_algorithm(); }

int traj_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, TRAJ_EINVAL, "null out");
  std::string e;
  int s = nccl_unique_id(out128, &e);
  return s ? fail(nullptr, s, e) : 0;
}

int64_t traj_comm_plan(int kind, int P, int rank, int64_t n, int64_t* out, int64_t max_entries) {
  if (P < 1 || P > 1024 || rank < 0 || rank >= P || max_entries < 0 || (max_entries > 0 && !out))
    return -fail(nullptr, TRAJ_EINVAL, "traj_comm_plan: bad arguments");
  std::vector<int64_t> flat;
  if (kind == 0 || kind == 1) {
    for (const CommOp& op : kind == 0 ? ring_plan(P, rank) : halo_plan(P, rank))
      flat.insert(flat.end(), {op.group, op.kind, op.peer, op.slot, op.block});
  } else if (kind == 2) {
    if (n < 1) return -fail(nullptr, TRAJ_EINVAL, "traj_comm_plan: n < 1");
    const char* dm = getenv("TRAJ_DIST_CHOL_MIN");
    const long long mn = dm ? atoll(dm) : 2048;
    std::vector<BcastOp> b;
    if (mn > 0) dist_chol_plan_rec(n, P, mn, &b);
    for (const BcastOp& op : b) flat.insert(flat.end(), {op.root, op.rows, op.cols});
  } else {
    return -fail(nullptr, TRAJ_EINVAL, "traj_comm_plan: unknown kind");
  }
  const int64_t w = kind == 2 ? 3 : 5, count = (int64_t)flat.size() / w;
  for (int64_t i = 0; i < std::min<int64_t>(count, max_entries) * w; ++i) out[i] = flat[i];
  return count;
}

int traj_shard_info(traj_handle h, int32_t* shard_size, int32_t* local_shards, int64_t* row0, int64_t* rows) {
  if (!h) return TRAJ_EINVAL;
  if (h->sh) {
    if (shard_size) *shard_size = h->sh->P;
    if (local_shards) *local_shards = h->sh->comm.P_local;
    if (row0) *row0 = (int64_t)h->sh->comm.rank0 * h->sh->Lp;
    if (rows) *rows = (int64_t)h->sh->comm.P_local * h->sh->Lp;
  } else {
    if (shard_size) *shard_size = 1;
    if (local_shards) *local_shards = 1;
    if (row0) *row0 = 0;
    if (rows) *rows = h->L;
  }
  return 0;
}

size_t traj_chol_scratch_bytes(int64_t n, int64_t batch) { return chol_scratch_bytes(n, batch); }

int traj_chol_inverse(void* stream, int64_t n, void* G, int64_t ldg, int64_t strideG, void* X, int64_t ldx,
                      int64_t strideX, int64_t batch, void* scratch, int32_t* failed) {
  if (n < 0 || batch < 0 || (n > 0 && (!G || !X || !scratch))) return fail(nullptr, TRAJ_EINVAL, "bad arguments");
  std::string e;
  int s = chol_inverse(reinterpret_cast<cudaStream_t>(stream), n, reinterpret_cast<cplx*>(G), ldg, strideG,
                       reinterpret_cast<cplx*>(X), ldx, strideX, batch, scratch, failed, &e);
  return s ? fail(nullptr, s, e) : 0;
}

}  // extern "C"
