// Row-sharded trajectory step (north star: "K and U are row-sharded,
// with an NCCL allgather of U over NVLink each step and an allreduce of the Gram matrix").
//
// Shard g owns rows [g Lp, (g+1) Lp) of K and U (Lp = L / P).  One step:
//   allgather U rows -> U_full;  U_g <- K_g U_full                           (a1)
//   homodyne: local rows, Philox at global site ids                          (a2)
//   projective: local clicks -> allgather (counts, sites, U_S rows) -> the replicated,
//     deterministic C_SS / sampling / W on every shard -> local rank-k update  (a2)
//   CholeskyQR2: G_g = U_g^dag U_g -> allreduce -> replicated factor -> U_g X  (a3)
// Replicated decisions are bitwise identical on every shard: the all-reduced / gathered
// inputs are identical and the kernels are deterministic.
#include <cusolverDn.h>
#include <math.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <complex>

#include "cholinv.h"
#include "monitor.h"
#include "shard.h"
#include "zgemm.h"
#include "banded.h"
#include "dgemm.h"
#include "planar.h"
#include "comm_plan.h"
#include "ozaki.h"

namespace traj {

namespace {

struct Lay {
  size_t off = 0;
  char* base = nullptr;
  template <typename P>
  void take(P*& p, size_t bytes) {
    off = (off + 255) & ~size_t(255);
    p = base ? reinterpret_cast<P*>(base + off) : nullptr;
    off += bytes;
  }
};

std::string cuerr(const char* what, cudaError_t e) { return std::string(what) + ": " + cudaGetErrorString(e); }

#define SCK(x)                            \
  do {                                    \
    cudaError_t e_ = (x);                 \
    if (e_ != cudaSuccess) {              \
      if (err) *err = cuerr(#x, e_);      \
      return TRAJ_ECUDA;                  \
    }                                     \
  } while (0)
#define STRY(x)             \
  do {                      \
    int s_ = (x);           \
    if (s_) return s_;      \
  } while (0)

int capacity(long long n, double p) {
  const double m = n * p, sd = sqrt(n * p * (1 - p));
  return (int)std::min<long long>(n, (long long)ceil(m + 12 * sd + 64));
}

}  // namespace

int ShardComm::begin(std::string* err) {
  const int s = wd.check(err);
  if (s) return s;
  wd.lock();
  if (wd.aborted()) {   // aborted while waiting for the lock
    wd.unlock();
    return wd.check(err);
  }
  return 0;
}

void ShardComm::end(cudaStream_t st) {
  wd.unlock();
  wd.mark(st, nullptr);   // the watchdog times every enqueued collective
}

int ShardComm::allgather(cudaStream_t st, void* const* send, void* recv, size_t bytes, std::string* err) {
  if (comm) {
    STRY(begin(err));
    ncclResult_t r = ncclAllGather(send[0], recv, bytes, ncclUint8, comm, st);
    end(st);
    if (r != ncclSuccess) {
      if (err) *err = std::string("ncclAllGather: ") + ncclGetErrorString(r);
      return TRAJ_ENCCL;
    }
    return 0;
  }
  for (int s = 0; s < P_local; ++s) {
    char* dst = reinterpret_cast<char*>(recv) + (size_t)(rank0 + s) * bytes;
    if (dst == send[s]) continue;
    cudaError_t e = cudaMemcpyAsync(dst, send[s], bytes, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
      if (err) *err = cuerr("allgather (emulated)", e);
      return TRAJ_ECUDA;
    }
  }
  return 0;
}

int ShardComm::allreduce(cudaStream_t st, double* const* part, double* out, size_t n, std::string* err) {
  if (comm) {
    STRY(begin(err));
    ncclResult_t r = ncclAllReduce(part[0], out, n, ncclFloat64, ncclSum, comm, st);
    end(st);
    if (r != ncclSuccess) {
      if (err) *err = std::string("ncclAllReduce: ") + ncclGetErrorString(r);
      return TRAJ_ENCCL;
    }
    return 0;
  }
  if (out != part[0]) {
    cudaError_t e = cudaMemcpyAsync(out, part[0], n * 8, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
      if (err) *err = cuerr("allreduce (emulated)", e);
      return TRAJ_ECUDA;
    }
  }
  for (int s = 1; s < P_local; ++s) STRY(add_inplace(st, out, part[s], (long long)n, err));
  return 0;
}

int ShardComm::halo(cudaStream_t st, void* const* send_lo, void* const* send_hi, void* const* recv_lo,
                    void* const* recv_hi, size_t bytes, std::string* err) {
  if (comm) {
    // the schedule of comm_plan.h halo_plan: NCCL pairs operations between two ranks in issue
    // order, and with P <= 2 left == right -- the plan's order makes both sides agree
    void* const* sendv[2] = {send_lo, send_hi};
    void* const* recvv[2] = {recv_lo, recv_hi};
    STRY(begin(err));
    ncclGroupStart();
    for (const CommOp& op : halo_plan(P, rank0)) {
      if (op.kind == COMM_SEND) ncclSend(sendv[op.slot][0], bytes, ncclUint8, op.peer, comm, st);
      else ncclRecv(recvv[op.slot][0], bytes, ncclUint8, op.peer, comm, st);
    }
    ncclResult_t r = ncclGroupEnd();
    end(st);
    if (r != ncclSuccess) {
      if (err) *err = std::string("nccl halo exchange: ") + ncclGetErrorString(r);
      return TRAJ_ENCCL;
    }
    return 0;
  }
  for (int s = 0; s < P_local; ++s) {
    const int left = (s + P - 1) % P, right = (s + 1) % P;
    cudaError_t e = cudaMemcpyAsync(recv_lo[s], send_hi[left], bytes, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(recv_hi[s], send_lo[right], bytes, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
      if (err) *err = cuerr("halo (emulated)", e);
      return TRAJ_ECUDA;
    }
  }
  return 0;
}

bool shard_banded_fits(const traj_config* c, int Wx, int Wy, std::string* why) {
  const long long L = c->Lx * c->Ly, Lp = L / c->shard_size;
  const long long H = c->Ly > 1 ? (long long)Wy * c->Lx : Wx;
  if (c->Ly > 1 && Lp % c->Lx) {
    *why = "banded + sharded 2d needs whole lattice rows per shard (Ly divisible by shard_size)";
    return false;
  }
  if (H > Lp) {
    *why = "banded + sharded needs the halo (W rows in 1d, W*Lx in 2d) within one neighbouring shard";
    return false;
  }
  return true;
}

int nccl_unique_id(void* out128, std::string* err) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    if (err) *err = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
    return TRAJ_ENCCL;
  }
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int shard_validate(const traj_config* c, std::string* why) {
  const long long L = c->Lx * c->Ly;
  if (c->shard_size < 1 || c->shard_size > 1024) {
    *why = "shard_size must be in [1, 1024]";
    return TRAJ_ECONFIG;
  }
  if (L % c->shard_size) {
    *why = "L must be divisible by shard_size";
    return TRAJ_ECONFIG;
  }
  if (c->n_traj != 1) {
    *why = "row sharding holds a single trajectory (n_traj = 1)";
    return TRAJ_ECONFIG;
  }
  if (c->nccl_id) {
    if (c->shard_rank < 0 || c->shard_rank >= c->shard_size) {
      *why = "shard_rank outside [0, shard_size)";
      return TRAJ_ECONFIG;
    }
  } else if (c->shard_rank != 0) {
    *why = "single-GPU shard emulation (nccl_id = NULL) needs shard_rank = 0";
    return TRAJ_ECONFIG;
  }
  return 0;
}

size_t shard_carve(ShardedCtx* sh, const traj_config* c, char* base, int lwork, bool banded, int Wx, int Wy) {
  Lay lay;
  lay.base = base;
  const long long L = c->Lx * c->Ly, N = c->N;
  const int P = c->shard_size;
  const bool emulate = c->nccl_id == nullptr;
  sh->comm.P = P;
  sh->comm.P_local = emulate ? P : 1;
  sh->comm.rank0 = emulate ? 0 : c->shard_rank;
  sh->L = (int)L;
  sh->N = (int)N;
  sh->Lx = (int)c->Lx;
  sh->Ly = (int)c->Ly;
  sh->P = P;
  sh->Lp = (int)(L / P);
  sh->ldN = round_up(N, 8);
  sh->ldL = round_up(L, 8);
  const double p = c->protocol == TRAJ_PROJECTIVE ? c->gamma[0] * c->dt : 0.0;
  sh->capr = c->protocol == TRAJ_PROJECTIVE ? capacity(sh->Lp, p) : 0;
  sh->cap = sh->capr * P;
  sh->ldcap = round_up(std::max(sh->cap, 1), 8);
  sh->lwork = lwork;
  sh->banded = banded;
  sh->Wx = Wx;
  sh->Wy = Wy;
  sh->H = banded ? (c->Ly > 1 ? Wy * (int)c->Lx : Wx) : 0;
  const long long Lp = sh->Lp, ldN = sh->ldN, ldL = sh->ldL, ldcap = sh->ldcap;
  const int capr = sh->capr, cap = sh->cap;
  {
    const char* pk = getenv("TRAJ_PLANAR_KU");
    const char* pc = getenv("TRAJ_PLANAR_CQR");
    const char* mn = getenv("TRAJ_PLANAR_MIN_N");
    const long long min_n = mn ? atoll(mn) : 512;
    // (K_g's chunk columns start at s Lp doubles: TMA needs them 16-byte aligned, so Lp even)
    sh->planar = !banded && !(pk && pk[0] == '0') && !(pc && pc[0] == '0') && N >= min_n && (L / P) % 2 == 0;
    sh->ldKs = round_up(L, 16);
    sh->ldPs = round_up(N, 16);
    // the modular engine replaces the planar one (K_g's chunk columns start at byte s Lp of its residue
    // rows: TMA needs 16-byte alignment, so Lp % 16 == 0 unless P == 1)
    const char* oz = getenv("TRAJ_OZAKI");
    const char* om = getenv("TRAJ_OZAKI_MODULI");
    const char* oc = getenv("TRAJ_OZAKI_CORR_MODULI");
    sh->oz_s = om ? atoi(om) : 16;
    sh->oz_s_corr = oc ? atoi(oc) : 10;
    if (sh->oz_s_corr != 0 && !oz_supported(sh->oz_s_corr)) sh->oz_s_corr = 10;
    sh->oz = !banded && !(oz && oz[0] == '0') && oz_supported(sh->oz_s) && N >= min_n && L / P <= 65535 &&
             N <= 65535 && (P == 1 || (L / P) % 16 == 0);
    if (sh->oz) sh->planar = false;
    const char* ck = getenv("TRAJ_SHARD_OZ_CHUNKS");
    sh->oz_chunked = ck && ck[0] == '1';
    if (sh->planar) {
      // the unsharded rule (traj_api.cu carve) on the Lp x Lp chunks
      const char* sv = getenv("TRAJ_STRASSEN");
      const char* sm = getenv("TRAJ_STRASSEN_MIN_N");
      const char* lv = getenv("TRAJ_STRASSEN_LEVELS");
      const long long smin = sm ? atoll(sm) : 2048, Lp = L / P;
      const bool one_ok = !(sv && sv[0] == '0') && Lp % 2 == 0 && N % 2 == 0 && N >= smin;
      const bool two_ok = one_ok && Lp % 4 == 0 && N % 4 == 0 &&
                          147.0 * P * (Lp / 4) * round_up(Lp / 4, 16) * 8 * sh->comm.P_local <= 24e9;
      sh->slv = !one_ok ? 0 : (lv ? (atoi(lv) >= 2 && two_ok ? 2 : 1) : (two_ok ? 2 : 1));
      if (sh->slv) {
        sh->ldS = round_up(Lp >> sh->slv, 16);
        sh->ldSM = round_up(N >> sh->slv, 16);
      }
    }
  }
  sh->loc.assign(sh->comm.P_local, ShardLocal());
  lay.take(sh->Ufull, (size_t)L * ldN * 16);
  lay.take(sh->G, (size_t)N * ldN * 16);
  lay.take(sh->X, (size_t)N * ldN * 16);
  lay.take(sh->chol_scratch, chol_scratch_bytes(N, 1));
  for (int s = 0; s < sh->comm.P_local; ++s) {
    ShardLocal& l = sh->loc[s];
    l.g = sh->comm.rank0 + s;
    l.row0 = (int)(l.g * Lp);
    if (banded) {
      lay.take(l.Uext, (size_t)(Lp + 2 * sh->H) * ldN * 16);
    } else if (sh->oz) {
      lay.take(l.RK, (size_t)oz_residue_bytes(2, sh->oz_s, 1, Lp, L));
      lay.take(l.eK, (size_t)Lp * 4);
    } else if (sh->planar) {
      lay.take(l.Kp, (size_t)3 * Lp * sh->ldKs * 8);
      if (sh->slv)
        lay.take(l.Ks, (size_t)P * strassen_products(sh->slv) * (Lp >> sh->slv) * sh->ldS * 8);
      lay.take(l.Pp, (size_t)3 * Lp * sh->ldPs * 8);
      lay.take(l.Up6, (size_t)6 * Lp * sh->ldPs * 8);
    } else {
      lay.take(l.K, (size_t)Lp * ldL * 16);
    }
    lay.take(l.U[0], (size_t)Lp * ldN * 16);
    lay.take(l.U[1], (size_t)Lp * ldN * 16);
    if (emulate) lay.take(l.Gpart, (size_t)N * ldN * 16);
    else l.Gpart = sh->G;
    if (cap > 0) {
      lay.take(l.flags, (size_t)Lp * 4);
      lay.take(l.Sloc, (size_t)capr * 4);
      lay.take(l.cnt, 16);
      lay.take(l.USloc, (size_t)capr * ldN * 16);
      lay.take(l.Tm, (size_t)Lp * ldcap * 16);
    }
  }
  if (banded) lay.take(sh->bcoef, (size_t)(2 * Wx + 2 * Wy + 2) * 16);
  if (sh->slv) {
    const size_t nb = (size_t)strassen_products(sh->slv) * (Lp >> sh->slv) * sh->ldSM * 8;
    lay.take(sh->Sb, nb);
    lay.take(sh->Sm, nb);
  }
  if (sh->planar) {
    lay.take(sh->Cp, (size_t)3 * Lp * sh->ldPs * 8);
    lay.take(sh->Gp, (size_t)3 * N * sh->ldPs * 8);
    lay.take(sh->Xp, (size_t)3 * N * sh->ldPs * 8);
  }
  if (sh->oz) {
    const int q = sh->oz_s;
    const long long mx = std::max(Lp, N);
    // (C_SS's 4-plane row split of U_S: at most N rows on the modular path)
    lay.take(sh->RU, (size_t)std::max({oz_residue_bytes(4, q, 1, N, Lp), oz_residue_bytes(3, q, 1, Lp, N),
                                       oz_residue_bytes(4, q, 1, std::min<long long>(cap, N), N),
                                       sh->oz_chunked ? 0ll : oz_residue_bytes(3, q, 1, N, L)}));
    lay.take(sh->RX, (size_t)oz_residue_bytes(3, q, 1, N, N));
    // (K_g is built there, complex, before its split)
    sh->RC_bytes = (size_t)std::max({oz_residue_bytes(3, q, 1, Lp, N), oz_residue_bytes(3, q, 1, N, N),
                                     (long long)Lp * ldL * 16});
    lay.take(sh->RC, sh->RC_bytes);
    lay.take(sh->eU, (size_t)mx * 4);
    lay.take(sh->eU2, (size_t)mx * 4);
    lay.take(sh->eX, (size_t)N * 4);
    lay.take(sh->eG, (size_t)N * 4);
    lay.take(sh->nu2, (size_t)N * 8);
    lay.take(sh->oz_part, (size_t)8 * mx * 8);
  }
  if (c->nccl_id && sh->planar) {   // packed, pipelined Gram allreduce: two panel buffers
    const char* gp = getenv("TRAJ_GRAM_PANEL");
    const long long pw = gp ? atoll(gp) : 1024;
    sh->gram_pw = pw > 0 ? (int)std::min<long long>(round_up(pw, 64), round_up(N, 64)) : 0;
    if (sh->gram_pw) lay.take(sh->gpack, (size_t)2 * N * sh->gram_pw * 16);
  }
  if (c->nccl_id && sh->P > 1) {   // distributed Cholesky: the largest shared block, (N/2 + 128)^2
    const long long hb = (long long)sh->N / 2 + 128;
    sh->dist_scratch_bytes = (size_t)(hb * hb * 16);
    lay.take(sh->dist_scratch, sh->dist_scratch_bytes);
  }
  lay.take(sh->gamma_dev, 16);
  lay.take(sh->failed_dev, 16);
  lay.take(sh->eig_w, (size_t)N * 8);
  lay.take(sh->eig_work, (size_t)std::max(lwork, 1) * 16);
  lay.take(sh->eig_info, 16);
  lay.take(sh->S_dev, 16);
  lay.take(sh->bad_dev, 16);
  lay.take(sh->gdev, 16);
  lay.take(sh->fb_dev, 16);
  lay.take(sh->gate, 16);
  lay.take(sh->region, (size_t)L * 4);
  lay.take(sh->kcoef, (size_t)(c->Lx + c->Ly) * 16);
  lay.take(sh->sites, (size_t)N * 4);
  lay.take(sh->obs_bins, (size_t)L * 8);
  lay.take(sh->obs_part, 1024 * 8);
  lay.take(sh->obs_out, 16);
  lay.take(sh->obs_mask, (size_t)L * 4);
  if (cap > 0) {
    lay.take(sh->Srecv, (size_t)cap * 4);
    lay.take(sh->cntrecv, (size_t)P * 4);
    lay.take(sh->USrecv, (size_t)cap * ldN * 16);
    lay.take(sh->S, (size_t)cap * 4);
    lay.take(sh->count, 16);
    lay.take(sh->US, (size_t)cap * ldN * 16);
    lay.take(sh->D0, (size_t)cap * ldcap * 16);
    lay.take(sh->Dw, (size_t)cap * ldcap * 16);
    lay.take(sh->Linv, 64 * 64 * 16);
    lay.take(sh->DLinv, 64 * 64 * 16);
    lay.take(sh->Ybuf, (size_t)64 * ldcap * 16);
    lay.take(sh->Zbuf, (size_t)64 * ldcap * 16);
    lay.take(sh->occ, (size_t)cap * 4);
    lay.take(sh->pos1, (size_t)cap * 4);
    lay.take(sh->S1, (size_t)cap * 4);
    lay.take(sh->S0, (size_t)cap * 4);
    lay.take(sh->pos0, (size_t)cap * 4);
    lay.take(sh->k1, 16);
    lay.take(sh->k0, 16);
    lay.take(sh->D11, (size_t)cap * ldcap * 16);
    lay.take(sh->X11, (size_t)cap * ldcap * 16);
    lay.take(sh->chol_scratch_small, chol_scratch_bytes(cap, 1));
    lay.take(sh->W, (size_t)N * ldcap * 16);
    // structured CholeskyQR pass 1 (structchol.h): Y [cap][b], C [b][b], X blocks [N][b], W, Z [cap][ldN]
    const char* sbv = getenv("TRAJ_STRUCT_B");
    const char* opm = getenv("TRAJ_OZAKI_PROJ_MIN");
    sh->oz_proj_min = opm ? atoi(opm) : 1024;
    // (the unsharded rule: wide blocks once the solve runs modular)
    const int b = sbv ? std::max(16, std::min(2048, atoi(sbv) / 16 * 16))
                      : (cap >= 1024 ? (sh->oz && cap >= sh->oz_proj_min ? 2048 : 512) : 128);
    sh->sc.b = b;
    sh->sc.N = (int)N;
    sh->sc.T = 1;
    sh->sc.M = sh->Dw;
    sh->sc.ldM = ldcap;
    sh->sc.sM = 0;
    lay.take(sh->sc.Y, (size_t)cap * b * 16);
    lay.take(sh->sc.C, (size_t)b * b * 16);
    lay.take(sh->sc.Xb, (size_t)round_up(N, b) * b * 16);
    lay.take(sh->sc.W, (size_t)cap * ldN * 16);
    lay.take(sh->sc.Z, (size_t)cap * ldN * 16);
    sh->sc.ldWZ = ldN;
    lay.take(sh->sc.chol_scratch, chol_scratch_bytes(b, 1));
  }
  return lay.off + 256;
}

namespace {

// make the row slices of a (ld-strided, ncols-wide) block computed by each rank visible everywhere:
// the owner packs its slice into the contiguous scratch, one grouped broadcast per owner, every
// other rank unpacks (only the block's columns travel)
int dist_share_rows(void* user, cplx* base, long long ld, long long ncols, const long long* bounds, int P,
                    cudaStream_t st, std::string* err) {
  ShardedCtx* sh = reinterpret_cast<ShardedCtx*>(user);
  const int me = sh->cdist.rank;
  cplx* scr = sh->dist_scratch;
  if ((bounds[P]) * ncols * 16 > (long long)sh->dist_scratch_bytes) {
    if (err) *err = "distributed Cholesky: share scratch too small";
    return TRAJ_ECUDA;
  }
  const size_t w = (size_t)ncols * 16;
  if (bounds[me + 1] > bounds[me])
    SCK(cudaMemcpy2DAsync(scr + bounds[me] * ncols, w, base + bounds[me] * ld, (size_t)ld * 16, w,
                          (size_t)(bounds[me + 1] - bounds[me]), cudaMemcpyDeviceToDevice, st));
  STRY(sh->comm.begin(err));
  ncclGroupStart();
  for (int i = 0; i < P; ++i) {
    if (bounds[i + 1] <= bounds[i]) continue;
    cplx* p = scr + bounds[i] * ncols;
    ncclBroadcast(p, p, (size_t)(bounds[i + 1] - bounds[i]) * w, ncclUint8, i, sh->comm.comm, st);
  }
  ncclResult_t r = ncclGroupEnd();
  sh->comm.end(st);
  if (r != ncclSuccess) {
    if (err) *err = std::string("ncclBroadcast (distributed Cholesky): ") + ncclGetErrorString(r);
    return TRAJ_ENCCL;
  }
  for (int i = 0; i < P; ++i) {
    if (i == me || bounds[i + 1] <= bounds[i]) continue;
    SCK(cudaMemcpy2DAsync(base + bounds[i] * ld, (size_t)ld * 16, scr + bounds[i] * ncols, w, w,
                          (size_t)(bounds[i + 1] - bounds[i]), cudaMemcpyDeviceToDevice, st));
  }
  return 0;
}

}  // namespace

int shard_init(ShardedCtx* sh, const traj_config* c, std::string* err) {
  sh->protocol = c->protocol;
  sh->dt = c->dt;
  sh->J = c->J;
  sh->gamma = c->gamma[0];
  sh->seed = c->seed;
  sh->traj_base = c->traj_base;
  sh->st = reinterpret_cast<cudaStream_t>(c->stream);
  if (c->nccl_id) {
    ncclUniqueId id;
    memcpy(&id, c->nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&sh->comm.comm, c->shard_size, id, c->shard_rank);
    if (r != ncclSuccess) {
      if (err) *err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      return TRAJ_ENCCL;
    }
    const char* to = getenv("TRAJ_NCCL_TIMEOUT_S");
    int dev = 0;
    SCK(cudaGetDevice(&dev));
    STRY(sh->comm.wd.start(sh->comm.comm, dev, to ? atof(to) : 600.0, err));
    const char* ts = getenv("TRAJ_WATCHDOG_TEST_STALL");
    sh->test_stall = ts && ts[0] == '1';
  }
  SCK(cudaMallocHost(&sh->h_small, std::max(sh->P + 8, 64) * 4));
  SCK(cudaMallocHost(&sh->h_dev, 64 * 8));
  {
    const char* dm = getenv("TRAJ_DIST_CHOL_MIN");
    const long long mn = dm ? atoll(dm) : 2048;
    sh->cdist.P = mn > 0 ? sh->P : 1;
    sh->cdist.rank = sh->comm.comm ? c->shard_rank : -1;
    sh->cdist.min_n = mn > 0 ? mn : (1ll << 40);
    sh->cdist.user = sh;
    sh->cdist.share_rows = dist_share_rows;
  }
  {
    const char* lg = getenv("TRAJ_LOWRANK_GRAM");
    sh->lowrank_gram = !(lg && lg[0] == '0');
    const char* scv = getenv("TRAJ_STRUCT_CHOL");
    sh->struct_chol = !(scv && scv[0] == '0');
    const char* sp = getenv("TRAJ_STRUCT_PIPELINE");
    sh->struct_serial = sp && sp[0] == '0';
    const char* co = getenv("TRAJ_CHOL_OVERLAP");
    int least = 0, greatest = 0;
    sh->chol_overlap = !(co && co[0] == '0') && cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess &&
                       cudaStreamCreateWithPriority(&sh->st_hi, cudaStreamNonBlocking, greatest) == cudaSuccess &&
                       cudaStreamCreateWithPriority(&sh->st_lo, cudaStreamNonBlocking, least) == cudaSuccess;
    for (cudaEvent_t* e : {&sh->ev_fork, &sh->ev_left, &sh->ev_lo_done, &sh->ev_hi_done})
      if (sh->chol_overlap && cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess)
        sh->chol_overlap = false;
  }
  if (sh->comm.comm && sh->gpack) {
    SCK(cudaStreamCreateWithFlags(&sh->gst, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&sh->ev_gpacked[0], &sh->ev_gpacked[1], &sh->ev_gfree[0], &sh->ev_gfree[1], &sh->ev_gdone})
      SCK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  const char* ov = getenv("TRAJ_SHARD_OVERLAP");
  sh->overlap = !(ov && ov[0] == '0');
  if (sh->comm.comm && sh->overlap && sh->P > 1) {
    SCK(cudaStreamCreateWithFlags(&sh->cst, cudaStreamNonBlocking));
    SCK(cudaEventCreateWithFlags(&sh->ev_start, cudaEventDisableTiming));
    sh->ev_chunk.assign(sh->P, nullptr);
    for (auto& e : sh->ev_chunk) SCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return 0;
}

// upload the K coefficient rows and the initial occupied sites, build K blocks and U0
int shard_build(ShardedCtx* sh, const std::vector<std::complex<double>>& kc, const std::vector<int32_t>& sites,
                std::string* err, const std::vector<std::complex<double>>* band) {
  cudaStream_t st = sh->st;
  if (sh->banded) {
    SCK(cudaMemcpyAsync(sh->bcoef, band->data(), band->size() * 16, cudaMemcpyHostToDevice, st));
    sh->band_host.resize(band->size());
    for (size_t i = 0; i < band->size(); ++i) sh->band_host[i] = make_double2((*band)[i].real(), (*band)[i].imag());
  }
  SCK(cudaMemcpyAsync(sh->kcoef, kc.data(), kc.size() * 16, cudaMemcpyHostToDevice, st));
  SCK(cudaMemcpyAsync(sh->sites, sites.data(), sites.size() * 4, cudaMemcpyHostToDevice, st));
  SCK(cudaMemcpyAsync(sh->gamma_dev, &sh->gamma, 8, cudaMemcpyHostToDevice, st));
  for (auto& l : sh->loc) {
    if (sh->planar) {
      if (build_k_planar(st, l.Kp, sh->ldKs, (long long)sh->Lp * sh->ldKs, sh->Lx, sh->Ly, sh->kcoef,
                         sh->kcoef + sh->Lx, err, l.row0, sh->Lp))
        return 4;
      // the Strassen operands of every chunk K_g[:, s] (Lp x Lp at column s Lp of the planes)
      const long long ns = strassen_products(sh->slv), hh = sh->Lp >> sh->slv;
      for (int c = 0; sh->slv && c < sh->P; ++c)
        if (strassen_k(st, sh->slv, l.Kp + (long long)c * sh->Lp, sh->ldKs, (long long)sh->Lp * sh->ldKs, sh->Lp,
                       l.Ks + c * ns * hh * sh->ldS, sh->ldS, err))
          return 4;
    } else if (sh->oz) {   // K_g in the product scratch, then its row residues (once)
      cplx* Kt = reinterpret_cast<cplx*>(sh->RC);
      if (build_k(st, Kt, sh->ldL, sh->Lx, sh->Ly, sh->kcoef, sh->kcoef + sh->Lx, err, l.row0, sh->Lp) ||
          oz_split_rows(st, Kt, sh->ldL, 0, sh->Lp, sh->L, 1, 0, sh->oz_s, l.RK, l.eK, 0, err))
        return 4;
    } else if (!sh->banded &&
               build_k(st, l.K, sh->ldL, sh->Lx, sh->Ly, sh->kcoef, sh->kcoef + sh->Lx, err, l.row0, sh->Lp)) {
      return 4;
    }
    if (init_state(st, l.U[0], sh->ldN, 0, sh->sites, sh->N, 1, err, l.row0, sh->Lp)) return 4;
  }
  SCK(cudaStreamSynchronize(st));
  return 0;
}

namespace {

OzWork oz_work(ShardedCtx* sh) {
  OzWork w;
  w.s = sh->oz_s;
  w.RU = sh->RU;
  w.RX = sh->RX;
  w.RC = sh->RC;
  w.RC_bytes = sh->RC_bytes;
  w.eU = sh->eU;
  w.eU2 = sh->eU2;
  w.eX = sh->eX;
  w.part = sh->oz_part;
  return w;
}

// one modular product (T = 1) on the sharded handle's scratch
int oz_prod1(ShardedCtx* sh, int M, int N, int K, const int8_t* RA, const int* eA, int a_planes, const int8_t* RB,
             const int* eB, int b_planes, cplx* C, long long ldc, const cplx* base, int flags, const int32_t* kdev,
             const int32_t* ndev, std::string* err) {
  OzProduct p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.s = sh->oz_s;
  p.RA = RA;
  p.a_planes = a_planes;
  p.eA = eA;
  p.RB = RB;
  p.b_planes = b_planes;
  p.eB = eB;
  p.RC = sh->RC;
  p.C = C;
  p.ldc = ldc;
  p.base = base;
  p.flags = flags;
  p.kdev = kdev;
  p.ndev = ndev;
  if (a_planes == 4 && b_planes == 4) p.pb[2] = 3;   // C_SS: (re + im)(re - im)^T
  return oz_product(sh->st, p, err);
}

int gather_full(ShardedCtx* sh, int which, std::string* err) {
  std::vector<void*> send;
  for (auto& l : sh->loc) send.push_back(l.U[which]);
  return sh->comm.allgather(sh->st, send.data(), sh->Ufull, (size_t)sh->Lp * sh->ldN * 16, err);
}

// NCCL mode, planar: G = sum over ranks of U_g^dag U_g by column panels [c0, c1): the panel's Gram
// (three real products, rows [0, c1), upper tiles) on st, packed with its plane combine into a
// contiguous buffer, all-reduced in place and unpacked into G on gst while st computes the next
// panel -- the collective moves the upper part only (N^2/2 + N w/2 instead of N ldN entries) and runs
// under the Gram GEMMs (SURVEY §8(e) "pipeline the Gram by column panels")
int gram_panels(ShardedCtx* sh, int src, std::string* err) {
  ShardLocal& l = sh->loc[0];
  const long long psU = (long long)sh->Lp * sh->ldPs, psG = (long long)sh->N * sh->ldPs;
  const int N = sh->N, pw = sh->gram_pw;
  STRY(split6_planes(sh->st, l.U[src], sh->ldN, 0, sh->Lp, N, 1, l.Up6, sh->ldPs, psU, 0, err));
  int j = 0;
  for (int c0 = 0; c0 < N; c0 += pw, ++j) {
    const int c1 = std::min(N, c0 + pw), w = c1 - c0, q = j & 1;
    cplx* buf = sh->gpack + (size_t)q * N * pw;
    STRY(dgemm(sh->st, 1, c1, w, sh->Lp, 1.0, l.Up6, sh->ldPs, psU, l.Up6 + 3 * psU + c0, sh->ldPs, psU, 0.0,
               sh->Gp + c0, sh->ldPs, psG, 3, DG_C_UPPER, err, 0, c0));
    if (j >= 2) SCK(cudaStreamWaitEvent(sh->st, sh->ev_gfree[q], 0));   // the buffer's last panel is unpacked
    STRY(pack_gram_panel(sh->st, sh->Gp, sh->ldPs, psG, c0, c1, buf, w, err));
    SCK(cudaEventRecord(sh->ev_gpacked[q], sh->st));
    SCK(cudaStreamWaitEvent(sh->gst, sh->ev_gpacked[q], 0));
    double* pb = reinterpret_cast<double*>(buf);
    STRY(sh->comm.allreduce(sh->gst, &pb, pb, (size_t)c1 * w * 2, err));
    SCK(cudaMemcpy2DAsync(sh->G + c0, (size_t)sh->ldN * 16, buf, (size_t)w * 16, (size_t)w * 16, c1,
                          cudaMemcpyDeviceToDevice, sh->gst));
    SCK(cudaEventRecord(sh->ev_gfree[q], sh->gst));
  }
  SCK(cudaEventRecord(sh->ev_gdone, sh->gst));
  SCK(cudaStreamWaitEvent(sh->st, sh->ev_gdone, 0));
  return 0;
}

int allreduce_gram(ShardedCtx* sh, std::string* err) {
  std::vector<double*> part;
  for (auto& l : sh->loc) part.push_back(reinterpret_cast<double*>(l.Gpart));
  return sh->comm.allreduce(sh->st, part.data(), reinterpret_cast<double*>(sh->G), (size_t)sh->N * sh->ldN * 2, err);
}

// dst[:, a:b] = src[:, 0:b] X[0:b, a:b] for every local shard (X upper triangular) on stream q;
// planar: into the product planes (combined later), U's planes 3..5 already split
int trmm_cols(ShardedCtx* sh, int src, long long a, long long b, cudaStream_t q, std::string* err) {
  if (b <= a) return 0;
  if (sh->planar) {
    const long long psU = (long long)sh->Lp * sh->ldPs, psX = (long long)sh->N * sh->ldPs;
    STRY(split_planes(q, sh->X + a, sh->ldN, 0, (int)b, (int)(b - a), 1, sh->Xp + a, sh->ldPs, psX, 0, err));
    for (auto& l : sh->loc)
      STRY(dgemm(q, 0, sh->Lp, b - a, b, 1.0, l.Up6 + 3 * psU, sh->ldPs, psU, sh->Xp + a, sh->ldPs, psX, 0.0, l.Pp + a,
                 sh->ldPs, psU, 3, DG_TRI_B_UPPER, err, 0, a));
    return 0;
  }
  for (auto& l : sh->loc)
    STRY(zgemm(q, 0, 0, sh->Lp, b - a, b, 1.0, 0.0, l.U[src], sh->ldN, 0, sh->X + a, sh->ldN, 0, 0.0, l.U[1 - src] + a,
               sh->ldN, 0, 1, TRAJ_TRI_B_UPPER_F, err, 0, a));
  return 0;
}

// CholeskyQR2 of the distributed U (local blocks src[s]); tmp[s] the other buffers.
int cqr2(ShardedCtx* sh, int src_which, std::string* err) {
  int src = src_which;
  const int lr = sh->lr_k0;
  sh->lr_k0 = -1;
  const bool structured = sh->struct_pending;
  sh->struct_pending = false;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 0 && lr == 0) continue;     // no row zeroed: pass 1 has R = I
    if (pass == 0 && lr > 0 && structured) {
      // factor I - V^dag V from the replicated V (no collective), solve on each shard's rows
      Phase p(sh->prof, sh->st, TRAJ_PH_CHOL);
      sh->sc.kc = lr;
      // the solve on the INT8 modular path once k0's capacity is large (the unsharded rule); the
      // factor chain on the high-priority stream under the solve (TRAJ_STRUCT_PIPELINE=0: serial)
      const bool oz_apply = sh->oz && lr >= sh->oz_proj_min;
      const bool pipe = sh->chol_overlap && sh->st_hi && !sh->struct_serial;
      const int nblk = (int)ceil_div(sh->N, sh->sc.b);
      if (pipe) {
        while ((int)sh->sc_ev.size() < nblk) {
          cudaEvent_t e;
          SCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          sh->sc_ev.push_back(e);
        }
        SCK(cudaEventRecord(sh->ev_fork, sh->st));
        SCK(cudaStreamWaitEvent(sh->st_hi, sh->ev_fork, 0));
      }
      if (pipe && !oz_apply && sh->loc.size() == 1) {
        ShardLocal& l = sh->loc[0];
        STRY(struct_chol_pipelined(sh->st, sh->st_hi, sh->sc_ev.data(), (int)sh->sc_ev.size(), sh->sc, sh->USrecv,
                                   sh->ldN, 0, sh->k0, sh->failed_dev, sh->Lp, l.U[src], l.U[1 - src], sh->ldN, 0,
                                   l.Tm, sh->ldcap, 0, err));
      } else {
        {
          Phase pf(sh->prof, pipe ? sh->st_hi : sh->st, TRAJ_PH_STRUCT_FACTOR);
          if (pipe)
            STRY(struct_chol_factor_events(sh->st_hi, sh->sc, sh->USrecv, sh->ldN, 0, sh->k0, sh->failed_dev,
                                           sh->sc_ev.data(), err));
          else
            STRY(struct_chol_factor(sh->st, sh->sc, sh->USrecv, sh->ldN, 0, sh->k0, sh->failed_dev, err));
        }
        const OzWork w = oz_work(sh);
        for (auto& l : sh->loc) {
          if (oz_apply) {
            STRY(struct_chol_apply_oz(sh->st, sh->sc, w, sh->Lp, l.U[src], l.U[1 - src], sh->ldN, 0, l.Tm, sh->ldcap,
                                      0, sh->k0, pipe ? sh->sc_ev.data() : nullptr, err));
          } else {
            if (pipe) SCK(cudaStreamWaitEvent(sh->st, sh->sc_ev[nblk - 1], 0));
            STRY(struct_chol_apply(sh->st, sh->sc, sh->Lp, l.U[src], l.U[1 - src], sh->ldN, 0, l.Tm, sh->ldcap, 0,
                                   sh->k0, err));
          }
        }
      }
      src = 1 - src;
      continue;
    }
    if (!(pass == 0 && lr > 0)) {            // else pass 1's G = I - V^dag V is already set, replicated
      Phase p(sh->prof, sh->st, TRAJ_PH_GRAM);
      if (sh->comm.comm && sh->gpack && sh->gst) {
        STRY(gram_panels(sh, src, err));
        goto gram_done;
      }
      for (auto& l : sh->loc) {
        if (sh->oz) {
          // local G_g = U_g^dag U_g on the INT8 tensor cores (the unsharded step's modular Gram)
          STRY(oz_split_cols(sh->st, l.U[src], sh->ldN, 0, sh->Lp, sh->N, 1, 4, sh->oz_s, sh->RU, sh->eU, 0,
                             sh->oz_part, err));
          OzProduct p;
          p.M = sh->N;
          p.N = sh->N;
          p.K = sh->Lp;
          p.s = sh->oz_s;
          p.RA = sh->RU;
          p.a_planes = 4;
          p.pa[2] = 3;
          p.eA = sh->eU;
          p.RB = sh->RU;
          p.b_planes = 4;
          p.eB = sh->eU;
          p.RC = sh->RC;
          p.C = l.Gpart;
          p.ldc = sh->ldN;
          p.flags = OZ_UPPER | OZ_NEG_P2;
          {
            Phase pm(sh->prof, sh->st, TRAJ_PH_GRAM_MMA);
            STRY(oz_product_mma(sh->st, p, err));
          }
          STRY(oz_product_combine(sh->st, p, err));
        } else if (sh->planar) {
          // local G_g = U_g^dag U_g as three real products (planes re, im, re - im | re, im, re + im)
          const long long psU = (long long)sh->Lp * sh->ldPs, psG = (long long)sh->N * sh->ldPs;
          STRY(split6_planes(sh->st, l.U[src], sh->ldN, 0, sh->Lp, sh->N, 1, l.Up6, sh->ldPs, psU, 0, err));
          STRY(dgemm(sh->st, 1, sh->N, sh->N, sh->Lp, 1.0, l.Up6, sh->ldPs, psU, l.Up6 + 3 * psU, sh->ldPs, psU, 0.0,
                     sh->Gp, sh->ldPs, psG, 3, DG_C_UPPER, err));
          STRY(combine_gram(sh->st, sh->Gp, sh->ldPs, psG, 0, sh->N, 1, l.Gpart, sh->ldN, 0, err));
        } else {
          STRY(zgemm(sh->st, 1, 0, sh->N, sh->N, sh->Lp, 1.0, 0.0, l.U[src], sh->ldN, 0, l.U[src], sh->ldN, 0, 0.0,
                     l.Gpart, sh->ldN, 0, 1, TRAJ_C_UPPER_F, err));
        }
      }
      STRY(allreduce_gram(sh, err));
    }
  gram_done:
    {
      Phase p(sh->prof, sh->st, TRAJ_PH_CHOL);
      const bool full = pass == 0 || sh->full_cqr2;
      if (!full) {
        // decided on the device from the all-reduced G2 (the same bits on every rank): the
        // first-order factor, overwritten by the gated full factorisation when it is needed
        // (replicated, not distributed: a gated-off step must not move the Cholesky's broadcasts)
        const double thr = 1e-9 / sqrt((double)sh->N);
        STRY(gram_deviation(sh->st, sh->G, sh->ldN, 0, sh->N, 1, sh->gdev, err));
        STRY(first_order_inverse(sh->st, sh->G, sh->ldN, 0, sh->X, sh->ldN, 0, sh->N, 1, err));
        if (sh->fbg_state == 0) {
          const char* fg = getenv("TRAJ_FALLBACK_GRAPH");
          std::string e2;
          sh->fbg_state = (fg && fg[0] == '0') || sh->fbg.build(sh->N, sh->G, sh->ldN, 0, sh->X, sh->ldN, 0, 1,
                                                                 sh->chol_scratch, sh->failed_dev, sh->gdev, thr,
                                                                 sh->fb_dev, &e2) ? -1 : 1;
        }
        if (sh->fbg_state == 1) {
          // the modular TRMM below keys its full-precision product on the same decision (gate)
          if (sh->oz) STRY(cqr2_decide(sh->st, sh->gdev, 1, thr, sh->gate, nullptr, err));
          STRY(sh->fbg.launch(sh->st, err));
        } else {
          STRY(cqr2_decide(sh->st, sh->gdev, 1, thr, sh->gate, sh->fb_dev, err));
          STRY(chol_inverse(sh->st, sh->N, sh->G, sh->ldN, 0, sh->X, sh->ldN, 0, 1, sh->chol_scratch,
                            sh->failed_dev, err, nullptr, nullptr, sh->gate));
        }
      }
      if (full && pass == 0 && sh->chol_overlap && sh->N > 64 && !sh->oz) {
        // factorise on st_hi; each newly final left column block's TRMM runs on st_lo
        SCK(cudaEventRecord(sh->ev_fork, sh->st));
        SCK(cudaStreamWaitEvent(sh->st_hi, sh->ev_fork, 0));
        SCK(cudaStreamWaitEvent(sh->st_lo, sh->ev_fork, 0));
        const long long psU = (long long)sh->Lp * sh->ldPs;
        if (sh->planar && lr > 0)   // pass 1's Gram was not measured: U's (re, im, re + im) planes
          for (auto& l : sh->loc)
            STRY(split_planes(sh->st_lo, l.U[src], sh->ldN, 0, sh->Lp, sh->N, 1, l.Up6 + 3 * psU, sh->ldPs, psU, 0,
                              err));
        struct HookUser {
          ShardedCtx* sh;
          int src;
          long long hs;
          int status;
          std::string* err;
        } hu{sh, src, 0, 0, err};
        CholHook hook;
        hook.user = &hu;
        hook.left_ready = [](void* u, long long hs) {
          HookUser* q = reinterpret_cast<HookUser*>(u);
          ShardedCtx* s2 = q->sh;
          if (q->status || hs <= q->hs) return;
          const long long a = q->hs;
          q->hs = hs;
          if (cudaEventRecord(s2->ev_left, s2->st_hi) != cudaSuccess ||
              cudaStreamWaitEvent(s2->st_lo, s2->ev_left, 0) != cudaSuccess) {
            q->status = TRAJ_ECUDA;
            return;
          }
          q->status = trmm_cols(s2, q->src, a, hs, s2->st_lo, q->err);
        };
        STRY(chol_inverse(sh->st_hi, sh->N, sh->G, sh->ldN, 0, sh->X, sh->ldN, 0, 1, sh->chol_scratch, sh->failed_dev,
                          err, &sh->cdist, &hook));
        if (hu.status) return hu.status;
        SCK(cudaEventRecord(sh->ev_lo_done, sh->st_lo));
        SCK(cudaStreamWaitEvent(sh->st_hi, sh->ev_lo_done, 0));   // the U planes / pieces before the right part
        STRY(trmm_cols(sh, src, hu.hs, sh->N, sh->st_hi, err));
        SCK(cudaEventRecord(sh->ev_hi_done, sh->st_hi));
        SCK(cudaStreamWaitEvent(sh->st, sh->ev_hi_done, 0));
        if (sh->planar)
          for (auto& l : sh->loc)
            STRY(combine_planes(sh->st, l.Pp, sh->ldPs, psU, 0, sh->Lp, sh->N, 1, l.U[1 - src], sh->ldN, 0, err));
        src = 1 - src;
        continue;   // this pass's TRMM is done (inside the Cholesky phase)
      }
      if (full)
        STRY(chol_inverse(sh->st, sh->N, sh->G, sh->ldN, 0, sh->X, sh->ldN, 0, 1, sh->chol_scratch, sh->failed_dev,
                          err, &sh->cdist));
    }
    {
      Phase p(sh->prof, sh->st, TRAJ_PH_TRMM);
      if (sh->oz) {
        // U_g X on the INT8 tensor cores (the unsharded step's modular TRMM): after the first-order
        // second-pass factor X = I + D, U_g + U_g D at oz_s_corr moduli, overwritten by the full
        // product when the device decided on the full factorisation (gate)
        const bool corr = pass == 1 && !sh->full_cqr2 && sh->oz_s_corr > 0;
        for (int full = corr ? 0 : 1; full < 2; ++full) {
          const int q = full ? sh->oz_s : sh->oz_s_corr;
          const int32_t* gate = corr && full ? sh->gate : nullptr;
          STRY(oz_split_cols(sh->st, sh->X, sh->ldN, 0, sh->N, sh->N, 1, 3, q, sh->RX, sh->eX, 0, sh->oz_part, err,
                             full ? 0 : 1, gate));
          for (auto& l : sh->loc) {
            STRY(oz_split_rows(sh->st, l.U[src], sh->ldN, 0, sh->Lp, sh->N, 1, 0, q, sh->RU, sh->eU, 0, err, gate));
            OzProduct op;
            op.M = sh->Lp;
            op.N = sh->N;
            op.K = sh->N;
            op.s = q;
            op.RA = sh->RU;
            op.eA = sh->eU;
            op.RB = sh->RX;
            op.eB = sh->eX;
            op.RC = sh->RC;
            op.C = l.U[1 - src];
            op.ldc = sh->ldN;
            op.flags = OZ_TRI_B;
            op.base = full ? nullptr : l.U[src];
            op.gate = gate;
            {
              Phase pm(sh->prof, sh->st, TRAJ_PH_TRMM_MMA);
              STRY(oz_product_mma(sh->st, op, err));
            }
            STRY(oz_product_combine(sh->st, op, err));
          }
        }
      } else if (sh->planar) {
        // U_g X as three real products on the Gram's planes of U_g and X's planes
        const long long psU = (long long)sh->Lp * sh->ldPs, psX = (long long)sh->N * sh->ldPs;
        STRY(split_planes(sh->st, sh->X, sh->ldN, 0, sh->N, sh->N, 1, sh->Xp, sh->ldPs, psX, 0, err));
        for (auto& l : sh->loc) {
          if (pass == 0 && lr > 0)   // no measured Gram split U this pass: its (re, im, re + im) planes
            STRY(split_planes(sh->st, l.U[src], sh->ldN, 0, sh->Lp, sh->N, 1, l.Up6 + 3 * psU, sh->ldPs, psU, 0, err));
          STRY(dgemm(sh->st, 0, sh->Lp, sh->N, sh->N, 1.0, l.Up6 + 3 * psU, sh->ldPs, psU, sh->Xp, sh->ldPs, psX, 0.0,
                     l.Pp, sh->ldPs, psU, 3, DG_TRI_B_UPPER, err));
          STRY(combine_planes(sh->st, l.Pp, sh->ldPs, psU, 0, sh->Lp, sh->N, 1, l.U[1 - src], sh->ldN, 0, err));
        }
      } else {
        for (auto& l : sh->loc)
          STRY(zgemm(sh->st, 0, 0, sh->Lp, sh->N, sh->N, 1.0, 0.0, l.U[src], sh->ldN, 0, sh->X, sh->ldN, 0, 0.0,
                     l.U[1 - src], sh->ldN, 0, 1, TRAJ_TRI_B_UPPER_F, err));
      }
    }
    src = 1 - src;
  }
  if (src != src_which)   // one pass ran: move the result back into src_which
    for (auto& l : sh->loc)
      SCK(cudaMemcpyAsync(l.U[src_which], l.U[src], (size_t)sh->Lp * sh->ldN * 16, cudaMemcpyDeviceToDevice, sh->st));
  return 0;   // the result is in src_which
}

int projective(ShardedCtx* sh, int which, long long step, std::string* err) {
  Phase p(sh->prof, sh->st, TRAJ_PH_PROJECT);
  cudaStream_t st = sh->st;
  const int capr = sh->capr, P = sh->P;
  // per-shard click counts on the host (the device's click_draw makes the same counter-based
  // decisions): they size every launch below, so the step needs no host round trip
  sh->hcnt.assign(P, 0);
  for (int q = 0; q < P; ++q)
    host_click_counts(sh->Lp, 1, step, sh->traj_base, sh->seed, &sh->gamma, sh->dt, &sh->hcnt[q], q * sh->Lp);
  int total = 0;
  for (int q = 0; q < P; ++q) {
    if (sh->hcnt[q] > capr) {
      if (err) *err = "click list overflow on shard " + std::to_string(q);
      return TRAJ_ENUMERIC;
    }
    total += sh->hcnt[q];
  }
  sh->last_nS = total;
  sh->last_n1 = 0;
  sh->k1_dev = false;
  if (total == 0) {
    if (sh->lowrank_gram) sh->lr_k0 = 0;     // U = K U is orthonormal: pass 1 has R = I
    return 0;
  }
  for (auto& l : sh->loc) {
    STRY(compact(st, l.flags, sh->Lp, 1, l.Sloc, capr, l.cnt, err, l.row0));
    STRY(gather_rows(st, l.U[which], sh->ldN, 0, l.Sloc, 0, l.cnt, capr, 1, l.USloc, sh->ldN, 0, sh->N, err, l.row0));
  }
  {
    std::vector<void*> b, c;
    for (auto& l : sh->loc) {
      b.push_back(l.Sloc);
      c.push_back(l.USloc);
    }
    STRY(sh->comm.allgather(st, b.data(), sh->Srecv, (size_t)capr * 4, err));
    STRY(sh->comm.allgather(st, c.data(), sh->USrecv, (size_t)capr * sh->ldN * 16, err));
  }
  // pack the per-shard blocks (shard order = ascending sites) into S and U_S
  int off = 0;
  for (int q = 0; q < P; ++q) {
    const int cq = sh->hcnt[q];
    if (cq == 0) continue;
    SCK(cudaMemcpyAsync(sh->S + off, sh->Srecv + (size_t)q * capr, cq * 4, cudaMemcpyDeviceToDevice, st));
    SCK(cudaMemcpyAsync(sh->US + (size_t)off * sh->ldN, sh->USrecv + (size_t)q * capr * sh->ldN,
                        (size_t)cq * sh->ldN * 16, cudaMemcpyDeviceToDevice, st));
    off += cq;
  }
  // the total on the device: the local counts of every shard are the host's (same draws)
  {
    std::vector<void*> a;
    for (auto& l : sh->loc) a.push_back(l.cnt);
    STRY(sh->comm.allgather(st, a.data(), sh->cntrecv, 4, err));
    STRY(sum_i32(st, sh->cntrecv, P, sh->count, err));
  }
  // C_SS = U_S U_S^dag: with an NCCL communicator each rank computes a slice of its rows and one
  // in-place allgather replicates it (the sampling and W below stay replicated); else replicated
  const int sr = (total + P - 1) / P;
  // the rank-k products on the INT8 modular path once the click count makes them large (the
  // unsharded rule, TRAJ_OZAKI_PROJ_MIN)
  const bool ozp = sh->oz && total >= sh->oz_proj_min && total <= sh->N;
  const char* css = getenv("TRAJ_SHARD_CSS_SPLIT");   // =0: replicated C_SS
  if (sh->comm.comm && P > 1 && (long long)sr * P <= sh->cap && !(css && css[0] == '0')) {
    const int me = sh->comm.rank0, r0 = me * sr, nr = std::max(0, std::min(sr, total - r0));
    if (nr > 0)
      STRY(zgemm(st, 0, 1, nr, total, sh->N, 1.0, 0.0, sh->US + (size_t)r0 * sh->ldN, sh->ldN, 0, sh->US, sh->ldN, 0,
                 0.0, sh->D0 + (size_t)r0 * sh->ldcap, sh->ldcap, 0, 1, 0, err));
    void* mine = sh->D0 + (size_t)r0 * sh->ldcap;
    STRY(sh->comm.allgather(st, &mine, sh->D0, (size_t)sr * sh->ldcap * 16, err));
  } else if (ozp) {
    // replicated C_SS on the INT8 modular path: one 4-plane row split of U_S serves both sides
    // (P1 = re re^T, P2' = im im^T, P3 = (re + im)(re - im)^T, OZ_NEG_P2)
    STRY(oz_split_rows(st, sh->US, sh->ldN, 0, total, sh->N, 1, 0, sh->oz_s, sh->RU, sh->eU, 0, err, nullptr, nullptr,
                       4));
    STRY(oz_prod1(sh, total, total, sh->N, sh->RU, sh->eU, 4, sh->RU, sh->eU, 4, sh->D0, sh->ldcap, nullptr,
                  OZ_NEG_P2, nullptr, nullptr, err));
  } else {
    STRY(zgemm(st, 0, 1, total, total, sh->N, 1.0, 0.0, sh->US, sh->ldN, 0, sh->US, sh->ldN, 0, 0.0, sh->D0,
               sh->ldcap, 0, 1, 0, err));
  }
  STRY(sample_outcomes(st, sh->D0, sh->Dw, sh->ldcap, 0, sh->S, sh->cap, sh->count, total, 1, step, sh->traj_base,
                       sh->seed, sh->occ, sh->Linv, sh->DLinv, sh->Ybuf, sh->Zbuf, sh->ldcap, sh->pos1, sh->S1, sh->S0,
                       sh->k1, sh->k0, err, sh->pos0));
  sh->k1_dev = true;
  if (getenv("TRAJ_DEBUG_SHARD")) {   // debugging aid: the device counts of this step
    int32_t v[4] = {0, 0, 0, 0};
    cudaMemcpyAsync(v, sh->count, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(v + 1, sh->k1, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(v + 2, sh->k0, 4, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[shard] step %lld: host total %d, device count %d, k1 %d, k0 %d\n", step, total, v[0], v[1], v[2]);
  }
  // k1, k0 stay on the device: launches sized by the click count `total`, bounded there (zgemm.h
  // DevBounds; identity past k1 in C_{S1 S1}, zero rows past k1 / k0 in the gathered blocks)
  DevBounds b1, bk, b0;
  b1.n = sh->k1;
  b1.k = sh->k1;
  bk.k = sh->k1;
  b0.k = sh->k0;
  STRY(gather_sub_batched(st, sh->D0, sh->ldcap, 0, sh->pos1, sh->cap, sh->k1, total, 1, sh->D11, sh->ldcap, 0, err));
  STRY(chol_inverse(st, total, sh->D11, sh->ldcap, 0, sh->X11, sh->ldcap, 0, 1, sh->chol_scratch_small, sh->failed_dev,
                    err));
  // U_{S1} = rows pos1 of U_S (into USrecv, free now; zero past k1)
  STRY(gather_rows(st, sh->US, sh->ldN, 0, sh->pos1, 0, sh->k1, total, 1, sh->USrecv, sh->ldN, 0, sh->N, err, 0, 1));
  STRY(zgemm(st, 1, 0, sh->N, total, total, 1.0, 0.0, sh->USrecv, sh->ldN, 0, sh->X11, sh->ldcap, 0, 0.0, sh->W,
             sh->ldcap, 0, 1, TRAJ_TRI_B_UPPER_F, err, 0, 0, &b1));
  if (ozp) {
    // per shard Tm = U_g W (columns < k1: W's columns past k1 taken as zero), then
    // U_g <- U_g - Tm W^dag over k < k1, on the INT8 modular path; W's column residues for the
    // first product are shared by the shards, its conjugated row residues for the second likewise
    // (RX holds one at a time: the shards' first products, then their second ones)
    STRY(oz_split_cols(st, sh->W, sh->ldcap, 0, sh->N, total, 1, 3, sh->oz_s, sh->RX, sh->eX, 0, sh->oz_part, err, 0,
                       nullptr, sh->k1));
    for (auto& l : sh->loc) {
      STRY(oz_split_rows(st, l.U[which], sh->ldN, 0, sh->Lp, sh->N, 1, 0, sh->oz_s, sh->RU, sh->eU, 0, err));
      STRY(oz_prod1(sh, sh->Lp, total, sh->N, sh->RU, sh->eU, 3, sh->RX, sh->eX, 3, l.Tm, sh->ldcap, nullptr, 0,
                    nullptr, sh->k1, err));
      STRY(sub_identity(st, l.Tm, sh->ldcap, sh->S1, total, err, l.row0, sh->Lp, sh->k1));
    }
    if (sh->lowrank_gram) {   // pass 1's V (below), first product: D11 = U_S0 W (replicated rows)
      STRY(gather_rows(st, sh->US, sh->ldN, 0, sh->pos0, 0, sh->k0, total, 1, sh->USrecv, sh->ldN, 0, sh->N, err, 0,
                       1));
      STRY(oz_split_rows(st, sh->USrecv, sh->ldN, 0, total, sh->N, 1, 0, sh->oz_s, sh->RU, sh->eU, 0, err));
      STRY(oz_prod1(sh, total, total, sh->N, sh->RU, sh->eU, 3, sh->RX, sh->eX, 3, sh->D11, sh->ldcap, nullptr, 0,
                    nullptr, sh->k1, err));
    }
    STRY(oz_split_rows(st, sh->W, sh->ldcap, 0, sh->N, total, 1, 1, sh->oz_s, sh->RX, sh->eX, 0, err, nullptr,
                       sh->k1));
    for (auto& l : sh->loc) {
      STRY(oz_split_rows(st, l.Tm, sh->ldcap, 0, sh->Lp, total, 1, 0, sh->oz_s, sh->RU, sh->eU, 0, err, nullptr,
                         sh->k1));
      STRY(oz_prod1(sh, sh->Lp, sh->N, total, sh->RU, sh->eU, 3, sh->RX, sh->eX, 3, l.U[which], sh->ldN, l.U[which],
                    OZ_NEGATE, sh->k1, nullptr, err));
    }
    if (sh->lowrank_gram) {   // V = U_S0 - D11 W^dag
      STRY(oz_split_rows(st, sh->D11, sh->ldcap, 0, total, total, 1, 0, sh->oz_s, sh->RU, sh->eU, 0, err, nullptr,
                         sh->k1));
      STRY(oz_prod1(sh, total, sh->N, total, sh->RU, sh->eU, 3, sh->RX, sh->eX, 3, sh->USrecv, sh->ldN, sh->USrecv,
                    OZ_NEGATE, sh->k1, nullptr, err));
    }
  } else {
    for (auto& l : sh->loc) {
      DevBounds bn;
      bn.n = sh->k1;
      STRY(zgemm(st, 0, 0, sh->Lp, total, sh->N, 1.0, 0.0, l.U[which], sh->ldN, 0, sh->W, sh->ldcap, 0, 0.0, l.Tm,
                 sh->ldcap, 0, 1, 0, err, 0, 0, &bn));
      STRY(sub_identity(st, l.Tm, sh->ldcap, sh->S1, total, err, l.row0, sh->Lp, sh->k1));
      STRY(zgemm(st, 0, 1, sh->Lp, sh->N, total, -1.0, 0.0, l.Tm, sh->ldcap, 0, sh->W, sh->ldcap, 0, 1.0, l.U[which],
                 sh->ldN, 0, 1, 0, err, 0, 0, &bk));
    }
  }
  for (auto& l : sh->loc) STRY(zero_rows(st, l.U[which], sh->ldN, sh->S0, total, sh->N, err, l.row0, sh->Lp, sh->k0));
  if (sh->lowrank_gram) {
    // U was orthonormal before the rows S0 were zeroed, so pass 1's Gram is I - V^dag V with V the
    // zeroed rows after the rank-k1 update: V = U_S0 - (U_S0 W) W^dag from the gathered rows (replicated)
    // (on the modular path V was formed with the rank-k update above)
    DevBounds bn;
    bn.n = sh->k1;
    if (!ozp) {
      STRY(gather_rows(st, sh->US, sh->ldN, 0, sh->pos0, 0, sh->k0, total, 1, sh->USrecv, sh->ldN, 0, sh->N, err, 0,
                       1));
      STRY(zgemm(st, 0, 0, total, total, sh->N, 1.0, 0.0, sh->USrecv, sh->ldN, 0, sh->W, sh->ldcap, 0, 0.0, sh->D11,
                 sh->ldcap, 0, 1, 0, err, 0, 0, &bn));
      STRY(zgemm(st, 0, 1, total, sh->N, total, -1.0, 0.0, sh->D11, sh->ldcap, 0, sh->W, sh->ldcap, 0, 1.0,
                 sh->USrecv, sh->ldN, 0, 1, 0, err, 0, 0, &bk));
    }
    sh->lr_k0 = total;
    if (sh->struct_chol && 2LL * total <= sh->N) {   // pass 1 on the structure of I - V^dag V (V in USrecv)
      sh->struct_pending = true;
      return 0;
    }
    STRY(set_identity(st, sh->G, sh->ldN, 0, sh->N, 1, err));
    STRY(zgemm(st, 1, 0, sh->N, sh->N, total, -1.0, 0.0, sh->USrecv, sh->ldN, 0, sh->USrecv, sh->ldN, 0, 1.0, sh->G,
               sh->ldN, 0, 1, TRAJ_C_UPPER_F, err, 0, 0, &b0));
    sh->lr_k0 = total;
  }
  return 0;
}

// NEXT-1 with sharding: 1d -- halo of W rows from each neighbour, one non-periodic pass;
// 2d -- the x pass is local (whole lattice rows per shard), then a halo of W*Lx rows for the
// y pass.  Uext = [H halo rows | Lp local rows | H halo rows].
int propagate_banded(ShardedCtx* sh, int cur, int nxt, std::string* err) {
  cudaStream_t st = sh->st;
  const long long H = sh->H, Lp = sh->Lp, ld = sh->ldN;
  const bool twod = sh->Ly > 1;
  std::vector<void*> slo, shi, rlo, rhi;
  for (auto& l : sh->loc) {
    cplx* mid = l.Uext + H * ld;
    if (twod) {
      STRY(banded_pass(st, l.U[cur], mid, ld, 0, sh->N, 1, sh->Lx, (int)(Lp / sh->Lx), sh->Lx, 1, sh->band_host.data(), sh->Wx,
                       err));
    } else {
      SCK(cudaMemcpyAsync(mid, l.U[cur], (size_t)Lp * ld * 16, cudaMemcpyDeviceToDevice, st));
    }
    slo.push_back(mid);
    shi.push_back(mid + (Lp - H) * ld);
    rlo.push_back(l.Uext);
    rhi.push_back(mid + Lp * ld);
  }
  STRY(sh->comm.halo(st, slo.data(), shi.data(), rlo.data(), rhi.data(), (size_t)H * ld * 16, err));
  for (auto& l : sh->loc) {
    if (twod)
      STRY(banded_pass(st, l.Uext, l.U[nxt], ld, 0, sh->N, 1, (int)(Lp / sh->Lx), sh->Lx, 1, sh->Lx,
                       sh->band_host.data() + 2 * sh->Wx + 1, sh->Wy, err, 0));
    else
      STRY(banded_pass(st, l.Uext, l.U[nxt], ld, 0, sh->N, 1, (int)Lp, 1, 0, 1, sh->band_host.data(), sh->Wx, err, 0));
  }
  return 0;
}

// a1 with sharding, SURVEY §8(e) "fusion with the collective": U_g' = sum_s K_g[:, s] U_s over
// the P row blocks s of U, in ring-distance order d = 0..P-1 (s = g - d mod P).  d = 0 is the
// local block and starts at once; in NCCL mode block d arrives by a send/recv pair on the comm
// stream (send U_g to g + d, receive U_{g-d}) and its GEMM waits only for that transfer, so
// the exchange of block d+1 runs under the GEMM of block d.  The emulation (one GPU) gathers
// first and then runs the same chunk GEMMs in the same order (the same arithmetic).
// TRAJ_SHARD_OVERLAP=0: one allgather, then one L-deep GEMM.
// planar 3M chunk: P_q (+)= K_g[:, s]_q U_s,q for the three products (one batch-3 launch), U_s split
// into (re, im, re + im) planes first
int planar_chunk(ShardedCtx* sh, ShardLocal& l, const cplx* Us, int s, bool accumulate, std::string* err,
                 int nxt = -1) {
  const long long Lp = sh->Lp, psC = Lp * sh->ldPs;
  if (sh->slv) {
    // Strassen on the chunk product K_g[:, s] U_s, accumulated into U_g' directly by the recombination
    const int np = strassen_products(sh->slv);
    const long long hh = Lp >> sh->slv, nh = sh->N >> sh->slv, bK = hh * sh->ldS, bM = hh * sh->ldSM;
    STRY(strassen_b(sh->st, sh->slv, Us, sh->ldN, 0, (int)Lp, sh->N, 1, sh->Sb, sh->ldSM, err));
    STRY(dgemm(sh->st, 0, hh, nh, hh, 1.0, l.Ks + s * np * bK, sh->ldS, bK, sh->Sb, sh->ldSM, bM, 0.0, sh->Sm,
               sh->ldSM, bM, np, 0, err));
    return strassen_c(sh->st, sh->slv, sh->Sm, sh->ldSM, (int)Lp, sh->N, 1, l.U[nxt], sh->ldN, 0, err,
                      accumulate ? 1 : 0);
  }
  STRY(split_planes(sh->st, Us, sh->ldN, 0, (int)Lp, sh->N, 1, sh->Cp, sh->ldPs, psC, 0, err));
  return dgemm(sh->st, 0, Lp, sh->N, Lp, 1.0, l.Kp + (long long)s * Lp, sh->ldKs, Lp * sh->ldKs, sh->Cp, sh->ldPs, psC,
               accumulate ? 1.0 : 0.0, l.Pp, sh->ldPs, psC, 3, 0, err);
}

int planar_finish(ShardedCtx* sh, ShardLocal& l, int nxt, std::string* err) {
  if (sh->slv) return 0;   // the Strassen recombination wrote U_g' already
  const long long psC = (long long)sh->Lp * sh->ldPs;
  return combine_planes(sh->st, l.Pp, sh->ldPs, psC, 0, sh->Lp, sh->N, 1, l.U[nxt], sh->ldN, 0, err);
}

// modular K_g U: the GLOBAL column exponents of U (column norms summed over the shards: one N-double
// allreduce), so that every chunk's residues U_s share one scale and their products add mod m_q
int oz_global_exponents(ShardedCtx* sh, int cur, std::string* err) {
  int i = 0;
  for (auto& l : sh->loc)
    STRY(oz_colnorm_accumulate(sh->st, l.U[cur], sh->ldN, 0, sh->Lp, sh->N, 1, sh->oz_part, sh->nu2, 0, i++ > 0,
                               err));
  if (sh->comm.comm && sh->P > 1) STRY(sh->comm.allreduce(sh->st, &sh->nu2, sh->nu2, (size_t)sh->N, err));
  return oz_exponents(sh->st, sh->nu2, 0, sh->N, 1, sh->oz_s, sh->eG, 0, err);
}

OzProduct oz_ku(ShardedCtx* sh, ShardLocal& l, int nxt) {
  OzProduct p;
  p.M = sh->Lp;
  p.N = sh->N;
  p.K = sh->Lp;
  p.T = 1;
  p.s = sh->oz_s;
  p.RA = l.RK;
  p.a_traj = 0;
  p.eA = l.eK;
  p.RB = sh->RU;
  p.eB = sh->eG;
  p.RC = sh->RC;
  p.C = l.U[nxt];
  p.ldc = sh->ldN;
  p.lda_override = oz_ld(sh->L);
  return p;
}

// residues of K_g[:, s] U_s (+)= into RC: U_s's column residues at the global exponents, K_g's
// row residues from byte s Lp of each row
int oz_chunk(ShardedCtx* sh, ShardLocal& l, const cplx* Us, int s, bool accumulate, int nxt, std::string* err) {
  STRY(oz_split_cols_e(sh->st, Us, sh->ldN, 0, sh->Lp, sh->N, 1, 3, sh->oz_s, sh->RU, sh->eG, 0, err));
  OzProduct p = oz_ku(sh, l, nxt);
  p.RA = l.RK + (long long)s * sh->Lp;
  p.mma_accumulate = accumulate ? 1 : 0;
  Phase pm(sh->prof, sh->st, TRAJ_PH_KU_MMA);
  return oz_product_mma(sh->st, p, err);
}

int propagate_dense(ShardedCtx* sh, int cur, int nxt, std::string* err) {
  cudaStream_t st = sh->st;
  const long long Lp = sh->Lp, ld = sh->ldN;
  const size_t bytes = (size_t)Lp * ld * 16;
  if (sh->oz) STRY(oz_global_exponents(sh, cur, err));
  if (sh->oz && !sh->oz_chunked) {
    // the gathered U's column residues once, then ONE product K_g U per shard over k = L: the P
    // chunk products of depth Lp run the INT8 pipe ~3x below it at P = 8 (each tile's epilogue
    // against 16 k-blocks), more than the exchange they would hide
    if (sh->P > 1) STRY(gather_full(sh, cur, err));
    const cplx* Uf = sh->P > 1 ? sh->Ufull : sh->loc[0].U[cur];
    STRY(oz_split_cols_e(st, Uf, ld, 0, sh->L, sh->N, 1, 3, sh->oz_s, sh->RU, sh->eG, 0, err));
    for (auto& l : sh->loc) {
      OzProduct p = oz_ku(sh, l, nxt);
      p.K = sh->L;
      {
        Phase pm(sh->prof, st, TRAJ_PH_KU_MMA);
        STRY(oz_product_mma(st, p, err));
      }
      STRY(oz_product_combine(st, p, err));
    }
    return 0;
  }
  if ((sh->planar || sh->oz) && !(sh->comm.comm && sh->overlap && sh->P > 1)) {
    // gathered first (emulation, one shard, or TRAJ_SHARD_OVERLAP=0), then the chunk products
    if (sh->P > 1) STRY(gather_full(sh, cur, err));
    for (auto& l : sh->loc) {
      for (int d = 0; d < sh->P; ++d) {
        const int s = (l.g - d + sh->P) % sh->P;
        const cplx* Us = sh->P > 1 ? sh->Ufull + (size_t)s * Lp * ld : l.U[cur];
        if (sh->oz) STRY(oz_chunk(sh, l, Us, s, d > 0, nxt, err));
        else STRY(planar_chunk(sh, l, Us, s, d > 0, err, nxt));
      }
      if (sh->oz) STRY(oz_product_combine(st, oz_ku(sh, l, nxt), err));
      else STRY(planar_finish(sh, l, nxt, err));
    }
    return 0;
  }
  if (!sh->overlap || sh->P == 1) {
    STRY(gather_full(sh, cur, err));
    for (auto& l : sh->loc)
      STRY(zgemm(st, 0, 0, Lp, sh->N, sh->L, 1.0, 0.0, l.K, sh->ldL, 0, sh->Ufull, ld, 0, 0.0, l.U[nxt], ld, 0, 1, 0,
                 err));
    return 0;
  }
  const int P = sh->P;
  if (sh->comm.comm) {
    ShardLocal& l = sh->loc[0];
    const int g = l.g;
    SCK(cudaEventRecord(sh->ev_start, st));
    SCK(cudaStreamWaitEvent(sh->cst, sh->ev_start, 0));
    // comm_plan.h ring_plan: group d - 1 sends U_g to g + d and receives U_{g-d}; the K-chunk
    // product of distance d waits for that group only
    const std::vector<CommOp> plan = ring_plan(P, g);
    for (size_t q = 0; q < plan.size();) {
      const int grp = plan[q].group;
      STRY(sh->comm.begin(err));
      ncclGroupStart();
      for (; q < plan.size() && plan[q].group == grp; ++q) {
        const CommOp& op = plan[q];
        if (op.kind == COMM_SEND) ncclSend(l.U[cur], bytes, ncclUint8, op.peer, sh->comm.comm, sh->cst);
        else ncclRecv(sh->Ufull + (size_t)op.block * Lp * ld, bytes, ncclUint8, op.peer, sh->comm.comm, sh->cst);
      }
      ncclResult_t r = ncclGroupEnd();
      sh->comm.end(sh->cst);
      if (r != ncclSuccess) {
        if (err) *err = std::string("nccl send/recv (propagate): ") + ncclGetErrorString(r);
        return TRAJ_ENCCL;
      }
      SCK(cudaEventRecord(sh->ev_chunk[grp + 1], sh->cst));
    }
    for (int d = 0; d < P; ++d) {
      const int s = (g - d + P) % P;
      const cplx* Us = l.U[cur];
      if (d > 0) {
        SCK(cudaStreamWaitEvent(st, sh->ev_chunk[d], 0));
        Us = sh->Ufull + (size_t)s * Lp * ld;
      }
      if (sh->oz) STRY(oz_chunk(sh, l, Us, s, d > 0, nxt, err));
      else if (sh->planar) STRY(planar_chunk(sh, l, Us, s, d > 0, err, nxt));
      else
        STRY(zgemm(st, 0, 0, Lp, sh->N, Lp, 1.0, 0.0, l.K + (size_t)s * Lp, sh->ldL, 0, Us, ld, 0, d ? 1.0 : 0.0,
                   l.U[nxt], ld, 0, 1, 0, err));
    }
    if (sh->oz) STRY(oz_product_combine(st, oz_ku(sh, l, nxt), err));
    else if (sh->planar) STRY(planar_finish(sh, l, nxt, err));
    return 0;
  }
  STRY(gather_full(sh, cur, err));
  for (auto& l : sh->loc)
    for (int d = 0; d < P; ++d) {
      const int s = (l.g - d + P) % P;
      STRY(zgemm(st, 0, 0, Lp, sh->N, Lp, 1.0, 0.0, l.K + (size_t)s * Lp, sh->ldL, 0, sh->Ufull + (size_t)s * Lp * ld,
                 ld, 0, d ? 1.0 : 0.0, l.U[nxt], ld, 0, 1, 0, err));
    }
  return 0;
}

}  // namespace

int shard_step(ShardedCtx* sh, long long* step, std::string* err) {
  STRY(sh->comm.wd.check(err));
  if (sh->test_stall) {   // test hook: a "collective" that never completes, and nothing behind it
    STRY(sh->comm.wd.stall(sh->st, err));
    return sh->comm.wd.mark(sh->st, err);
  }
  return shard_step_impl(sh, step, err);
}

int shard_step_impl(ShardedCtx* sh, long long* step, std::string* err) {
  const int cur = sh->cur, nxt = 1 - sh->cur;
  if (sh->banded) {
    Phase p(sh->prof, sh->st, TRAJ_PH_PROPAGATE);
    STRY(propagate_banded(sh, cur, nxt, err));
  } else {
    Phase p(sh->prof, sh->st, TRAJ_PH_PROPAGATE);
    STRY(propagate_dense(sh, cur, nxt, err));
  }
  {
    Phase p(sh->prof, sh->st, TRAJ_PH_MONITOR);
    for (auto& l : sh->loc) {
      if (sh->protocol == TRAJ_HOMODYNE)
        STRY(row_monitor(sh->st, l.U[nxt], sh->ldN, 0, sh->Lp, sh->N, 1, 1, *step, sh->traj_base, sh->seed,
                         sh->gamma_dev, sh->dt, nullptr, err, l.row0));
      else
        STRY(click_draw(sh->st, sh->Lp, 1, *step, sh->traj_base, sh->seed, sh->gamma_dev, sh->dt, l.flags, err,
                        l.row0));
    }
  }
  if (sh->protocol == TRAJ_PROJECTIVE) STRY(projective(sh, nxt, *step, err));
  STRY(cqr2(sh, nxt, err));
  sh->cur = nxt;
  *step += 1;
  return 0;
}

int shard_orthonormalize(ShardedCtx* sh, std::string* err) { return cqr2(sh, sh->cur, err); }

int shard_entropy(ShardedCtx* sh, const int64_t* A, int64_t nA, double* S_out, std::string* err) {
  STRY(sh->comm.wd.check(err));
  cudaStream_t st = sh->st;
  // split A by owning shard (order within a shard preserved; the spectrum is order-free)
  std::vector<std::vector<int32_t>> part(sh->P);
  for (int64_t q = 0; q < nA; ++q) part[A[q] / sh->Lp].push_back((int32_t)A[q]);
  std::vector<int32_t> flat;
  std::vector<size_t> offs(sh->P + 1, 0);
  for (int q = 0; q < sh->P; ++q) {
    offs[q] = flat.size();
    flat.insert(flat.end(), part[q].begin(), part[q].end());
  }
  offs[sh->P] = flat.size();
  SCK(cudaMemcpyAsync(sh->region, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice, st));
  SCK(cudaMemsetAsync(sh->bad_dev, 0, 4, st));
  const int other = 1 - sh->cur;
  int n;
  if (nA > sh->N) {
    // distributed Gram of U_A: sum over shards of U_{A,g}^dag U_{A,g}
    for (auto& l : sh->loc) {
      const int c = (int)part[l.g].size();
      if (c) STRY(gather_rows(st, l.U[sh->cur], sh->ldN, 0, sh->region + offs[l.g], 0, nullptr, c, 1, l.U[other],
                              sh->ldN, 0, sh->N, err, l.row0));
      STRY(zgemm(st, 1, 0, sh->N, sh->N, c, 1.0, 0.0, l.U[other], sh->ldN, 0, l.U[other], sh->ldN, 0, 0.0, l.Gpart,
                 sh->ldN, 0, 1, 0, err));
    }
    STRY(allreduce_gram(sh, err));
    n = sh->N;
  } else {
    // gather the rows of A from every shard, then C_A = U_A U_A^dag
    size_t capA = 0;
    for (int q = 0; q < sh->P; ++q) capA = std::max(capA, part[q].size());
    std::vector<void*> send;
    for (auto& l : sh->loc) {
      const int c = (int)part[l.g].size();
      if (c) STRY(gather_rows(st, l.U[sh->cur], sh->ldN, 0, sh->region + offs[l.g], 0, nullptr, c, 1, l.U[other],
                              sh->ldN, 0, sh->N, err, l.row0));
      send.push_back(l.U[other]);
    }
    STRY(sh->comm.allgather(st, send.data(), sh->Ufull, capA * sh->ldN * 16, err));
    for (int q = 0; q < sh->P; ++q)
      if (!part[q].empty())
        SCK(cudaMemcpyAsync(sh->X + offs[q] * sh->ldN, sh->Ufull + (size_t)q * capA * sh->ldN,
                            part[q].size() * sh->ldN * 16, cudaMemcpyDeviceToDevice, st));
    STRY(zgemm(st, 0, 1, nA, nA, sh->N, 1.0, 0.0, sh->X, sh->ldN, 0, sh->X, sh->ldN, 0, 0.0, sh->G, sh->ldN, 0, 1, 0,
               err));
    n = (int)nA;
  }
  cusolverStatus_t r = cusolverDnZheevd(sh->solver, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                        reinterpret_cast<cuDoubleComplex*>(sh->G), (int)sh->ldN, sh->eig_w,
                                        reinterpret_cast<cuDoubleComplex*>(sh->eig_work), sh->lwork, sh->eig_info);
  if (r != CUSOLVER_STATUS_SUCCESS) {
    if (err) *err = "cusolverDnZheevd failed: " + std::to_string(r);
    return TRAJ_ECUDA;
  }
  STRY(entropy_reduce(st, sh->eig_w, n, sh->S_dev, sh->bad_dev, err));
  int32_t flags[2];
  SCK(cudaMemcpyAsync(S_out, sh->S_dev, 8, cudaMemcpyDeviceToHost, st));
  SCK(cudaMemcpyAsync(&flags[0], sh->bad_dev, 4, cudaMemcpyDeviceToHost, st));
  SCK(cudaMemcpyAsync(&flags[1], sh->failed_dev, 4, cudaMemcpyDeviceToHost, st));
  SCK(cudaStreamSynchronize(st));
  if (flags[1]) S_out[0] = nan("");
  if (flags[0] && !flags[1]) {
    int32_t one = 1;
    SCK(cudaMemcpy(sh->failed_dev, &one, 4, cudaMemcpyHostToDevice));
    if (err) *err = "spectrum of C_A outside [-1e-8, 1+1e-8]";
    return TRAJ_ENUMERIC;
  }
  return 0;
}

int shard_occupations(ShardedCtx* sh, double* n_out, long long step, std::string* err) {
  for (size_t s = 0; s < sh->loc.size(); ++s)
    STRY(row_monitor(sh->st, sh->loc[s].U[sh->cur], sh->ldN, 0, sh->Lp, sh->N, 1, 0, step, sh->traj_base, sh->seed,
                     sh->gamma_dev, sh->dt, n_out + s * sh->Lp, err, sh->loc[s].row0));
  return 0;
}

int shard_full_state(ShardedCtx* sh, std::string* err) { return gather_full(sh, sh->cur, err); }

int shard_correlation_rows(ShardedCtx* sh, int64_t row0, int64_t nrows, void* C_out, std::string* err) {
  STRY(gather_full(sh, sh->cur, err));
  return zgemm(sh->st, 0, 1, nrows, sh->L, sh->N, 1.0, 0.0, sh->Ufull + row0 * sh->ldN, sh->ldN, 0, sh->Ufull,
               sh->ldN, 0, 0.0, reinterpret_cast<cplx*>(C_out), sh->L, 0, 1, 0, err);
}

int shard_get_state(ShardedCtx* sh, void* U_out, std::string* err) {
  for (size_t s = 0; s < sh->loc.size(); ++s)
    SCK(cudaMemcpy2DAsync(reinterpret_cast<char*>(U_out) + s * (size_t)sh->Lp * sh->N * 16, (size_t)sh->N * 16,
                          sh->loc[s].U[sh->cur], (size_t)sh->ldN * 16, (size_t)sh->N * 16, sh->Lp, cudaMemcpyDefault,
                          sh->st));
  SCK(cudaStreamSynchronize(sh->st));
  return 0;
}

int shard_set_state(ShardedCtx* sh, const void* U_in, std::string* err) {
  for (size_t s = 0; s < sh->loc.size(); ++s)
    SCK(cudaMemcpy2DAsync(sh->loc[s].U[sh->cur], (size_t)sh->ldN * 16,
                          reinterpret_cast<const char*>(U_in) + s * (size_t)sh->Lp * sh->N * 16, (size_t)sh->N * 16,
                          (size_t)sh->N * 16, sh->Lp, cudaMemcpyDefault, sh->st));
  SCK(cudaStreamSynchronize(sh->st));
  return 0;
}

int shard_failed(ShardedCtx* sh, int32_t* flag, std::string* err) {
  SCK(cudaMemcpyAsync(sh->h_small, sh->failed_dev, 4, cudaMemcpyDeviceToHost, sh->st));
  SCK(cudaStreamSynchronize(sh->st));
  STRY(sh->comm.wd.check(err));
  *flag = sh->h_small[0];
  return 0;
}

void shard_destroy(ShardedCtx* sh) {
  if (sh->st) cudaStreamSynchronize(sh->st);
  if (sh->cst) {
    cudaStreamSynchronize(sh->cst);
    cudaStreamDestroy(sh->cst);
  }
  if (sh->ev_start) cudaEventDestroy(sh->ev_start);
  if (sh->gst) {
    cudaStreamSynchronize(sh->gst);
    cudaStreamDestroy(sh->gst);
  }
  for (cudaEvent_t e : {sh->ev_gpacked[0], sh->ev_gpacked[1], sh->ev_gfree[0], sh->ev_gfree[1], sh->ev_gdone})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t q : {sh->st_hi, sh->st_lo})
    if (q) {
      cudaStreamSynchronize(q);
      cudaStreamDestroy(q);
    }
  for (cudaEvent_t e : {sh->ev_fork, sh->ev_left, sh->ev_lo_done, sh->ev_hi_done})
    if (e) cudaEventDestroy(e);
  for (auto e : sh->ev_chunk)
    if (e) cudaEventDestroy(e);
  for (auto e : sh->sc_ev)
    if (e) cudaEventDestroy(e);
  sh->sc_ev.clear();
  sh->fbg.destroy();
  const bool aborted = sh->comm.wd.stop();   // an aborted communicator is already freed
  if (sh->comm.comm && !aborted) ncclCommDestroy(sh->comm.comm);
  if (sh->h_small) cudaFreeHost(sh->h_small);
  if (sh->h_dev) cudaFreeHost(sh->h_dev);
}

}  // namespace traj
