// Fused small-lattice trajectory step (small_step.cu): every row a1-a3 of the step for one
// trajectory per CTA, the state resident in shared memory across a run of steps.
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

struct SmallStepArgs {
  cplx* U;                  // [T][L][ldU], updated in place
  long long ldU, sU;
  const cplx* K;            // [L][ldK] dense propagator, shared by the batch
  long long ldK;
  int L, N, T;
  int projective;           // 1: projective clicks, 0: homodyne (Eq. A3)
  long long step0;          // step index of the first step (Philox counter word 1)
  long long n_steps;
  long long traj_base;      // global id of trajectory 0 (Philox counter word 2)
  uint64_t seed;
  const double* gamma;      // [T] device
  double dt;
  int32_t* failed;          // [T]: set on a non-positive Cholesky pivot; that trajectory then stops
  int32_t* last;            // [T][2]: clicks and occupied outcomes of the last step (projective)
  cplx* Dg;                 // [T][cap][ldDg] global C_SS for click lists too long for the scratch
  long long ldDg, sDg;      //   buffer in shared memory (m (m + 1) > L (N + 1), e.g. gamma dt = 1)
  int cap;                  // click-list capacity: more clicks flag the trajectory as failed
  int full_cqr2;            // 1: always factor the second Gram (TRAJ_CQR2_FULL=1)
  int skip_orthonormal_pass;  // 1: projective step with no zeroed row skips CholeskyQR pass 1
  unsigned long long* fallbacks;   // second passes that needed the full factorisation (atomic count)
};

// Dynamic shared memory the fused kernel needs for (L, N), in bytes.
size_t small_step_smem_bytes(int L, int N, bool projective);
// True when the state and the step's scratch fit one CTA's shared memory on the current device.
bool small_step_fits(int L, int N, bool projective);
int small_steps(cudaStream_t st, const SmallStepArgs& a, std::string* err);

}  // namespace traj
