// Internal interface of the event-driven projective protocol (pm_events.cu, NEXT-4).
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

// Axis taps: neighbour offsets lo .. lo+n-1 (mod the extent) with coefficients c[0..n).
// yhat = r_j / |r_j| with r_j row j of K(tau) U; coef = [alpha, beta, occ, p]; ++*occ_count if occupied
int event_prep(cudaStream_t st, const cplx* U, long long ld, int N, int Lx, int Ly, int j, const cplx* cx, int xlo,
               int xn, const cplx* cy, int ylo, int yn, double pc, cplx* yhat, double* coef, int32_t* occ_count,
               std::string* err);
// out = K(tau) U + x yhat, x = alpha (K(tau) U yhat^dag) + beta e_j (coef == nullptr: propagation only)
int event_update(cudaStream_t st, const cplx* U, cplx* out, long long ld, int N, int Lx, int Ly, const cplx* cx,
                 int xlo, int xn, const cplx* cy, int ylo, int yn, const cplx* yhat, const double* coef, int j,
                 std::string* err);

// ---- one-pass form (pm_events.cu): yhat kept unnormalised, coef = [alpha, beta, occ, p, s = 1/|r|]
// prepare event (site j, Born threshold pc): r = row j of K(c) U + X y_prev s_prev, where c are
// the taps of tau_prev + tau (or tau alone when coef_prev == nullptr) and X = (K(o) x)_j for
// x_m = alpha_prev (K(tau_prev) g_prev)_m + beta_prev delta_{m, j_prev} (own taps o: tau), evaluated as
// alpha_prev (K(c) g_prev)_j + beta_prev K(o)_{j, j_prev}.  Writes y_out = r, coef_out, ++*occ_count if
// occupied.  part: >= 64 doubles.
int ev_prep(cudaStream_t st, const cplx* U, long long ld, int N, int Lx, int Ly, int j, const cplx* cxc, int cxlo,
            int cxn, const cplx* cyc, int cylo, int cyn, const cplx* oxc, int oxlo, int oxn, const cplx* oyc, int oylo,
            int oyn, const double* coef_prev, const double2* g_prev, const cplx* y_prev, int j_prev, double pc,
            cplx* y_out, double* part, double* coef_out, int32_t* occ_count, std::string* err);
// g_i = s sum_k U_ik conj(y_k)
int ev_gemv(cudaStream_t st, const cplx* U, long long ld, int N, int L, const cplx* y, const double* coef, double2* g,
            std::string* err);
// out = K(tau) U + x y s (x_i = alpha (K g)_i + beta delta_ij; coef == nullptr: propagation only), and
// gn_i = sn <out_i, yn> when yn != nullptr.  1d bands of half-width <= 9 use the row-blocked
// kernel with the HOST taps cx_host passed by value; otherwise the device taps, one CTA per row.  On a 2d lattice
// with tmp (L x ld) and gx (L) given, the pass is separable: the x-axis taps into tmp (and g into gx), then the
// y-axis taps with the rank-1 term into out (TRAJ_EV_SEPARABLE=0: the (2w+1)^2 product taps in one kernel); each
// half runs on the row-blocked kernel over the axis's rings when its band fits (HOST taps cx_host / cy_host).
int ev_pass(cudaStream_t st, const cplx* U, cplx* out, long long ld, int N, int Lx, int Ly, const cplx* cx_dev,
            const cplx* cx_host, int xlo, int xn, const cplx* cy_dev, const cplx* cy_host, int ylo, int yn_taps,
            const cplx* y, const double* coef, const double2* g, int j, const cplx* yn, const double* coefn,
            double2* gn, cplx* tmp, double2* gx, std::string* err);

}  // namespace traj
