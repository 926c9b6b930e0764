// Internal interface of the banded circulant propagator pass (banded.cu, NEXT-1).
#pragma once
#include <string>
#include "common.cuh"

namespace traj {

// smallest compiled half-bandwidth >= w, or -1 (then use the dense K)
int banded_template_width(int w);

// V[site(line,p)] = sum_{d=-W..W} coef[d+W] U[site(line,(p+d) mod len)], site(line,p) =
// line*line_stride + p*pos_stride (rows of the row-major [rows][ld] complex U), N columns,
// T batch entries of stride sU.  coef_host: HOST, 2W+1 complex (zero-padded beyond the true w), copied
// into the launch's parameter space.
// periodic = 0 (halo mode): output position p reads input positions p .. p+2W (the input holds
// W halo positions before and after the len outputs), no wrap-around.
int banded_pass(cudaStream_t st, const cplx* U, cplx* V, long long ld, long long sU, int N, int T, int len, int lines,
                long long line_stride, long long pos_stride, const cplx* coef_host, int W, std::string* err,
                int periodic = 1);

}  // namespace traj
