// F_ref probe: the STRAIGHTFORWARD matvec pair evaluation of
// Eqs. (10), (12)-(13) written with libdevice exp() and rsqrt(), no algebraic tuning.
// Its SASS loop body defines the frozen per-pair FLOP count F_ref used for the
// roofline's algorithmic FLOPs (ncu convention: DFMA = 2, DMUL = DADD = 1).
// Build + count:  python tools/fref_probe.py
#include <cuda_runtime.h>
__global__ void fref_pair_loop(const double* __restrict__ src, int n, double X, double Y, double Z, double NX,
                               double NY, double NZ, double kappa, double eps, double* out) {
  double s1 = 0, s2 = 0;
  for (int j = 0; j < n; ++j) {
    const double* s = src + 8 * j;  // x, y, z, nx, ny, nz, W u_phi, W u_dphi
    double dx = X - s[0], dy = Y - s[1], dz = Z - s[2];
    double r2 = dx * dx + dy * dy + dz * dz;
    double ir = rsqrt(r2), r = r2 * ir;  // the paper's "fast CUDA operators like rsqrt"
    double ir3 = ir * ir * ir, ir5 = ir3 * ir * ir;
    double e = exp(-kappa * r);
    double dnx = dx * NX + dy * NY + dz * NZ;
    double dny = dx * s[3] + dy * s[4] + dz * s[5];
    double nxy = NX * s[3] + NY * s[4] + NZ * s[5];
    double kr = kappa * r;
    double K1 = ir * (1.0 - e);
    double K2 = dny * ir3 * (eps * e * (1.0 + kr) - 1.0);
    double K3 = -dnx * ir3 * (1.0 - e * (1.0 + kr) / eps);
    double K4 = nxy * ir3 * (e * (1.0 + kr) - 1.0) - dnx * dny * ir5 * (e * (3.0 + 3.0 * kr + kr * kr) - 3.0);
    s1 += K1 * s[7] + K2 * s[6];
    s2 += K3 * s[7] + K4 * s[6];
  }
  out[threadIdx.x] = s1;
  out[threadIdx.x + blockDim.x] = s2;
}
