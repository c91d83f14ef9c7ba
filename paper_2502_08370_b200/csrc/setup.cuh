// setup.cuh -- one-off kernels run at context creation: sine tables and
// the precomputed pivots of every stage matrix (I - tau A_d), tau in {Delta T, delta t}.
#pragma once
#include "common.cuh"

namespace prs {

// sin tables: sinpi[i] = sin(pi x_i), s2n[i] = sin(2 pi x_i), s2f[f] = sin(2 pi (f + 1/2) h)
__global__ void setup_sines(int n, double h, double *sinpi, double *s2n, double *s2f) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const double PI = 3.14159265358979323846;
    if (i < n) {
        const double x = (double)(i + 1) * h;
        sinpi[i] = sin(PI * (double)(i + 1) * h);
        s2n[i] = sin(2.0 * PI * x);
    }
    if (i <= n) s2f[i] = sin(2.0 * PI * (((double)i + 0.5) * h));
}

// pivots of (I - tau A_d), kappa = 1: off-diagonal o = -tau/h^2, diagonal 1 + 2 tau/h^2 + tau c/M
__global__ void setup_const_tab(int n, double tau, double h2inv, double creact, double *m,
                                double *id, double *cc) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    const double o = -tau * h2inv;
    const double bd = 1.0 + 2.0 * tau * h2inv + tau * creact;
    double d = bd;
    id[0] = 1.0 / d;
    m[0] = 0.0;
    for (int i = 1; i < n; ++i) {
        d = bd - o * o * id[i - 1];
        id[i] = 1.0 / d;
        m[i] = o * id[i - 1];
        cc[i - 1] = o * id[i - 1];
    }
    cc[n - 1] = 0.0;
}

// per-point inverse pivots of (I - tau A_x) (axis 0, one thread per row j) or (I - tau A_y)
// (axis 1, one thread per column i) for kappa = 1 + 0.5 sin(2 pi x) sin(2 pi y) (2-D, M = 2)
__global__ void setup_var_invd(int n, int axis, double tau, double h2inv, double creact,
                               const double *s2n, const double *s2f, double *invd) {
    const int L = blockIdx.x * blockDim.x + threadIdx.x;
    if (L >= n) return;
    const double sl = s2n[L];
    double idp = 0.0;
    for (int k = 0; k < n; ++k) {
        const double km = 1.0 + 0.5 * s2f[k] * sl;      // face k - 1/2
        const double kp = 1.0 + 0.5 * s2f[k + 1] * sl;  // face k + 1/2
        const double bd = 1.0 + tau * (km + kp) * h2inv + tau * creact;
        const double am = -tau * km * h2inv;
        const double d = (k == 0) ? bd : bd - am * am * idp;
        idp = 1.0 / d;
        const long long at = (axis == 0) ? (long long)L * n + k : (long long)k * n + L;
        invd[at] = idp;
    }
}

// max |u| over a state (u0 norm): bit pattern max of non-negative doubles
__global__ void absmax_kernel(const double *u, long long N, unsigned long long *out) {
    double m = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x)
        m = fmax(m, fabs(u[i]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

}  // namespace prs
