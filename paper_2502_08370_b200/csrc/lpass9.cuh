// lpass9.cuh -- the x-stage of a 2-D step on long lines (n >= 2048) as 64 x 64 tile kernels,
// persistent over slice groups like lpass8.cuh.
//
// The x-stage solves (I - tau A_x) V_1 = r_1 along every row, r_1 = U + tau F (FIE) or
// U + tau A_y U + tau F (DR, M = 2 form, R1).  A row of 4096
// points is cut into 64-point blocks coupled through block tuples (lpass4.cuh):
//   K_xt  (MODE 0): per tile, the rows' block tuples from r_1;
//   lp5_scan      : per row, the incoming y / outgoing x of every block;
//   K_xf  (MODE 1): per tile, the exact forward / backward recurrences from those, the
//                   y-stage right-hand side r_2 = V_1 (- w for DR) written out, and -- since a
//                   tile holds 64 complete rows of r_2 for its 64 columns -- the y-stage block
//                   tuples of its columns (what lpass8's tuple kernel would re-read r_2 for).
// Then lp5_scan (y) and lpass8's finish complete the step.  Per point and step: read U twice,
// write r_2, read r_2, write U' (40 B) plus the coefficient tiles once per slice group.
// A thread walks 16 consecutive x of one row (rows across lanes, odd shared row stride:
// conflict-free); the DR stencil reads rows j +- 1 from the same tile (one halo row each side).
#pragma once
#include "common.cuh"
#include "lpass4.cuh"
#include "lpass5.cuh"
#include "lpass8.cuh"
#include "xpass3.cuh"

namespace prs {

constexpr int L9ROWS = L5RB + 2;     // tile rows + DR halo rows
constexpr int L9S = L5W + 1;         // shared row stride (odd)
constexpr int L9TILE = L9ROWS * L9S;
constexpr int L9SLOTS = 3;

struct L9Args {
    const double *in;
    double *out;          // MODE 1: r_2 (may not alias in)
    long long vol;        // slice stride
    int n, nrb, ncb;
    long long nsq;        // states in the batch
    int s8, nsg8;         // slices per CTA, slice groups
    double tau, h2inv, creact, src_amp;
    const double *sinpi;
    TimeArgs ta;
    CoefTab tab;
    const double *invdx, *invdy, *s2n, *s2f;
    double *ttx, *yxx;    // x block tuples [5][B][ncb][n] (line = row), scan results [2][...]
    long long tsx;        // B * ncb * n
    double *tty;          // y block tuples [5][B][nrb][n] (MODE 1)
    long long tsy;        // B * nrb * n
};

inline size_t lpass9_smem_bytes() { return sizeof(double) * (size_t)L9SLOTS * L9TILE; }

__device__ __forceinline__ void cp_async8b(void *smem_dst, const void *gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}

template <int COEF, int DR, int SRC, int MODE>
__global__ void __launch_bounds__(L5T, 2) lp9_kernel(L9Args a) {
    extern __shared__ __align__(16) double ring[];
    __shared__ double st[5][L5CP][L5W];
    __shared__ double tfx[L5W + 1], tnx[L5W], tpx[L5W], tfy[L5RB + 1];
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int n = a.n;
    const long long pos = blockIdx.x / a.nsg8;
    const int sg = (int)(blockIdx.x - pos * a.nsg8);
    const int cb = (int)(pos % a.ncb), rb = (int)(pos / a.ncb);
    const int j0 = rb * L5RB, i0 = cb * L5W;
    const long long b0 = (long long)sg * a.s8;
    const long long b1 = min(a.nsq, b0 + a.s8);
    const double tauh = a.tau * a.h2inv;

    // x-walk mapping: chunk xc of row xr (rows across the lanes of a warp)
    const int xc = wp & 3, xr = (wp >> 2) * 32 + lane;
    const int j = j0 + xr;
    const int xe0 = xc * LCH;  // first column of the chunk within the tile
    // y-walk mapping (MODE 1): column yw, chunk yt of 16 rows
    const int yw = tid % L5W, yt = tid / L5W;

    // ---- per tile position, once: face / node tables and coefficients ----
    for (int e = tid; e <= L5W; e += L5T) tfx[e] = COEF ? __ldg(a.s2f + i0 + e) : 0.0;
    for (int e = tid; e < L5W; e += L5T) {
        tnx[e] = COEF ? 0.5 * __ldg(a.s2n + i0 + e) : 0.0;
        tpx[e] = SRC ? __ldg(a.sinpi + i0 + e) : 0.0;
    }
    for (int e = tid; e <= L5RB; e += L5T) tfy[e] = (COEF && MODE == 1) ? __ldg(a.s2f + j0 + e) : 0.0;
    double idx[LCH], idxm1 = 0.0;  // x pivots of this thread's chunk (COEF) / kappa = 1 tables
    double tmx[LCH], tix[LCH], tcx[LCH];
    if (COEF) {
        const double *p = a.invdx + (long long)j * n + i0 + xe0;
#pragma unroll
        for (int i = 0; i < LCH; ++i) idx[i] = __ldg(p + i);
        idxm1 = (i0 + xe0 > 0) ? __ldg(p - 1) : 0.0;
    } else {
#pragma unroll
        for (int i = 0; i < LCH; ++i) {
            tmx[i] = __ldg(a.tab.m + i0 + xe0 + i);
            tix[i] = __ldg(a.tab.id + i0 + xe0 + i);
            tcx[i] = __ldg(a.tab.cc + i0 + xe0 + i);
        }
    }
    const double hsxr = COEF ? 0.5 * __ldg(a.s2n + j) : 0.0;  // kappa on the x faces of row j
    const double sfm = COEF ? __ldg(a.s2f + j) : 0.0, sfp = COEF ? __ldg(a.s2f + j + 1) : 0.0;
    const double spj = SRC ? __ldg(a.sinpi + j) : 0.0;
    double idy[LCH], idym1 = 0.0;  // y pivots of the y-walk column chunk (MODE 1, COEF)
    double tmy[LCH], tiy[LCH], tcy[LCH];
    const int yr0 = j0 + yt * LCH, ycol = i0 + yw;
    if (MODE == 1) {
        if (COEF) {
            const double *p = a.invdy + (long long)yr0 * n + ycol;
#pragma unroll
            for (int i = 0; i < LCH; ++i) idy[i] = __ldg(p + (long long)i * n);
            idym1 = (yr0 > 0) ? __ldg(p - n) : 0.0;
        } else {
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                tmy[i] = __ldg(a.tab.m + yr0 + i);
                tiy[i] = __ldg(a.tab.id + yr0 + i);
                tcy[i] = __ldg(a.tab.cc + yr0 + i);
            }
        }
    }
    const double hsxc = (COEF && MODE == 1) ? 0.5 * __ldg(a.s2n + ycol) : 0.0;  // kappa on y faces of col

    auto afx = [&](int i) { return -tauh * fma(hsxr, tfx[xe0 + i], 1.0); };
    auto cmx = [&](int i) { return COEF ? afx(i) * (i == 0 ? idxm1 : idx[i - 1]) : tmx[i]; };
    auto cix = [&](int i) { return COEF ? idx[i] : tix[i]; };
    auto ccx = [&](int i) { return COEF ? afx(i + 1) * idx[i] : tcx[i]; };
    auto afy = [&](int i) { return -tauh * fma(hsxc, tfy[yt * LCH + i], 1.0); };
    auto cmy = [&](int i) { return COEF ? afy(i) * (i == 0 ? idym1 : idy[i - 1]) : tmy[i]; };
    auto ciy = [&](int i) { return COEF ? idy[i] : tiy[i]; };
    auto ccy = [&](int i) { return COEF ? afy(i + 1) * idy[i] : tcy[i]; };

    // ---- state tiles (rows j0-1 .. j0+64) through the ring ----
    auto issue = [&](long long b, int slot) {
        const double *src = a.in + b * a.vol + (long long)(j0 - 1) * n + i0;
        double *dst = ring + slot * L9TILE;
        for (int e = tid; e < L9ROWS * L5W; e += L5T) {
            const int rr = e >> 6, cc = e & 63;
            const int jj = j0 - 1 + rr;
            if (jj >= 0 && jj < n) cp_async8b(dst + rr * L9S + cc, src + (long long)rr * n + cc);
        }
    };
    if (b0 < b1) issue(b0, 0);
    cp_async_commit();
    if (b0 + 1 < b1) issue(b0 + 1, 1);
    cp_async_commit();

    int slot = 0;
    for (long long b = b0; b < b1; ++b) {
        {
            int s2 = slot + 2;
            if (s2 >= L9SLOTS) s2 -= L9SLOTS;
            if (b + 2 < b1) issue(b + 2, s2);
            cp_async_commit();
        }
        cp_async_wait<2>();
        __syncthreads();
        double *tile = ring + slot * L9TILE;
        double *trow = tile + (xr + 1) * L9S + xe0;
        // ---- r_1 of this chunk ----
        double v[LCH];
        // w = tau A_y U (2-D, M = 2: reaction share c/2) at element i of the chunk, from the
        // tile's original rows j-1, j, j+1 (recomputed where it is subtracted again: the tile
        // is only overwritten after a barrier)
        auto wdr = [&](int i) {
            const double uu = trow[i];
            const double dm = (j > 0) ? trow[i - L9S] : 0.0, dp = (j < n - 1) ? trow[i + L9S] : 0.0;
            const double km = COEF ? fma(tnx[xe0 + i], sfm, 1.0) : 1.0;
            const double kp = COEF ? fma(tnx[xe0 + i], sfp, 1.0) : 1.0;
            return a.tau * ((kp * (dp - uu) - km * (uu - dm)) * a.h2inv - a.creact * uu);
        };
#pragma unroll
        for (int i = 0; i < LCH; ++i) v[i] = DR ? trow[i] + wdr(i) : trow[i];
        if (SRC) {
            const double f = a.tau * a.src_amp * exp(-src_time(a.ta, b)) * spj;
#pragma unroll
            for (int i = 0; i < LCH; ++i) v[i] = fma(f, tpx[xe0 + i], v[i]);
        }
        // ---- chunk tuple (walk with y_in = 0) ----
        Tup u;
        {
            double y0 = 0.0, g = 1.0, cp = 1.0, Q = 0.0, R = 0.0;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                const double m = cmx(i);
                y0 = fma(-m, y0, v[i]);
                g = -m * g;
                const double cid = cp * cix(i);
                Q = fma(cid, y0, Q);
                R = fma(cid, g, R);
                cp *= -ccx(i);
            }
            u = Tup{g, y0, cp, Q, R};
        }
        st[0][xc][xr] = u.A;
        st[1][xc][xr] = u.B;
        st[2][xc][xr] = u.P;
        st[3][xc][xr] = u.Q;
        st[4][xc][xr] = u.R;
        __syncthreads();  // chunk tuples visible
        if (MODE == 0) {
            if (xc == 0) {
                Tup tot = tup_id();
#pragma unroll
                for (int q = 0; q < L5CP; ++q)
                    tot = tup_cat(tot, Tup{st[0][q][xr], st[1][q][xr], st[2][q][xr], st[3][q][xr], st[4][q][xr]});
                const long long o = (b * a.ncb + cb) * n + j;
                a.ttx[o] = tot.A;
                a.ttx[a.tsx + o] = tot.B;
                a.ttx[2 * a.tsx + o] = tot.P;
                a.ttx[3 * a.tsx + o] = tot.Q;
                a.ttx[4 * a.tsx + o] = tot.R;
            }
        } else {
            const long long ob = (b * a.ncb + cb) * n + j;
            const double Yblk = a.yxx[ob], Xblk = a.yxx[a.tsx + ob];
            double Y = Yblk;
#pragma unroll
            for (int q = 0; q < L5CP; ++q)
                if (q < xc) Y = fma(st[0][q][xr], Y, st[1][q][xr]);
            const double Ylast = fma(u.A, Y, u.B);
            Tup s = tup_id();
#pragma unroll
            for (int q = L5CP - 1; q >= 0; --q)
                if (q > xc) s = tup_cat(Tup{st[0][q][xr], st[1][q][xr], st[2][q][xr], st[3][q][xr], st[4][q][xr]}, s);
            const double X = fma(s.P, Xblk, fma(s.R, Ylast, s.Q));
            double y = Y;
#pragma unroll
            for (int i = 0; i < LCH; ++i) {
                y = fma(-cmx(i), y, v[i]);
                v[i] = y;
            }
            double x = X;
#pragma unroll
            for (int i = LCH - 1; i >= 0; --i) {
                x = fma(cix(i), v[i], -ccx(i) * x);
                v[i] = DR ? x - wdr(i) : x;
            }
            if (DR) __syncthreads();  // every read of the original tile rows is done
            // r_2 of this chunk back into the tile
#pragma unroll
            for (int i = 0; i < LCH; ++i) trow[i] = v[i];
            __syncthreads();  // tile = r_2; the chunk tuples above are consumed
            // ---- y-stage block tuples of this tile's columns (walk down yw, rows of chunk yt) ----
            {
                const double *cptr = tile + (yt * LCH + 1) * L9S + yw;
                double y0 = 0.0, g = 1.0, cp = 1.0, Q = 0.0, R = 0.0;
#pragma unroll
                for (int i = 0; i < LCH; ++i) {
                    const double m = cmy(i);
                    y0 = fma(-m, y0, cptr[i * L9S]);
                    g = -m * g;
                    const double cid = cp * ciy(i);
                    Q = fma(cid, y0, Q);
                    R = fma(cid, g, R);
                    cp *= -ccy(i);
                }
                st[0][yt][yw] = g;
                st[1][yt][yw] = y0;
                st[2][yt][yw] = cp;
                st[3][yt][yw] = Q;
                st[4][yt][yw] = R;
            }
            // ---- store r_2 (coalesced rows) ----
            {
                double *o = a.out + b * a.vol + (long long)j0 * n + i0;
                for (int e = tid; e < L5RB * L5W; e += L5T) {
                    const int rr = e >> 6, cc = e & 63;
                    o[(long long)rr * n + cc] = tile[(rr + 1) * L9S + cc];
                }
            }
            __syncthreads();
            if (yt == 0) {
                Tup tot = tup_id();
#pragma unroll
                for (int q = 0; q < L5CP; ++q)
                    tot = tup_cat(tot, Tup{st[0][q][yw], st[1][q][yw], st[2][q][yw], st[3][q][yw], st[4][q][yw]});
                const long long o = (b * a.nrb + rb) * n + ycol;
                a.tty[o] = tot.A;
                a.tty[a.tsy + o] = tot.B;
                a.tty[2 * a.tsy + o] = tot.P;
                a.tty[3 * a.tsy + o] = tot.Q;
                a.tty[4 * a.tsy + o] = tot.R;
            }
        }
        __syncthreads();  // ring slot and tuple scratch free for the next slice
        slot = (slot + 1 == L9SLOTS) ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}

}  // namespace prs
