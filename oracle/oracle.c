/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, serial fp64 CPU oracle of the parareal-with-splitting method of
 * arXiv 2502.08370 (PAPER.md in the reference). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library. It shares
 * no code, header or table with the CUDA path (paper_2502_08370_b200/csrc).
 *
 * Everything is computed literally, in the paper's order and notation:
 *   - operator rows      : PAPER.md:45-57 (eq. cont_problem, L = div(D grad u) - c u),
 *                          PAPER.md:63-67 (dimensional split, reaction share c/M),
 *                          PAPER.md:111-134 (partition of unity, L_j = div(rho_j D grad u) - rho_j c u),
 *                          face-centred conservative FD as SPEC.md:52.
 *   - FIE step           : PAPER.md:151-157 (eq. FIE_method).
 *   - DR step            : PAPER.md:165-171 (eq. DR_method), predictor (I + tau A)U_n
 *                          evaluated literally with the unsplit A (reading R1).
 *   - IE step            : unsplit implicit Euler, the Parareal/IE-IE baseline (PAPER.md:455,
 *                          SPEC.md:206-214), band elimination of the whole system (NEXT-4).
 *   - stage solves       : Thomas per grid line (dimensional, "one-dimensional
 *                          uncoupled systems"), band Gaussian elimination per strip block
 *                          (DD, "q independent subsystems"); factorised on the fly.
 *   - propagators        : G = one step of Delta T, F^s = s steps of delta t.
 *   - parareal           : PAPER.md:194-206, U^{k+1}_{n+1} = G(U^{k+1}_n) + F^s(U^k_n) - G(U^k_n)
 *                          evaluated left to right.
 *
 * Threads: orc_set_threads(k) lets orc_parareal_iteration run its F^s(U^k_n) and G(U^k_n)
 * evaluations -- independent per slice n ("can be computed in parallel for
 * every n") -- on k POSIX threads, one slice per task, each with its own buffers; the values
 * are bitwise those of the serial loop (tests/test_oracle_pins.py).  Everything else is serial.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC -pthread (no FMA contraction).
 * Parity pins for every function live in tests/test_oracle_*.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>

#include "oracle_problem.h"

#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------ grid ---- */
/* Interior nodes i = 1..n per axis, x_i = i h, h = 1/(n+1). */
static double grid_h(const orc_problem *p) { return 1.0 / (double)(p->n + 1); }

static long npoints(const orc_problem *p) {
    long n = p->n;
    return p->dim == 3 ? n * n * n : n * n;
}

/* x-fastest linear index of the 1-based node (i, l, m) */
static long node_index(const orc_problem *p, int i, int l, int m) {
    long n = p->n;
    return ((long)(m - 1) * n + (l - 1)) * n + (i - 1);
}

/* diffusion coefficient kappa at physical point (x, y) -- D = kappa I */
static double kappa_at(const orc_problem *p, double x, double y) {
    if (p->coef == 1) return 1.0 + 0.5 * sin(2.0 * ORC_PI * x) * sin(2.0 * ORC_PI * y);
    return 1.0;
}

double orc_rho(const orc_problem *p, int j, double xpos); /* partition of unity, below */

/* coef == 2: the full diffusion tensor of PAPER.md:523-528 (section 5.2),
 * d11 = d22 = 1 / (2 + cos(3 pi x) cos(2 pi y)), d12 = 1/4. */
static double dfull_diag(double x, double y) { return 1.0 / (2.0 + cos(3.0 * ORC_PI * x) * cos(2.0 * ORC_PI * y)); }
static double dfull_offd(double x, double y) { (void)x; (void)y; return 0.25; }

/* Row of the full-tensor operator (coef == 2, 2-D) into the 3 x 3 stencil cf[di+1][dl+1]:
 *   L_j u = div(rho_j D grad u) - rho_j c u   (unsplit: rho = 1)
 * discretised conservatively: flux differences over the four faces of the node's
 * cell, (F^x_{i+1/2} - F^x_{i-1/2}) / h + (F^y_{l+1/2} - F^y_{l-1/2}) / h, with
 *   F^x_{i+1/2,l} = rho(i+1/2) [ d11 (u_{i+1,l} - u_{i,l}) / h + avg over the corners
 *                   (i+1/2, l +- 1/2) of d12 (u_y)_corner ]
 *   F^y_{i,l+1/2} = rho(i) d22 (u_{i,l+1} - u_{i,l}) / h + avg over the corners
 *                   (i +- 1/2, l+1/2) of rho(corner x) d12 (u_x)_corner
 * where a corner derivative is the mean of the two differences across the corner's cell
 * side, e.g. (u_x)_(i+1/2,l+1/2) = [(u_{i+1,l} - u_{i,l}) + (u_{i+1,l+1} - u_{i,l+1})] / 2h.
 * Readings (R21, R22): the paper does not give its mixed-derivative stencil
 * (SPEC.md:92, 103); this is the standard 9-point cross scheme (for rho = 1 the mixed part is
 * d12 (u_{i+1,l+1} - u_{i+1,l-1} - u_{i-1,l+1} + u_{i-1,l-1}) / (2 h^2)), with d12 taken at the
 * corners ("the four diagonal neighbours' midpoints").  The DD weight of a mixed
 * flux piece is rho_j at its corner's x (rho depends on x only): at a block's edge columns the
 * corner weights vanish with the face weight, so (I - tau A_j) stays block diagonal
 * and sum_j A_j = A by linearity. */
static void row_full(const orc_problem *p, int term, int i, int l, double cf[3][3]) {
    double h = grid_h(p), h2 = h * h;
    double x = i * h, y = l * h;
    double rxm = 1.0, rxp = 1.0, rn = 1.0;
    if (term >= 0) {
        rxm = orc_rho(p, term, (double)i - 0.5);
        rxp = orc_rho(p, term, (double)i + 0.5);
        rn = orc_rho(p, term, (double)i);
    }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) cf[a][b] = 0.0;
#define ADD(di, dl, v) (cf[(di) + 1][(dl) + 1] += (v))
    /* diffusion: x faces (d11 at (x_{i -+ 1/2}, y_l)), y faces (d22 at (x_i, y_{l -+ 1/2})) */
    double axp = rxp * dfull_diag(((double)i + 0.5) * h, y) / h2;
    double axm = rxm * dfull_diag(((double)i - 0.5) * h, y) / h2;
    double ayp = rn * dfull_diag(x, ((double)l + 0.5) * h) / h2;
    double aym = rn * dfull_diag(x, ((double)l - 0.5) * h) / h2;
    ADD(1, 0, axp); ADD(0, 0, -axp);
    ADD(-1, 0, axm); ADD(0, 0, -axm);
    ADD(0, 1, ayp); ADD(0, 0, -ayp);
    ADD(0, -1, aym); ADD(0, 0, -aym);
    /* mixed: corner (sx/2, sy/2) relative to the node, sx, sy in {-1, +1} */
    for (int sx = -1; sx <= 1; sx += 2)
        for (int sy = -1; sy <= 1; sy += 2) {
            double xc = ((double)i + 0.5 * sx) * h, yc = ((double)l + 0.5 * sy) * h;
            double rc = (sx > 0) ? rxp : rxm;       /* rho at the corner's x */
            double g = rc * dfull_offd(xc, yc) / (4.0 * h2); /* 1/2 (avg) x 1/(2h) x 1/h */
            /* x-face term: sign sx (outer difference), d12 (u_y)_corner, u_y across the corner
             * in direction sy: nodes (0 or sx, sy) minus (0 or sx, 0) times sy */
            double gx = sx * sy * g;
            ADD(0, sy, gx); ADD(0, 0, -gx); ADD(sx, sy, gx); ADD(sx, 0, -gx);
            /* y-face term: sign sy, d12 (u_x)_corner, u_x across the corner in direction sx */
            double gy = sy * sx * g;
            ADD(sx, 0, gy); ADD(0, 0, -gy); ADD(sx, sy, gy); ADD(0, sy, -gy);
        }
#undef ADD
    cf[1][1] -= rn * p->c; /* reaction, rho_j at the node */
}

/* ------------------------------------------------------ partition of unity -- */
/* Strip geometry in index space (reading R6): S = dd_strips strips of
 * w = n/S nodes; interface m (m = 1..S-1) at 1-based position w m + 1/2; the ramp of
 * width beta = dd_overlap cells is centred on it.  Colour 0 ("Omega_1")
 * = strips 0, 2, 4, ... (contains x = 0), colour 1 = odd strips.  rho_0 is evaluated at a
 * 1-based position xpos (integer = node, half-integer = face); rho_1 = 1 - rho_0. */
static double ramp_down(const orc_problem *p, double xpos, double xl) {
    /* descending ramp from 1 at xl to 0 at xl + beta */
    double beta = (double)p->dd_overlap;
    double u = (xpos - xl) / beta;
    if (u <= 0.0) return 1.0;
    if (u >= 1.0) return 0.0;
    if (p->dd_ramp == 1) return 0.5 * (1.0 + cos(ORC_PI * u)); /* SPEC.md:138 cosine ramp */
    return 1.0 - u;                                            /* BASELINE c4 linear ramp */
}

double orc_rho0(const orc_problem *p, double xpos) {
    int S = p->dd_strips;
    int w = p->n / S;
    /* strip that contains xpos (by the interface positions w m + 1/2) */
    int k = (int)floor((xpos - 0.5) / (double)w);
    if (k < 0) k = 0;
    if (k > S - 1) k = S - 1;
    double own = (k % 2 == 0) ? 1.0 : 0.0; /* rho_0 inside strip k away from interfaces */
    double half = 0.5 * (double)p->dd_overlap;
    /* right interface of strip k: m = k+1 */
    if (k + 1 <= S - 1) {
        double xi = (double)(w * (k + 1)) + 0.5;
        if (xpos > xi - half) {
            double d = ramp_down(p, xpos, xi - half); /* value of the colour on the left */
            return (k % 2 == 0) ? d : 1.0 - d;
        }
    }
    /* left interface of strip k: m = k */
    if (k >= 1) {
        double xi = (double)(w * k) + 0.5;
        if (xpos < xi + half) {
            double d = ramp_down(p, xpos, xi - half); /* value of the colour of strip k-1 */
            return ((k - 1) % 2 == 0) ? d : 1.0 - d;
        }
    }
    return own;
}

double orc_rho(const orc_problem *p, int j, double xpos) {
    double r0 = orc_rho0(p, xpos);
    return j == 0 ? r0 : 1.0 - r0; /* rho_2 = 1 - rho_1 */
}

/* ---------------------------------------------------------- operator rows -- */
/* Row of a (sub)operator at node (i, l, m): coefficients of
 *   out[0] centre, out[1] (-x), out[2] (+x), out[3] (-y), out[4] (+y), out[5] (-z), out[6] (+z),
 *   and for the full tensor (coef == 2) the corners out[7] (-x,-y), out[8] (+x,-y),
 *   out[9] (-x,+y), out[10] (+x,+y).
 * term = -1 : the unsplit A;
 * split == 0: term d = dimension d, L_d u = (kappa u_{x_d})_{x_d} - (c/M) u;
 * split == 1: term j = colour j, L_j u = div(rho_j kappa grad u) - rho_j c u,
 *             x-faces weighted by rho_j at the face, y-faces and reaction by rho_j at the node
 *             (SPEC.md:147).  Neighbours outside the domain are Dirichlet zero: their
 *             coefficient is still present in the centre but the off-diagonal is dropped. */
void orc_row(const orc_problem *p, int term, int i, int l, int m, double out[11]) {
    double h = grid_h(p), h2 = h * h;
    int n = p->n, M = p->dim;
    double x = i * h, y = l * h;
    for (int k = 0; k < 11; ++k) out[k] = 0.0;
    if (p->coef == 2) { /* full tensor (2-D; dimensional splitting does not apply) */
        double cf[3][3];
        row_full(p, term, i, l, cf);
        out[0] = cf[1][1];
        if (i > 1) out[1] = cf[0][1];
        if (i < n) out[2] = cf[2][1];
        if (l > 1) out[3] = cf[1][0];
        if (l < n) out[4] = cf[1][2];
        if (i > 1 && l > 1) out[7] = cf[0][0];
        if (i < n && l > 1) out[8] = cf[2][0];
        if (i > 1 && l < n) out[9] = cf[0][2];
        if (i < n && l < n) out[10] = cf[2][2];
        (void)m; (void)x; (void)y; (void)h2; (void)M;
        return;
    }
    double cen = 0.0;
    /* face coefficients kappa at midpoints; a face coordinate is formed from its
     * half-integer index, ((double)i + 0.5) h, so both neighbours see the same value */
    double kxm = kappa_at(p, ((double)i - 0.5) * h, y), kxp = kappa_at(p, ((double)i + 0.5) * h, y);
    double kym = kappa_at(p, x, ((double)l - 0.5) * h), kyp = kappa_at(p, x, ((double)l + 0.5) * h);
    double kzm = 1.0, kzp = 1.0; /* 3-D configs use kappa = 1 */
    double wx = 1.0, wxm = 1.0, wxp = 1.0, wy = 1.0, wz = 1.0, wc = 1.0;
    int use_x = 1, use_y = 1, use_z = (M == 3);
    if (term >= 0 && p->split == 0) {
        use_x = (term == 0); use_y = (term == 1); use_z = (term == 2);
        wc = 1.0 / (double)M;
    } else if (term >= 0 && p->split == 1) {
        wxm = orc_rho(p, term, (double)i - 0.5);
        wxp = orc_rho(p, term, (double)i + 0.5);
        wx = orc_rho(p, term, (double)i);
        wy = wx; wz = wx; wc = wx;
    }
    (void)wx;
    if (use_x) {
        double am = wxm * kxm / h2, ap = wxp * kxp / h2;
        cen -= am + ap;
        if (i > 1) out[1] = am;
        if (i < n) out[2] = ap;
    }
    if (use_y) {
        double am = wy * kym / h2, ap = wy * kyp / h2;
        cen -= am + ap;
        if (l > 1) out[3] = am;
        if (l < n) out[4] = ap;
    }
    if (use_z) {
        double am = wz * kzm / h2, ap = wz * kzp / h2;
        cen -= am + ap;
        if (m > 1) out[5] = am;
        if (m < n) out[6] = ap;
    }
    cen -= wc * p->c;
    out[0] = cen;
}

/* out = A_term u  (term = -1: unsplit A) */
void orc_apply(const orc_problem *p, int term, const double *u, double *out) {
    int n = p->n, nz = (p->dim == 3) ? n : 1;
    long sy = n, sz = (long)n * n;
    double r[11];
    for (int m = 1; m <= nz; ++m)
        for (int l = 1; l <= n; ++l)
            for (int i = 1; i <= n; ++i) {
                long P = node_index(p, i, l, m);
                orc_row(p, term, i, l, m, r);
                double v = r[0] * u[P];
                if (i > 1) v += r[1] * u[P - 1];
                if (i < n) v += r[2] * u[P + 1];
                if (l > 1) v += r[3] * u[P - sy];
                if (l < n) v += r[4] * u[P + sy];
                if (p->dim == 3) {
                    if (m > 1) v += r[5] * u[P - sz];
                    if (m < n) v += r[6] * u[P + sz];
                }
                if (p->coef == 2) {
                    if (i > 1 && l > 1) v += r[7] * u[P - sy - 1];
                    if (i < n && l > 1) v += r[8] * u[P - sy + 1];
                    if (i > 1 && l < n) v += r[9] * u[P + sy - 1];
                    if (i < n && l < n) v += r[10] * u[P + sy + 1];
                }
                out[P] = v;
            }
}

/* Dense copy of A_term (row-major, npts x npts); tests only, tiny grids. */
void orc_dense(const orc_problem *p, int term, double *Mat) {
    int n = p->n, nz = (p->dim == 3) ? n : 1;
    long N = npoints(p), sy = n, sz = (long)n * n;
    double r[11];
    memset(Mat, 0, sizeof(double) * N * N);
    for (int m = 1; m <= nz; ++m)
        for (int l = 1; l <= n; ++l)
            for (int i = 1; i <= n; ++i) {
                long P = node_index(p, i, l, m);
                orc_row(p, term, i, l, m, r);
                Mat[P * N + P] = r[0];
                if (i > 1) Mat[P * N + P - 1] = r[1];
                if (i < n) Mat[P * N + P + 1] = r[2];
                if (l > 1) Mat[P * N + P - sy] = r[3];
                if (l < n) Mat[P * N + P + sy] = r[4];
                if (p->dim == 3) {
                    if (m > 1) Mat[P * N + P - sz] = r[5];
                    if (m < n) Mat[P * N + P + sz] = r[6];
                }
                if (p->coef == 2) {
                    if (i > 1 && l > 1) Mat[P * N + P - sy - 1] = r[7];
                    if (i < n && l > 1) Mat[P * N + P - sy + 1] = r[8];
                    if (i > 1 && l < n) Mat[P * N + P + sy - 1] = r[9];
                    if (i < n && l < n) Mat[P * N + P + sy + 1] = r[10];
                }
            }
}

/* ---------------------------------------------------------------- source --- */
/* F(t) = f sampled at the nodes, g = 0.  source == 1:
 * f = u_t - L u for u = e^{-t} prod_d sin(pi x_d), kappa = 1, i.e.
 * f = (dim pi^2 + c - 1) e^{-t} prod_d sin(pi x_d)  (BASELINE c0/c2/c4). */
void orc_source(const orc_problem *p, double t, double *F) {
    long N = npoints(p);
    if (p->source == 2) {
        /* source == 2 (2-D, D = I): the solution u = sin(2 pi t) sin(2 pi x) sin(2 pi y) of the
         * section-5.1 experiments, f = u_t - Delta u + c u
         *   = (2 pi cos(2 pi t) + (8 pi^2 + c) sin(2 pi t)) sin(2 pi x) sin(2 pi y) */
        int n = p->n;
        double h = grid_h(p);
        double amp = 2.0 * ORC_PI * cos(2.0 * ORC_PI * t) + (8.0 * ORC_PI * ORC_PI + p->c) * sin(2.0 * ORC_PI * t);
        for (int l = 1; l <= n; ++l)
            for (int i = 1; i <= n; ++i)
                F[node_index(p, i, l, 1)] = amp * sin(2.0 * ORC_PI * i * h) * sin(2.0 * ORC_PI * l * h);
        return;
    }
    if (p->source != 1) {
        for (long k = 0; k < N; ++k) F[k] = 0.0;
        return;
    }
    int n = p->n, nz = (p->dim == 3) ? n : 1;
    double h = grid_h(p);
    double amp = ((double)p->dim * ORC_PI * ORC_PI + p->c - 1.0) * exp(-t);
    for (int m = 1; m <= nz; ++m)
        for (int l = 1; l <= n; ++l)
            for (int i = 1; i <= n; ++i) {
                double v = amp * sin(ORC_PI * i * h) * sin(ORC_PI * l * h);
                if (p->dim == 3) v *= sin(ORC_PI * m * h);
                F[node_index(p, i, l, m)] = v;
            }
}

/* ----------------------------------------------------------- stage solves -- */
/* Thomas algorithm on one tridiagonal system: sub a[k] (k>=1), diag b[k], super c[k]
 * (k<len-1); overwrites r with the solution.  Plain forward elimination + back
 * substitution, factorised on the fly. */
static void thomas(int len, const double *a, const double *b, const double *c, double *r,
                   double *work) {
    double *cp = work; /* modified super-diagonal */
    double beta = b[0];
    cp[0] = c[0] / beta;
    r[0] = r[0] / beta;
    for (int k = 1; k < len; ++k) {
        beta = b[k] - a[k] * cp[k - 1];
        cp[k] = (k < len - 1) ? c[k] / beta : 0.0;
        r[k] = (r[k] - a[k] * r[k - 1]) / beta;
    }
    for (int k = len - 2; k >= 0; --k) r[k] = r[k] - cp[k] * r[k + 1];
}

/* (I - tau A_d) v = r along every grid line of axis d (dimensional split). */
static void solve_dim(const orc_problem *p, int d, double tau, const double *r, double *v) {
    int n = p->n, nz = (p->dim == 3) ? n : 1;
    long N = npoints(p);
    long stride = (d == 0) ? 1 : (d == 1 ? (long)n : (long)n * n);
    double *a = malloc(sizeof(double) * n), *b = malloc(sizeof(double) * n),
           *c = malloc(sizeof(double) * n), *x = malloc(sizeof(double) * n),
           *w = malloc(sizeof(double) * n);
    double row[11];
    memcpy(v, r, sizeof(double) * N);
    for (int m = 1; m <= nz; ++m)
        for (int l = 1; l <= n; ++l)
            for (int i = 1; i <= n; ++i) {
                /* visit each line once: at its first node along axis d */
                int coord = (d == 0) ? i : (d == 1 ? l : m);
                if (coord != 1) continue;
                long P0 = node_index(p, i, l, m);
                for (int k = 0; k < n; ++k) {
                    int ii = i, ll = l, mm = m;
                    if (d == 0) ii = k + 1; else if (d == 1) ll = k + 1; else mm = k + 1;
                    orc_row(p, d, ii, ll, mm, row);
                    double lo = (d == 0) ? row[1] : (d == 1 ? row[3] : row[5]);
                    double hi = (d == 0) ? row[2] : (d == 1 ? row[4] : row[6]);
                    a[k] = -tau * lo;
                    b[k] = 1.0 - tau * row[0];
                    c[k] = -tau * hi;
                    x[k] = r[P0 + k * stride];
                }
                thomas(n, a, b, c, x, w);
                for (int k = 0; k < n; ++k) v[P0 + k * stride] = x[k];
            }
    free(a); free(b); free(c); free(x); free(w);
}

/* (I - tau A_j) v = r for DD colour j (2-D): the matrix is block diagonal with one block
 * per connected x-range of nodes where rho_j > 0, identity rows elsewhere
 * (SPEC.md:234).  Each block (width W columns x n rows, x-fastest, bandwidth W) is solved
 * by plain band Gaussian elimination without pivoting (the block is symmetric and strictly
 * diagonally dominant). */
static void solve_dd(const orc_problem *p, int j, double tau, const double *r, double *v) {
    int n = p->n;
    long N = npoints(p);
    memcpy(v, r, sizeof(double) * N);
    int i = 1;
    double row[11];
    while (i <= n) {
        if (!(orc_rho(p, j, (double)i) > 0.0)) { ++i; continue; }
        int i0 = i;
        while (i <= n && orc_rho(p, j, (double)i) > 0.0) ++i;
        int i1 = i - 1;
        int W = i1 - i0 + 1;
        long Nb = (long)W * n;
        int bw = (p->coef == 2) ? W + 1 : W; /* 9-point rows reach q -+ (W +- 1) */
        long ld = 2L * bw + 1;
        double *Ab = calloc((size_t)(Nb * ld), sizeof(double));
        double *bb = malloc(sizeof(double) * Nb);
        /* assemble: block row q = (l-1) W + (ii - i0), band column offset col - q + bw */
        for (int l = 1; l <= n; ++l)
            for (int ii = i0; ii <= i1; ++ii) {
                long q = (long)(l - 1) * W + (ii - i0);
                orc_row(p, j, ii, l, 1, row);
                Ab[q * ld + bw] = 1.0 - tau * row[0];
                if (ii > i0) Ab[q * ld + bw - 1] = -tau * row[1];
                if (ii < i1) Ab[q * ld + bw + 1] = -tau * row[2];
                if (l > 1) Ab[q * ld + bw - W] = -tau * row[3];
                if (l < n) Ab[q * ld + bw + W] = -tau * row[4];
                if (p->coef == 2) {
                    if (ii > i0 && l > 1) Ab[q * ld + bw - W - 1] = -tau * row[7];
                    if (ii < i1 && l > 1) Ab[q * ld + bw - W + 1] = -tau * row[8];
                    if (ii > i0 && l < n) Ab[q * ld + bw + W - 1] = -tau * row[9];
                    if (ii < i1 && l < n) Ab[q * ld + bw + W + 1] = -tau * row[10];
                }
                bb[q] = r[node_index(p, ii, l, 1)];
            }
        /* forward elimination */
        for (long k = 0; k < Nb; ++k) {
            double piv = Ab[k * ld + bw];
            long iend = k + bw < Nb - 1 ? k + bw : Nb - 1;
            for (long q = k + 1; q <= iend; ++q) {
                double f = Ab[q * ld + (k - q + bw)] / piv;
                if (f == 0.0) continue;
                for (long c = k; c <= iend; ++c) Ab[q * ld + (c - q + bw)] -= f * Ab[k * ld + (c - k + bw)];
                bb[q] -= f * bb[k];
            }
        }
        /* back substitution */
        for (long k = Nb - 1; k >= 0; --k) {
            double s = bb[k];
            long cend = k + bw < Nb - 1 ? k + bw : Nb - 1;
            for (long c = k + 1; c <= cend; ++c) s -= Ab[k * ld + (c - k + bw)] * bb[c];
            bb[k] = s / Ab[k * ld + bw];
        }
        for (int l = 1; l <= n; ++l)
            for (int ii = i0; ii <= i1; ++ii) v[node_index(p, ii, l, 1)] = bb[(long)(l - 1) * W + (ii - i0)];
        free(Ab);
        free(bb);
    }
}

int orc_nterms(const orc_problem *p) { return p->split == 1 ? 2 : p->dim; }

/* (I - tau A_term) v = r */
void orc_solve(const orc_problem *p, int term, double tau, const double *r, double *v) {
    if (p->split == 1) solve_dd(p, term, tau, r, v);
    else solve_dim(p, term, tau, r, v);
}

/* ----------------------------------------------------------- integrators -- */
/* FIE, eq. FIE_method:
 *   (I - tau A_1) U_{n,1} = U_n + tau F_{n+1};  (I - tau A_j) U_{n,j} = U_{n,j-1};  U_{n+1} = U_{n,M}. */
static void fie_step(const orc_problem *p, double tau, double t_next, const double *u, double *out) {
    long N = npoints(p);
    int M = orc_nterms(p);
    double *r = malloc(sizeof(double) * N), *F = malloc(sizeof(double) * N);
    orc_source(p, t_next, F);
    for (long k = 0; k < N; ++k) r[k] = u[k] + tau * F[k];
    for (int j = 0; j < M; ++j) {
        orc_solve(p, j, tau, r, out);
        if (j < M - 1) memcpy(r, out, sizeof(double) * N);
    }
    free(r); free(F);
}

/* DR, eq. DR_method, literally:
 *   U_{n,0} = (I + tau A) U_n + tau F_{n+1};
 *   (I - tau A_j) U_{n,j} = U_{n,j-1} - tau A_j U_n,  j = 1..M;  U_{n+1} = U_{n,M}. */
static void dr_step(const orc_problem *p, double tau, double t_next, const double *u, double *out) {
    long N = npoints(p);
    int M = orc_nterms(p);
    double *prev = malloc(sizeof(double) * N), *F = malloc(sizeof(double) * N),
           *Au = malloc(sizeof(double) * N), *rhs = malloc(sizeof(double) * N);
    orc_source(p, t_next, F);
    orc_apply(p, -1, u, Au);
    for (long k = 0; k < N; ++k) prev[k] = (u[k] + tau * Au[k]) + tau * F[k];
    for (int j = 0; j < M; ++j) {
        orc_apply(p, j, u, Au);
        for (long k = 0; k < N; ++k) rhs[k] = prev[k] - tau * Au[k];
        orc_solve(p, j, tau, rhs, out);
        if (j < M - 1) memcpy(prev, out, sizeof(double) * N);
    }
    free(prev); free(F); free(Au); free(rhs);
}

/* Unsplit implicit Euler (the Parareal/IE-IE baseline of PAPER.md:455):
 *   (I - tau A) U_{n+1} = U_n + tau F_{n+1},  A the unsplit operator (term -1).
 * Plain band Gaussian elimination (no pivoting: I - tau A is an M-matrix, diagonally dominant)
 * of the whole n^dim system in node order, half bandwidth n (2-D 5-point), n + 1 (2-D 9-point
 * full tensor) or n^2 (3-D 7-point); factorised on the fly.  O(n^dim bw^2): tiny grids only. */
static void ie_step(const orc_problem *p, double tau, double t_next, const double *u, double *out) {
    int n = p->n, nz = (p->dim == 3) ? n : 1;
    long Nb = npoints(p), sy = n, sz = (long)n * n;
    long bw = (p->dim == 3) ? sz : (p->coef == 2 ? n + 1 : n);
    long ld = 2 * bw + 1;
    double *Ab = calloc((size_t)(Nb * ld), sizeof(double));
    double *F = malloc(sizeof(double) * Nb);
    double row[11];
    orc_source(p, t_next, F);
    for (long k = 0; k < Nb; ++k) out[k] = u[k] + tau * F[k];
    for (int m = 1; m <= nz; ++m)
        for (int l = 1; l <= n; ++l)
            for (int i = 1; i <= n; ++i) {
                long q = node_index(p, i, l, m);
                orc_row(p, -1, i, l, m, row);
                Ab[q * ld + bw] = 1.0 - tau * row[0];
                if (i > 1) Ab[q * ld + bw - 1] = -tau * row[1];
                if (i < n) Ab[q * ld + bw + 1] = -tau * row[2];
                if (l > 1) Ab[q * ld + bw - sy] = -tau * row[3];
                if (l < n) Ab[q * ld + bw + sy] = -tau * row[4];
                if (p->dim == 3) {
                    if (m > 1) Ab[q * ld + bw - sz] = -tau * row[5];
                    if (m < n) Ab[q * ld + bw + sz] = -tau * row[6];
                }
                if (p->coef == 2) {
                    if (i > 1 && l > 1) Ab[q * ld + bw - sy - 1] = -tau * row[7];
                    if (i < n && l > 1) Ab[q * ld + bw - sy + 1] = -tau * row[8];
                    if (i > 1 && l < n) Ab[q * ld + bw + sy - 1] = -tau * row[9];
                    if (i < n && l < n) Ab[q * ld + bw + sy + 1] = -tau * row[10];
                }
            }
    /* forward elimination */
    for (long k = 0; k < Nb; ++k) {
        double piv = Ab[k * ld + bw];
        long iend = k + bw < Nb - 1 ? k + bw : Nb - 1;
        for (long q = k + 1; q <= iend; ++q) {
            double f = Ab[q * ld + (k - q + bw)] / piv;
            if (f == 0.0) continue;
            for (long c = k; c <= iend; ++c) Ab[q * ld + (c - q + bw)] -= f * Ab[k * ld + (c - k + bw)];
            out[q] -= f * out[k];
        }
    }
    /* back substitution */
    for (long k = Nb - 1; k >= 0; --k) {
        double s = out[k];
        long cend = k + bw < Nb - 1 ? k + bw : Nb - 1;
        for (long c = k + 1; c <= cend; ++c) s -= Ab[k * ld + (c - k + bw)] * out[c];
        out[k] = s / Ab[k * ld + bw];
    }
    free(Ab);
    free(F);
}

/* one step of scheme (0 FIE, 1 DR, 2 IE) of size tau; the source is sampled at t_next = t_{n+1} */
void orc_step(const orc_problem *p, int scheme, double tau, double t_next, const double *u, double *out) {
    if (scheme == 2) ie_step(p, tau, t_next, u, out);
    else if (scheme == 1) dr_step(p, tau, t_next, u, out);
    else fie_step(p, tau, t_next, u, out);
}

/* ------------------------------------------------------------ propagators -- */
/* Time grid: Delta T = T/N_c, delta t = T/(s N_c), t_{ns+j} = (ns+j) delta t,
 * T_n = n Delta T.  Times are formed as (integer index) * step (reading R2). */
static double coarse_dt(const orc_problem *p) { return p->T / (double)p->N; }
static double fine_dt(const orc_problem *p) { return p->T / ((double)p->N * (double)p->s); }

/* G_{Delta T}(T_n, T_{n+1}, v): one step */
void orc_coarse(const orc_problem *p, int slice, const double *v, double *out) {
    orc_step(p, p->G, coarse_dt(p), (double)(slice + 1) * coarse_dt(p), v, out);
}

/* F^s_{delta t}(T_n, T_{n+1}, v): s fine steps */
void orc_fine(const orc_problem *p, int slice, const double *v, double *out) {
    long N = npoints(p);
    double *cur = malloc(sizeof(double) * N), *nxt = malloc(sizeof(double) * N);
    memcpy(cur, v, sizeof(double) * N);
    double dt = fine_dt(p);
    for (int j = 0; j < p->s; ++j) {
        double t_next = (double)((long)slice * p->s + j + 1) * dt;
        orc_step(p, p->F, dt, t_next, cur, nxt);
        double *tmp = cur; cur = nxt; nxt = tmp;
    }
    memcpy(out, cur, sizeof(double) * N);
    free(cur); free(nxt);
}

/* -------------------------------------------------------------- parareal -- */
/* Initial guess U^0_0 = P u_0, U^0_{n+1} = G(U^0_n).
 * traj holds N+1 states of npts values. */
void orc_coarse_sweep(const orc_problem *p, const double *u0, double *traj) {
    long N = npoints(p);
    memcpy(traj, u0, sizeof(double) * N);
    for (int n = 0; n < p->N; ++n) orc_coarse(p, n, traj + (long)n * N, traj + (long)(n + 1) * N);
}

/* One parareal iteration k -> k+1:
 *   U^{k+1}_0 = P u_0,
 *   U^{k+1}_{n+1} = G(U^{k+1}_n) + F^s(U^k_n) - G(U^k_n),  n = 0..N_c-1.
 * The F^s(U^k_n) are independent in n; computed serially here. */
static int orc_threads = 1;
void orc_set_threads(int k) { orc_threads = k < 1 ? 1 : k; }

typedef struct {
    const orc_problem *p;
    const double *traj_k;
    double *Fk, *Gk;
    int next;  /* next slice to take (under lock) */
    pthread_mutex_t lock;
} slice_work;

static void *slice_worker(void *arg) {
    slice_work *w = (slice_work *)arg;
    long N = npoints(w->p);
    for (;;) {
        pthread_mutex_lock(&w->lock);
        int n = w->next++;
        pthread_mutex_unlock(&w->lock);
        if (n >= w->p->N) return NULL;
        orc_fine(w->p, n, w->traj_k + (long)n * N, w->Fk + (long)n * N);
        orc_coarse(w->p, n, w->traj_k + (long)n * N, w->Gk + (long)n * N);
    }
}

void orc_parareal_iteration(const orc_problem *p, const double *traj_k, double *traj_k1) {
    long N = npoints(p);
    int Nc = p->N;
    double *Fk = malloc(sizeof(double) * N * Nc), *Gk = malloc(sizeof(double) * N * Nc);
    double *g = malloc(sizeof(double) * N);
    /* F^s(U^k_n), G(U^k_n) for every n (independent slices; serial when orc_threads == 1) */
    slice_work w = {p, traj_k, Fk, Gk, 0};
    pthread_mutex_init(&w.lock, NULL);
    int nt = orc_threads < Nc ? orc_threads : Nc;
    pthread_t th[256];
    if (nt > 256) nt = 256;
    for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, slice_worker, &w);
    slice_worker(&w);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&w.lock);
    memcpy(traj_k1, traj_k, sizeof(double) * N); /* U^{k+1}_0 = U^k_0 = P u_0 */
    for (int n = 0; n < Nc; ++n) {
        orc_coarse(p, n, traj_k1 + (long)n * N, g);
        double *dst = traj_k1 + (long)(n + 1) * N;
        const double *fk = Fk + (long)n * N, *gk = Gk + (long)n * N;
        for (long q = 0; q < N; ++q) dst[q] = (g[q] + fk[q]) - gk[q];
    }
    free(Fk); free(Gk); free(g);
}

/* Sequential fine solution at the coarse points: U^F_{n+1} = F^s(U^F_n). */
void orc_fine_solution(const orc_problem *p, const double *u0, double *traj) {
    long N = npoints(p);
    memcpy(traj, u0, sizeof(double) * N);
    for (int n = 0; n < p->N; ++n) orc_fine(p, n, traj + (long)n * N, traj + (long)(n + 1) * N);
}
