/* abi_smoke.c -- a plain C client of include/prs.h (no Python, no torch): proves the C ABI
 * independently of the ctypes binding.  Builds a small problem, runs the coarse sweep and
 * parareal to a tolerance, and writes k, the update history and U^k_N (host buffers) to a
 * binary file for the GPU test to compare with the CPU oracle.
 *
 *   abi_smoke <out.bin>     exit 0 on success, 1 on a library error (message on stderr)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "prs.h"

#define PI_ 3.14159265358979323846

#define CHECK(call)                                                                   \
    do {                                                                              \
        int rc_ = (call);                                                             \
        if (rc_ != PRS_OK) {                                                          \
            fprintf(stderr, "%s failed: %d (%s)\n", #call, rc_, ctx ? prs_last_error(ctx) : ""); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

int main(int argc, char **argv) {
    if (argc < 2) return 2;
    prs_problem p = {0};
    p.dim = 2;
    p.n = 48;
    p.c = 1.0;
    p.coef_kind = 1; /* kappa = 1 + 0.5 sin(2 pi x) sin(2 pi y) */
    p.split = 0;
    p.source_kind = 1;
    p.T = 1.0;
    p.N = 6;
    p.s = 5;
    p.G = PRS_FIE;
    p.F = PRS_DR;
    prs_ctx *ctx = NULL;
    const int n = p.n, npts = n * n;
    double *u0 = malloc(sizeof(double) * npts), *out = malloc(sizeof(double) * npts);
    double hist[6];
    int k = 0;
    /* U_0 = sin(pi x) sin(pi y) at the interior nodes (x-fastest) */
    const double h = 1.0 / (n + 1);
    for (int l = 0; l < n; ++l)
        for (int i = 0; i < n; ++i) u0[l * n + i] = sin(PI_ * (i + 1) * h) * sin(PI_ * (l + 1) * h);
    CHECK(prs_create(&p, 0, 1, NULL, NULL, &ctx));
    CHECK(prs_set_initial(ctx, u0, 0));
    CHECK(prs_coarse_sweep(ctx));
    CHECK(prs_iterate(ctx, p.N, 1e-9, &k, hist));
    CHECK(prs_get_slice(ctx, p.N, out, 0));
    prs_destroy(ctx);
    FILE *f = fopen(argv[1], "wb");
    if (!f) return 1;
    fwrite(&k, sizeof(int), 1, f);
    fwrite(hist, sizeof(double), (size_t)k, f);
    fwrite(out, sizeof(double), (size_t)npts, f);
    fclose(f);
    printf("abi_smoke: k = %d, last update %.3e\n", k, k ? hist[k - 1] : 0.0);
    free(u0);
    free(out);
    return 0;
}
