/* oracle_problem.h -- TEST INFRASTRUCTURE ONLY (see oracle.c).  Private to oracle/;
 * the CUDA library has its own, unrelated header (include/prs.h). */
#ifndef ORACLE_PROBLEM_H
#define ORACLE_PROBLEM_H

typedef struct {
    int dim;        /* 2 or 3 spatial dimensions (unit square / cube)                 */
    int n;          /* interior nodes per axis, h = 1/(n+1)                           */
    double c;       /* reaction coefficient c > 0                        */
    int coef;       /* 0: kappa = 1;  1: kappa = 1 + 0.5 sin(2 pi x) sin(2 pi y);
                       2: full tensor d11 = d22 = 1/(2 + cos 3pi x cos 2pi y), d12 = 1/4
                          (2-D, DD splitting only)                       */
    int split;      /* 0: dimensional; 1: domain decomposition (2-D)  */
    int dd_strips;  /* DD: total number of vertical strips (2q)           */
    int dd_overlap; /* DD: overlap width beta in cells                                 */
    int dd_ramp;    /* DD: 0 linear ramp, 1 cosine ramp                                */
    int source;     /* 0: f = 0;  1: manufactured f for u = e^{-t} prod sin(pi x_d);   */
                    /* 2: f for u = sin(2 pi t) sin(2 pi x) sin(2 pi y) (2-D, D = I) */
    double T;       /* final time                                                      */
    int N;          /* coarse slices N_c                                               */
    int s;          /* fine steps per slice                                            */
    int G, F;       /* scheme of the coarse / fine propagator: 0 FIE, 1 DR, 2 IE      */
} orc_problem;

#endif
