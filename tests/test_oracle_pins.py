"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the pin and the passage it follows.
"""
from __future__ import annotations

import math
import os

import mpmath as mp
import numpy as np
import pytest

import oracle
import synth
from synth import DR, FIE, Problem
from tests import modal

GOLD = {}
with open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.txt")) as fh:
    for line in fh:
        line = line.split("#")[0].strip()
        if line:
            k, v = line.split("=")
            GOLD[k.strip()] = float(v)


def nrm_err(a, b, scale):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / scale


# ---------------------------------------------------------------- P4 scalars
def one_point(dim=2, c=0.0, **kw):
    # n = 1, h = 1/2: every dimensional A_d is the 1x1 matrix -(8 + c/M)  (mu_1 = 16 sin^2(pi/4))
    return Problem(dim=dim, n=1, c=c, source=0, **kw)


@pytest.mark.parametrize("scheme,key", [(FIE, "r_fie_m1_m1"), (DR, "r_dr_m1_m1")])
def test_stability_values_one_point(scheme, key):
    """P4: one step on a 1-point grid, z_j = tau * (-8) = -1."""
    o = oracle.Oracle(one_point())
    out = o.step(scheme, 1.0 / 8.0, 0.125, np.ones(1))
    assert abs(out.item() - GOLD[key]) <= 1e-15


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("scheme", [FIE, DR])
def test_stability_functions_general_z(dim, scheme):
    """P4: R_FIE / R_DR for M = 2, 3 at several z (general M)."""
    for c in (0.0, 1.0, 7.5):
        for tau in (1e-3, 0.05, 0.7, 13.0):
            o = oracle.Oracle(one_point(dim=dim, c=c))
            zs = [mp.mpf(tau) * (-(8 + mp.mpf(c) / dim))] * dim
            want = modal.r_fie(zs) if scheme == FIE else modal.r_dr(zs)
            got = o.step(scheme, tau, tau, np.ones(1)).item()
            assert abs(got - float(want)) <= 1e-14 * max(1.0, abs(float(want)))


def test_dr_reduces_to_backward_euler_when_A2_is_zero():
    """P4/P11: R_DR(z, 0) = 1/(1-z); a one-strip DD split has rho_1 = 1,
    so A_1 = A and A_2 = 0."""
    p = Problem(dim=2, n=1, c=2.0, split=1, dd_strips=1, dd_overlap=0, source=0)
    o = oracle.Oracle(p)
    tau = 0.3
    z = tau * -(16.0 + 2.0)  # A = -(2*8 + c) on the 1-point grid
    got = o.step(DR, tau, tau, np.ones(1)).item()
    assert abs(got - 1.0 / (1.0 - z)) <= 1e-15
    assert abs(o.step(FIE, tau, tau, np.ones(1)).item() - 1.0 / (1.0 - z)) <= 1e-15


def test_fie_sweep_and_dahlquist_coarse_values():
    """P4: FIE sweep s = 4 at z = -1/4 per term gives 0.64^4 (SPEC.md:222 erratum, R18);
    two coarse FIE steps at z = -1 give 1/16."""
    # delta t = T/(N s) = 1/32, lambda = -8 -> z = -1/4
    o = oracle.Oracle(one_point(T=0.125, N=1, s=4))
    assert abs(o.fine(0, np.ones(1)).item() - GOLD["fie_sweep_s4_tau_quarter"]) <= 1e-15
    # Delta T = 1/8 -> z = -1
    o = oracle.Oracle(one_point(T=0.25, N=2, s=1))
    tr = o.coarse_sweep(np.ones(1))
    assert abs(tr[2].item() - GOLD["coarse_dahlquist_U2"]) <= 1e-16


# ------------------------------------------------------ operator: eigenpairs
@pytest.mark.parametrize("dim,n", [(2, 7), (2, 16), (3, 6)])
def test_dimensional_terms_have_sine_eigenpairs(dim, n):
    """Pins the stencil rows: A_d sin(j pi x) = -(mu_j + c/M) sin(j pi x) (PAPER.md:237-250,
    discrete Dirichlet sine basis)."""
    c = 1.3
    p = Problem(dim=dim, n=n, c=c)
    o = oracle.Oracle(p)
    rng = np.random.default_rng(1)
    for _ in range(4):
        modes = tuple(int(m) for m in rng.integers(1, n + 1, size=dim))
        vecs = [np.array(modal.sines(n, m)) for m in modes]
        if dim == 2:
            u = np.outer(vecs[1], vecs[0])
        else:
            u = vecs[2][:, None, None] * vecs[1][None, :, None] * vecs[0][None, None, :]
        lam = [float(v) for v in modal.lambdas(modes, n, c, dim)]
        for d in range(dim):
            got = o.apply(d, u)
            assert nrm_err(got, lam[d] * u, abs(lam[d])) <= 2e-13
        got = o.apply(-1, u)
        lam_full = sum(lam)
        assert nrm_err(got, lam_full * u, abs(lam_full)) <= 2e-13


# ------------------------------------------------ P10: spatial consistency
def _lu_exact_variable_kappa(x, y, c):
    # u = sin(pi x) sin(2 pi y); kappa = 1 + 0.5 sin(2 pi x) sin(2 pi y)
    pi = math.pi
    u = np.sin(pi * x) * np.sin(2 * pi * y)
    ux = pi * np.cos(pi * x) * np.sin(2 * pi * y)
    uy = 2 * pi * np.sin(pi * x) * np.cos(2 * pi * y)
    lap = -(pi ** 2 + 4 * pi ** 2) * u
    k = 1 + 0.5 * np.sin(2 * pi * x) * np.sin(2 * pi * y)
    kx = pi * np.cos(2 * pi * x) * np.sin(2 * pi * y)
    ky = pi * np.sin(2 * pi * x) * np.cos(2 * pi * y)
    return u, k * lap + kx * ux + ky * uy - c * u


def test_variable_kappa_operator_is_second_order():
    """P10: ||A u - L u||_inf = O(h^2) for div(kappa grad u) - c u."""
    errs, hs = [], []
    for n in (31, 63, 127):
        p = Problem(dim=2, n=n, c=1.0, coef=1)
        o = oracle.Oracle(p)
        h = 1.0 / (n + 1)
        xs = h * np.arange(1, n + 1)
        X, Y = np.meshgrid(xs, xs)  # X varies along axis 1 (x-fastest)
        u, lu = _lu_exact_variable_kappa(X, Y, 1.0)
        errs.append(np.max(np.abs(o.apply(-1, u) - lu)))
        hs.append(h)
    slope = np.polyfit(np.log(hs), np.log(errs), 1)[0]
    assert 1.8 <= slope <= 2.2, (errs, slope)


# -------------------------------------------- P6 / P9: exactness, M-matrix
SPLIT_CASES = [
    Problem(dim=2, n=9, c=1.0),
    Problem(dim=2, n=9, c=1.0, coef=1),
    Problem(dim=3, n=5, c=1.0),
    Problem(dim=2, n=32, c=1.0, split=1, dd_strips=4, dd_overlap=4, dd_ramp=0),
    Problem(dim=2, n=32, c=1.0, split=1, dd_strips=4, dd_overlap=4, dd_ramp=1),
    Problem(dim=2, n=32, c=1.0, coef=1, split=1, dd_strips=8, dd_overlap=2, dd_ramp=0),
]


@pytest.mark.parametrize("p", SPLIT_CASES, ids=lambda p: p.label() + f"_k{p.coef}_r{p.dd_ramp}")
def test_split_exactness_and_m_matrix(p):
    """P6: sum_j A_j = A to 1e-13.  P9: I - tau A_j symmetric,
    non-positive off-diagonals, strictly diagonally dominant."""
    o = oracle.Oracle(p)
    A = o.dense(-1)
    terms = [o.dense(j) for j in range(o.nterms())]
    assert np.max(np.abs(sum(terms) - A)) <= 1e-13 * np.max(np.abs(A))
    for Aj in terms:
        B = np.eye(A.shape[0]) - 0.01 * Aj
        assert np.array_equal(B, B.T)
        off = B - np.diag(np.diag(B))
        assert np.all(off <= 0.0)
        assert np.all(np.diag(B) - np.sum(np.abs(off), axis=1) >= 1.0 - 1e-12)


def test_dimensional_terms_commute_dd_terms_do_not():
    """constant-coefficient dimensional terms commute; DD terms do not."""
    o = oracle.Oracle(Problem(dim=2, n=8, c=1.0))
    A1, A2 = o.dense(0), o.dense(1)
    assert np.max(np.abs(A1 @ A2 - A2 @ A1)) <= 1e-10 * np.max(np.abs(A1)) * np.max(np.abs(A2))
    o = oracle.Oracle(SPLIT_CASES[3])
    A1, A2 = o.dense(0), o.dense(1)
    assert np.max(np.abs(A1 @ A2 - A2 @ A1)) > 1e-3 * np.max(np.abs(A1)) * np.max(np.abs(A2))


# ------------------------------------------------------------ P7 partition
@pytest.mark.parametrize("ramp", [0, 1])
def test_partition_of_unity(ramp):
    """P7: rho_1 + rho_2 = 1 exactly, 0 <= rho <= 1, supp rho_j in Omega_j;
    linear ramp node values are (2k+1)/16 (R6)."""
    n, S, ov = 1024, 8, 8
    p = Problem(dim=2, n=n, split=1, dd_strips=S, dd_overlap=ov, dd_ramp=ramp)
    o = oracle.Oracle(p)
    w = n // S
    pos = np.arange(1, 2 * n + 2) * 0.5  # all nodes and faces 0.5 .. n + 0.5
    r0 = np.array([o.rho(0, x) for x in pos])
    r1 = np.array([o.rho(1, x) for x in pos])
    assert np.all(r0 + r1 == 1.0)
    assert np.all((r0 >= 0) & (r0 <= 1))
    for x, v in zip(pos, r0):
        k = min(int((x - 0.5) // w), S - 1)
        d_left = x - (w * k + 0.5)
        d_right = (w * (k + 1) + 0.5) - x
        near = (k > 0 and d_left < ov / 2) or (k < S - 1 and d_right < ov / 2)
        if not near:
            assert v == (1.0 if k % 2 == 0 else 0.0)
    if ramp == 0:
        m = 3
        vals = [o.rho(0, float(w * m + d)) for d in range(-3, 5)]
        # interface 3 lies between strip 2 (colour 0) and strip 3 (colour 1): descending
        assert vals == [(2 * k + 1) / 16 for k in range(7, -1, -1)]
    else:
        assert o.rho(0, w * 1 + 0.5) == pytest.approx(0.5, abs=1e-15)
    # every node and face of every ramp against the ramp written out here: across interface m
    # (face w m + 1/2) the colour of the strip on the left falls from 1 at x_l = w m + 1/2 - beta/2
    # to 0 at x_l + beta, linearly (BASELINE c4) or as (1 + cos(pi u))/2,
    # u = (x - x_l)/beta; it is colour 0 when the left strip is even (R6)
    for m in range(1, S):
        xl = w * m + 0.5 - ov / 2
        for d2 in range(0, 2 * ov + 1):
            x = xl + 0.5 * d2
            u = (x - xl) / ov
            down = (1.0 - u) if ramp == 0 else 0.5 * (1.0 + math.cos(math.pi * u))
            want = down if (m - 1) % 2 == 0 else 1.0 - down
            assert abs(o.rho(0, x) - want) <= 2e-16, (m, x)
            assert abs(o.rho(1, x) - (1.0 - want)) <= 2e-16, (m, x)


# -------------------------------------------------- P5 dense solves
DENSE_CASES = [
    Problem(dim=2, n=3, c=1.0), Problem(dim=2, n=8, c=1.0), Problem(dim=2, n=7, c=1.0, coef=1),
    Problem(dim=3, n=4, c=1.0), Problem(dim=3, n=5, c=2.0),
    Problem(dim=2, n=32, c=1.0, split=1, dd_strips=4, dd_overlap=4, dd_ramp=0),
    Problem(dim=2, n=32, c=1.0, split=1, dd_strips=4, dd_overlap=4, dd_ramp=1),
    Problem(dim=2, n=24, c=1.0, coef=1, split=1, dd_strips=8, dd_overlap=2, dd_ramp=0),
]


@pytest.mark.parametrize("p", DENSE_CASES, ids=lambda p: p.label() + f"_k{p.coef}_r{p.dd_ramp}")
def test_stage_solves_match_dense_lu(p):
    """P5: each stage solve (Thomas / band elimination / identity rows) equals a dense
    partial-pivoting LU solve of I - tau A_j (numpy.linalg.solve) to 1e-14."""
    o = oracle.Oracle(p)
    rng = np.random.default_rng(7)
    for tau in (1e-3, 0.03, 1.0):
        for j in range(o.nterms()):
            r = rng.standard_normal(o.shape)
            B = np.eye(o.npts) - tau * o.dense(j)
            want = np.linalg.solve(B, r.ravel())
            got = o.solve(j, tau, r).ravel()
            assert nrm_err(got, want, np.max(np.abs(want))) <= 1e-14


@pytest.mark.parametrize("p", DENSE_CASES[:2] + DENSE_CASES[3:4] + DENSE_CASES[5:6],
                         ids=lambda p: p.label())
def test_steps_match_dense_matrix_form(p):
    """FIE / DR steps written as dense products of the paper's formulas
     with numpy.linalg.solve as the stage solver."""
    p = p.replace(source=1)
    o = oracle.Oracle(p)
    rng = np.random.default_rng(3)
    u = rng.standard_normal(o.shape).ravel()
    tau, t1 = 0.02, 0.37
    I = np.eye(o.npts)
    A = o.dense(-1)
    F = o.source(t1).ravel()
    terms = [o.dense(j) for j in range(o.nterms())]
    v = u + tau * F
    for Aj in terms:
        v = np.linalg.solve(I - tau * Aj, v)
    assert nrm_err(o.step(FIE, tau, t1, u).ravel(), v, np.max(np.abs(v))) <= 1e-13
    v = u + tau * (A @ u) + tau * F
    for Aj in terms:
        v = np.linalg.solve(I - tau * Aj, v - tau * (Aj @ u))
    assert nrm_err(o.step(DR, tau, t1, u).ravel(), v, np.max(np.abs(v))) <= 1e-13


# ----------------------------------------------------------- source term
def test_manufactured_source_values():
    """F(t) = (d pi^2 + c - 1) e^{-t} prod sin(pi x_d) at the nodes (BASELINE c0)."""
    for dim, n in ((2, 5), (3, 4)):
        p = Problem(dim=dim, n=n, c=1.7, source=1)
        o = oracle.Oracle(p)
        h = 1.0 / (n + 1)
        t = 0.3
        F = o.source(t)
        idx = (1,) * dim
        want = (dim * math.pi ** 2 + 0.7) * math.exp(-t) * math.sin(2 * math.pi * h) ** dim
        assert F[idx] == pytest.approx(want, rel=1e-14)


# ------------------------------------------------------- P1 modal closed form
def test_c0_modal_closed_form_all_iterations():
    """P1: c0 every parareal iterate equals a^k_n * phi where a^k_n is the scalar FIE-FIE
    parareal recurrence of mode (1,1), evaluated in mpmath."""
    p = synth.CONFIGS["c0"]
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    trajs, _ = o.parareal(u0, p.N, fixed=True)
    lam = modal.lambdas((1, 1), p.n, p.c, 2)
    sp = modal.ScalarParareal(lam, p.T, p.N, p.s, FIE, FIE, src_amp=2 * mp.pi ** 2 + p.c - 1)
    want = sp.run(1, p.N)
    for k in range(p.N + 1):
        for n in range(p.N + 1):
            assert nrm_err(trajs[k][n], float(want[k][n]) * u0, 1.0) <= 1e-13, (k, n)


def test_random_modes_dr_dr_modal_closed_form():
    """P1: DR-DR parareal on random-mode data (the c1 recipe on a 32^2 grid) equals the
    superposition of per-mode scalar DR-DR parareal recurrences."""
    p = Problem(dim=2, n=32, c=1.0, source=0, N=6, s=5, G=DR, F=DR, init="modes", seed=1)
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    trajs, _ = o.parareal(u0, 3, fixed=True)
    table = synth.mode_table(p.seed)
    scale = max(np.max(np.abs(t)) for t in trajs)
    per_mode = []
    for j, l, a in table:
        lam = modal.lambdas((j, l), p.n, p.c, 2)
        sp = modal.ScalarParareal(lam, p.T, p.N, p.s, DR, DR)
        per_mode.append((np.outer(modal.sines(p.n, l), modal.sines(p.n, j)), a, sp.run(1, 3)))
    for k in range(4):
        for n in range(p.N + 1):
            want = sum(a * float(r[k][n]) * sh for sh, a, r in per_mode)
            assert nrm_err(trajs[k][n], want, scale) <= 1e-13, (k, n)


def test_3d_fie_modal_closed_form():
    """P1 for the 3-D, M = 3 FIE-FIE path (c2 recipe on a 12^3 grid)."""
    p = Problem(dim=3, n=12, c=1.0, source=1, N=4, s=3, G=FIE, F=FIE, init="phi")
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    trajs, _ = o.parareal(u0, 2, fixed=True)
    lam = modal.lambdas((1, 1, 1), p.n, p.c, 3)
    sp = modal.ScalarParareal(lam, p.T, p.N, p.s, FIE, FIE, src_amp=3 * mp.pi ** 2 + p.c - 1)
    want = sp.run(1, 2)
    for k in range(3):
        for n in range(p.N + 1):
            assert nrm_err(trajs[k][n], float(want[k][n]) * u0, 1.0) <= 1e-13


# ---------------------------------------------------- P2 finite termination
FT_CASES = [
    Problem(dim=2, n=10, N=4, s=3, G=FIE, F=FIE, source=1),
    Problem(dim=2, n=10, N=4, s=3, G=DR, F=DR, init="modes"),
    Problem(dim=2, n=10, N=4, s=3, G=FIE, F=DR, coef=1, init="random"),
    Problem(dim=2, n=10, N=4, s=3, G=DR, F=FIE, coef=1, init="random"),
    Problem(dim=3, n=6, N=3, s=2, G=FIE, F=FIE, source=1),
    Problem(dim=2, n=16, N=4, s=2, split=1, dd_strips=4, dd_overlap=2, G=FIE, F=FIE, source=1),
    Problem(dim=2, n=16, N=4, s=2, split=1, dd_strips=4, dd_overlap=2, G=FIE, F=DR, source=1),
    Problem(dim=2, n=16, N=4, s=2, split=1, dd_strips=4, dd_overlap=2, G=DR, F=FIE, source=1),
    Problem(dim=2, n=16, N=4, s=2, split=1, dd_strips=4, dd_overlap=2, G=DR, F=DR, source=1),
]


@pytest.mark.parametrize("p", FT_CASES, ids=lambda p: p.label())
def test_finite_termination(p):
    """P2: after N_c iterations parareal equals the sequential fine solution,
    and slices n <= k are fixed from iteration k on."""
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    fine = o.fine_solution(u0)
    trajs, _ = o.parareal(u0, p.N, fixed=True)
    scale = max(max(np.max(np.abs(t)) for t in trajs), np.max(np.abs(u0)))
    assert nrm_err(trajs[p.N], fine, scale) <= 1e-12
    for k in range(1, p.N + 1):
        assert nrm_err(trajs[k][: k + 1], fine[: k + 1], scale) <= 1e-12


def test_g_equals_f_converges_in_one_iteration():
    """P11: G = F with s = 1 -- the correction telescopes, U^1 = fine."""
    for sch in (FIE, DR):
        p = Problem(dim=2, n=9, N=5, s=1, G=sch, F=sch, source=1, coef=1)
        o = oracle.Oracle(p)
        u0 = synth.initial_state(p)
        trajs, _ = o.parareal(u0, 1, fixed=True)
        assert nrm_err(trajs[1], o.fine_solution(u0), 1.0) <= 1e-14


def test_zero_operator_and_source_is_identity():
    """P11: A = 0 (one-point DD colour with rho = 0 support) and F = 0 -> identity
    (SPEC.md:194).  Here A_2 = 0 on a one-strip decomposition."""
    p = Problem(dim=2, n=4, c=1.0, split=1, dd_strips=1, dd_overlap=0)
    o = oracle.Oracle(p)
    u = np.random.default_rng(0).standard_normal(o.shape)
    assert np.array_equal(o.solve(1, 0.5, u), u)
    assert np.all(o.apply(1, u) == 0.0)


# --------------------------------------------------- P3 convergence factor
def test_paper_proof_constants():
    """P14: H(0,0) = 4, H(-3,-3) = 16(1 + 3/e^6); DR: 2, 4(1 + 1/e^2)
    (PAPER.md:380); K_FIE-FIE(-1,-1,1000) <= 1/3;
    K_FIE-DR(-1e4,-1e4,20) < 1."""
    H = lambda z1, z2: (1 - z1) * (1 - z2) * (3 * mp.exp(z1 + z2) + 1)
    Hdr = lambda z1, z2: (1 - z1) * (1 - z2) * (mp.exp(z1 + z2) + 1)
    assert float(H(0, 0)) == GOLD["h_fie_0_0"]
    assert float(H(-3, -3)) == pytest.approx(GOLD["h_fie_m3_m3"], rel=1e-15)
    assert float(Hdr(0, 0)) == GOLD["h_dr_0_0"]
    assert float(Hdr(-1, -1)) == pytest.approx(GOLD["h_dr_m1_m1"], rel=1e-15)
    k1 = float(modal.conv_factor([mp.mpf(-1), mp.mpf(-1)], 1000))
    assert k1 <= GOLD["k_fie_fie_bound"] and k1 == pytest.approx(0.15271, abs=5e-5)
    k2 = float(modal.conv_factor([mp.mpf(-1e4)] * 2, 20, "FIE", "DR"))
    assert 0.9 < k2 < GOLD["k_fie_dr_bound"]


def test_observed_contraction_respects_convergence_factor_c0():
    """P3: sup_n |y^F_n - y^k_n| <= K^k sup_n |y^F_n - y^0_n| per mode,
    with K <= 1/3 for FIE-FIE -- c0 config."""
    p = synth.CONFIGS["c0"]
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    fine = o.fine_solution(u0)
    trajs, _ = o.parareal(u0, p.N, fixed=True)
    dT = mp.mpf(p.T) / p.N
    lam = modal.lambdas((1, 1), p.n, p.c, 2)
    K = float(modal.conv_factor([dT * l for l in lam], p.s))
    assert K <= 1.0 / 3.0
    e0 = np.max(np.abs(trajs[0][1:] - fine[1:]))
    for k in range(1, p.N + 1):
        ek = np.max(np.abs(trajs[k][1:] - fine[1:]))
        assert ek <= K ** k * e0 * (1 + 1e-9) + 1e-15


def test_dd_fie_g_error_decreases():
    """P3 (DD): the theory does not apply directly; the error vs fine still
    decreases for the FIE-G pairings."""
    for F in (FIE, DR):
        p = Problem(dim=2, n=32, N=8, s=4, split=1, dd_strips=4, dd_overlap=4, G=FIE, F=F, source=1)
        o = oracle.Oracle(p)
        u0 = synth.initial_state(p)
        fine = o.fine_solution(u0)
        trajs, _ = o.parareal(u0, 5, fixed=True)
        errs = [np.max(np.abs(t - fine)) for t in trajs]
        assert all(b < a for a, b in zip(errs, errs[1:])), errs


# --------------------------------------------------- P8 temporal order
def test_first_order_in_time_against_semidiscrete_closed_form():
    """P8: FIE and DR fine propagators are first order against the exact
    semi-discrete mode-(1,1) solution a_sd(t) = e^{-L t}[1 + amp (e^{(L-1)t} - 1)/(L-1)];
    DR's error is smaller (second-order splitting error)."""
    n = 32
    lam = modal.lambdas((1, 1), n, 1.0, 2)
    Lam = -(lam[0] + lam[1])
    amp = 2 * mp.pi ** 2
    a_sd = lambda t: mp.exp(-Lam * t) * (1 + amp * (mp.exp((Lam - 1) * t) - 1) / (Lam - 1))
    errs = {FIE: [], DR: []}
    for s in (16, 32, 64, 128):  # delta t = 1/128 .. 1/1024
        for sch in (FIE, DR):
            p = Problem(dim=2, n=n, c=1.0, source=1, N=8, s=s, G=sch, F=sch)
            o = oracle.Oracle(p)
            u0 = synth.initial_state(p)
            fine = o.fine_solution(u0)
            e = max(abs(fine[k][n // 2, n // 2] / u0[n // 2, n // 2] - float(a_sd(mp.mpf(k) / 8)))
                    for k in range(1, 9))
            errs[sch].append(e)
    for sch in (FIE, DR):
        ratios = [a / b for a, b in zip(errs[sch], errs[sch][1:])]
        assert all(1.7 <= r <= 3.2 for r in ratios), (sch, errs[sch])
    assert all(d < f for d, f in zip(errs[DR], errs[FIE]))
    # delta t = 1/128: FIE error 3.2506e-2 (an exact consequence of the closed form)
    assert errs[FIE][0] == pytest.approx(3.2506e-2, rel=1e-4)


def test_dd_fine_propagator_is_first_order():
    """P8 (DD): the unsplit A has phi as an eigenvector, so the DD fine solution converges at
    first order to the same semi-discrete a_sd * phi."""
    n = 32
    lam = modal.lambdas((1, 1), n, 1.0, 2)
    Lam = -(lam[0] + lam[1])
    amp = 2 * mp.pi ** 2
    a_sd = lambda t: mp.exp(-Lam * t) * (1 + amp * (mp.exp((Lam - 1) * t) - 1) / (Lam - 1))
    errs = []
    for s in (4, 8, 16, 32):
        p = Problem(dim=2, n=n, c=1.0, source=1, N=4, s=s, split=1, dd_strips=4, dd_overlap=4)
        o = oracle.Oracle(p)
        u0 = synth.initial_state(p)
        fine = o.fine_solution(u0)
        exact = np.array([float(a_sd(mp.mpf(k) / 4)) for k in range(5)])
        errs.append(max(np.max(np.abs(fine[k] - exact[k] * u0)) for k in range(1, 5)))
    ratios = [a / b for a, b in zip(errs, errs[1:])]
    assert all(1.6 <= r <= 2.4 for r in ratios), errs


def test_determinism():
    """P12: bitwise identical reruns, also with the per-slice F / G
    evaluations of an iteration spread over threads (independent slices)."""
    p = Problem(dim=2, n=12, N=5, s=3, G=FIE, F=DR, coef=1, init="random")
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    a, _ = o.parareal(u0, 3, fixed=True)
    b, _ = o.parareal(u0, 3, fixed=True)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    try:
        oracle.set_threads(4)
        c, _ = o.parareal(u0, 3, fixed=True)
    finally:
        oracle.set_threads(1)
    assert all(np.array_equal(x, y) for x, y in zip(a, c))


def test_c1_paper_pairing_fie_dr_contracts_per_mode():
    """NEXT-1: on c1's 16 excited modes the paper's pairing Parareal/FIE-DR
    has convergence factor K < 1 (Theorem), and the error of each mode's
    parareal iterate against its fine solution contracts at least like K^k.
    Scalar recurrences in mpmath; the GPU field is checked against their superposition in
    test_gpu_parity.py."""
    p = synth.CONFIGS["c1p"]
    dT = mp.mpf(p.T) / p.N
    for j, l, _a in synth.mode_table(p.seed):
        lam = modal.lambdas((j, l), p.n, p.c, 2)
        K = float(modal.conv_factor([dT * x for x in lam], p.s, "FIE", "DR"))
        assert K < 1.0, (j, l, K)
        sp = modal.ScalarParareal(lam, p.T, p.N, p.s, FIE, DR)
        fine = sp.fine_solution(1)
        trs = sp.run(1, 4)
        e0 = max(abs(x - y) for x, y in zip(trs[0][1:], fine[1:]))
        for k in range(1, 5):
            ek = max(abs(x - y) for x, y in zip(trs[k][1:], fine[1:]))
            assert float(ek) <= K ** k * float(e0) * (1 + 1e-9) + 1e-30, (j, l, k, float(ek), K)


# --------------------------- NEXT-3: full diffusion tensor (section 5.2)
# d11 = d22 = 1 / (2 + cos(3 pi x) cos(2 pi y)), d12 = 1/4; DD splitting only (mixed
# derivatives).  DESIGN.md R21 (9-point cross stencil, d12 at the cell corners)
# and R22 (DD weight of a mixed flux piece = rho_j at its corner's x).

def _lu_exact_full_tensor(x, y, c):
    """L u = div(D grad u) - c u for u = sin(2 pi x) sin(2 pi y) and the section-5.2 tensor,
    differentiated by hand: (d u_x)_x + (d u_y)_y + 2 d12 u_xy - c u with d = 1/g,
    g = 2 + cos(3 pi x) cos(2 pi y) (constant d12)."""
    pi = np.pi
    u = np.sin(2 * pi * x) * np.sin(2 * pi * y)
    ux = 2 * pi * np.cos(2 * pi * x) * np.sin(2 * pi * y)
    uy = 2 * pi * np.sin(2 * pi * x) * np.cos(2 * pi * y)
    uxx = -4 * pi ** 2 * u
    uyy = -4 * pi ** 2 * u
    uxy = 4 * pi ** 2 * np.cos(2 * pi * x) * np.cos(2 * pi * y)
    g = 2 + np.cos(3 * pi * x) * np.cos(2 * pi * y)
    gx = -3 * pi * np.sin(3 * pi * x) * np.cos(2 * pi * y)
    gy = -2 * pi * np.cos(3 * pi * x) * np.sin(2 * pi * y)
    d, dx, dy = 1 / g, -gx / g ** 2, -gy / g ** 2
    return u, dx * ux + d * uxx + dy * uy + d * uyy + 2 * 0.25 * uxy - c * u


def test_full_tensor_operator_is_second_order():
    """the discrete full-tensor operator on the interpolant of sin(2 pi x)
    sin(2 pi y) matches L u pointwise to O(h^2), slope ~ 2 over h = 1/32, 1/64, 1/128."""
    errs, hs = [], []
    for n in (31, 63, 127):
        p = Problem(dim=2, n=n, c=1.0, coef=2, split=1, dd_strips=2, dd_overlap=2)
        o = oracle.Oracle(p)
        h = 1.0 / (n + 1)
        xs = h * np.arange(1, n + 1)
        X, Y = np.meshgrid(xs, xs)
        u, lu = _lu_exact_full_tensor(X, Y, 1.0)
        errs.append(np.max(np.abs(o.apply(-1, u) - lu)))
        hs.append(h)
    slope = np.polyfit(np.log(hs), np.log(errs), 1)[0]
    assert 1.8 <= slope <= 2.2, (errs, slope)


def test_full_tensor_mixed_stencil_is_the_cross_difference():
    """For rho = 1 away from the boundary the row is the conservative 5-point part plus
    d12 (u_{++} - u_{+-} - u_{-+} + u_{--}) / (2 h^2): corners +-d12/(2h^2), and the mixed
    contributions cancel on the centre and the four edge neighbours (row sum = -c for a
    constant field's interior row)."""
    n = 15
    p = Problem(dim=2, n=n, c=0.7, coef=2, split=1, dd_strips=2, dd_overlap=2)
    o = oracle.Oracle(p)
    h = 1.0 / (n + 1)
    i, l = 7, 9
    r = o.row(-1, i, l)
    g = 0.25 / (2 * h * h)
    assert r[10] == pytest.approx(g, rel=1e-14) and r[7] == pytest.approx(g, rel=1e-14)
    assert r[8] == pytest.approx(-g, rel=1e-14) and r[9] == pytest.approx(-g, rel=1e-14)
    d = lambda x, y: 1.0 / (2 + np.cos(3 * np.pi * x) * np.cos(2 * np.pi * y))
    x, y = i * h, l * h
    assert r[1] == pytest.approx(d(x - h / 2, y) / h ** 2, rel=1e-13)
    assert r[2] == pytest.approx(d(x + h / 2, y) / h ** 2, rel=1e-13)
    assert r[3] == pytest.approx(d(x, y - h / 2) / h ** 2, rel=1e-13)
    assert r[4] == pytest.approx(d(x, y + h / 2) / h ** 2, rel=1e-13)
    assert sum(r) == pytest.approx(-0.7, abs=1e-9 / h ** 2)


FULL_DD = [
    Problem(dim=2, n=32, c=1.0, coef=2, split=1, dd_strips=4, dd_overlap=4, dd_ramp=0),
    Problem(dim=2, n=32, c=1.0, coef=2, split=1, dd_strips=4, dd_overlap=4, dd_ramp=1),
    Problem(dim=2, n=24, c=2.0, coef=2, split=1, dd_strips=8, dd_overlap=2, dd_ramp=0),
]


@pytest.mark.parametrize("p", FULL_DD, ids=lambda p: f"n{p.n}_S{p.dd_strips}_b{p.dd_overlap}_r{p.dd_ramp}")
def test_full_tensor_dd_split(p):
    """The unsplit operator is symmetric and negative definite; sum_j A_j = A to
    1e-13; each (I - tau A_j) is block diagonal with identity rows outside the
    support of rho_j -- the corner weights of R22 vanish at the
    block edges -- and the oracle's band elimination equals LAPACK's dense solve."""
    o = oracle.Oracle(p)
    A = o.dense(-1)
    assert np.max(np.abs(A - A.T)) <= 1e-13 * np.max(np.abs(A))
    assert np.max(np.linalg.eigvalsh(0.5 * (A + A.T))) < 0.0
    terms = [o.dense(j) for j in range(2)]
    assert np.max(np.abs(terms[0] + terms[1] - A)) <= 1e-13 * np.max(np.abs(A))
    n = p.n
    col = np.tile(np.arange(1, n + 1), n)  # x index (1-based) of every unknown, x-fastest
    rng = np.random.default_rng(5)
    for j in range(2):
        sup = np.array([o.rho(j, float(i)) > 0.0 for i in range(1, n + 1)])
        insup = sup[col - 1]
        # block id per column: connected runs of the support
        bid = np.cumsum(np.concatenate([[1], (sup[1:] & ~sup[:-1]).astype(int)])) * sup
        B = np.eye(A.shape[0]) - 0.05 * terms[j]
        # identity rows outside the support
        assert np.array_equal(B[~insup], np.eye(A.shape[0])[~insup])
        # no coupling between different blocks or from a block to outside nodes
        bcol = bid[col - 1]
        for q in np.flatnonzero(insup):
            nz = np.flatnonzero(B[q])
            assert np.all(bcol[nz] == bcol[q]), (j, q)
        r = rng.standard_normal(A.shape[0])
        v = o.solve(j, 0.05, r).reshape(-1)
        assert np.max(np.abs(v - np.linalg.solve(B, r))) <= 1e-12 * np.max(np.abs(r))


# ------------------------------------------- extended-precision bound of one step
XPREC_CASES = [
    Problem(dim=2, n=17, c=1.0, coef=0, source=1),
    Problem(dim=2, n=33, c=1.0, coef=1),
    Problem(dim=3, n=9, c=1.0, source=1),
    Problem(dim=2, n=32, c=1.0, split=1, dd_strips=4, dd_overlap=4, dd_ramp=0, source=1),
    Problem(dim=2, n=32, c=1.0, split=1, dd_strips=4, dd_overlap=4, dd_ramp=1),
    Problem(dim=2, n=24, c=1.0, coef=1, split=1, dd_strips=8, dd_overlap=2),
]


@pytest.mark.parametrize("p", XPREC_CASES, ids=lambda p: p.label() + f"_k{p.coef}_r{p.dd_ramp}")
def test_steps_within_rounding_of_extended_precision(p):
    """Noisy inputs (white noise, the worst case for DR's explicit term): the oracle's FIE / DR
    steps sit within 8 eps64 (|U_n| + |tau A U_n| + |tau F| + |U_{n+1}|) of the step evaluated in
    80-bit extended precision from the paper's formulas (tests/xprec.py; PAPER.md:151-157,
    165-171).  A relative coefficient error of 1e-9 anywhere in the operators would exceed it."""
    from tests.xprec import XStep, err_in_eps
    xs = XStep(p)
    o = oracle.Oracle(p)
    u = np.random.default_rng(3 + p.n).standard_normal((p.n,) * p.dim)
    for sch in ((FIE, DR) if p.dim == 2 else (FIE,)):
        for tau, t in ((1e-4, 0.3), (0.37, 0.74)):
            ref, scale = xs.step(sch, tau, t, u)
            assert err_in_eps(o.step(sch, tau, t, u), ref, scale) <= 8.0, (sch, tau)
