"""Pins of the oracle's unsplit implicit Euler step (the Parareal/IE-IE baseline, SURVEY.md
8(f) NEXT-4; "the implicit Euler as both propagators"
ie_step: (I - tau A) U_{n+1} = U_n + tau F(t_n + tau)).

The oracle solves the whole n^dim system by band elimination (oracle.c ie_step); these tests
hold it to what the mathematics fixes independently of that code:
  * the discrete sine modes are eigenvectors of the constant-coefficient A (PAPER.md:237-250
    remark), so one IE step scales mode (j, l[, m]) by exactly 1 / (1 + tau (c + sum mu));
  * a dense partial-pivoting LU solve (numpy.linalg.solve) of I - tau A for the
    variable-coefficient and full-tensor operators, where no modal form exists;
  * scalar parareal recurrences (mpmath, tests/modal.py) for IE-IE and the mixed pairings,
    every iterate, and finite termination at k = N.
"""
from __future__ import annotations

import mpmath as mp
import numpy as np
import pytest

import oracle
import synth
from synth import DR, FIE, IE, Problem
from tests import modal


def nrm_err(a, b, scale):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / scale


def mode_shape(n, modes):
    """sin(j pi x) sin(l pi y) [sin(m pi z)] on the interior nodes, x fastest"""
    s = [np.array(modal.sines(n, j)) for j in modes]
    out = s[0]
    for v in s[1:]:
        out = np.multiply.outer(v, out)
    return out


@pytest.mark.parametrize("dim,n,modes,c", [(2, 9, (1, 1), 1.0), (2, 9, (3, 7), 0.0),
                                           (2, 16, (16, 2), 2.5), (3, 6, (1, 2, 5), 1.0)])
def test_ie_step_scales_sine_mode_by_closed_form(dim, n, modes, c):
    """one IE step on a sine mode, F = 0: U_1 = U_0 / (1 + tau (c + sum_d mu_{j_d}))"""
    p = Problem(dim=dim, n=n, c=c, source=0)
    o = oracle.Oracle(p)
    u = mode_shape(n, modes)
    for tau in (1e-3, 0.05, 1.0):
        lam = sum(modal.mu(j, n) for j in modes) + c
        want = u / float(1 + tau * lam)
        got = o.step(IE, tau, 0.3, u)
        assert nrm_err(got, want, 1.0) <= 1e-14, tau


@pytest.mark.parametrize("p", [
    Problem(dim=2, n=7, c=1.0, coef=1, source=1),
    Problem(dim=2, n=8, c=0.5, coef=2, split=1, dd_strips=2, dd_overlap=2, source=1),
    Problem(dim=3, n=4, c=1.0, source=1),
], ids=["kappa", "full_tensor", "3d"])
def test_ie_step_matches_dense_solve(p):
    """(I - tau A) U_1 = U_0 + tau F(t_1) solved densely with numpy (LAPACK partial pivoting)"""
    o = oracle.Oracle(p)
    rng = np.random.default_rng(11)
    u = rng.standard_normal(o.shape)
    A = o.dense(-1)
    I = np.eye(o.npts)
    for tau, t1 in ((1e-3, 0.1), (0.05, 0.7), (2.0, 1.0)):
        rhs = u.ravel() + tau * o.source(t1).ravel()
        want = np.linalg.solve(I - tau * A, rhs)
        got = o.step(IE, tau, t1, u).ravel()
        assert nrm_err(got, want, np.max(np.abs(want))) <= 1e-13, tau


def test_ie_equals_fie_when_one_term_carries_the_whole_operator():
    """SPEC.md:214 'matches fie_step exactly when M = 1 term': on n = 1 (one node, h = 1/2) the
    2-D operator is the scalar -(16 + c); FIE's two terms each carry -(8 + c/2) and give
    1 / ((1 + tau(8 + c/2))^2), IE gives 1 / (1 + tau (16 + c)) -- the product formula's
    splitting error tau^2 (8 + c/2)^2 is the only difference."""
    c, tau = 0.5, 0.1
    o = oracle.Oracle(Problem(dim=2, n=1, c=c, source=0))
    u = np.ones((1, 1))
    assert abs(o.step(IE, tau, 1.0, u)[0, 0] - 1.0 / (1.0 + tau * (16.0 + c))) <= 1e-16
    fie = 1.0 / (1.0 + tau * (8.0 + c / 2)) ** 2
    assert abs(o.step(FIE, tau, 1.0, u)[0, 0] - fie) <= 1e-16


@pytest.mark.parametrize("G,F", [(IE, IE), (FIE, IE), (IE, DR)])
def test_ie_parareal_modal_closed_form_all_iterations(G, F):
    """P1 for the IE pairings: every parareal iterate of the manufactured problem (mode (1,1)
    with source amplitude (2 pi^2 + c - 1) e^{-t}) equals the scalar recurrence in mpmath"""
    p = Problem(dim=2, n=12, c=1.0, source=1, N=5, s=4, G=G, F=F, init="phi")
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    trajs, _ = o.parareal(u0, p.N, fixed=True)
    M = 1 if (G == IE and F == IE) else 2
    lam = modal.lambdas((1, 1), p.n, p.c, 2)
    sp = modal.ScalarParareal(lam, p.T, p.N, p.s, G, F, src_amp=2 * mp.pi ** 2 + p.c - 1)
    want = sp.run(1, p.N)
    for k in range(p.N + 1):
        for n in range(p.N + 1):
            assert nrm_err(trajs[k][n], float(want[k][n]) * u0, 1.0) <= 1e-13, (k, n, M)


def test_ie_ie_finite_termination_variable_kappa():
    """P2: at k = N the IE-IE iterate equals the sequential fine IE solution"""
    p = Problem(dim=2, n=10, N=4, s=3, G=IE, F=IE, coef=1, init="random", source=1)
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    trajs, _ = o.parareal(u0, p.N, fixed=True)
    fine = o.fine_solution(u0)
    scale = max(np.max(np.abs(t)) for t in fine)
    for n in range(p.N + 1):
        assert nrm_err(trajs[p.N][n], fine[n], scale) <= 1e-14
    # and not earlier: the k = 1 iterate is still off at the last slice
    assert nrm_err(trajs[1][p.N], fine[p.N], scale) > 1e-8


# ------------------------------------------ the section-5.1 problem (source 2, R29)
def _u51(t, x, y):
    return mp.sin(2 * mp.pi * t) * mp.sin(2 * mp.pi * x) * mp.sin(2 * mp.pi * y)


def test_section51_source_is_ut_minus_laplacian_plus_cu():
    """F = u_t - (u_xx + u_yy) + c u for u = sin(2 pi t) sin(2 pi x) sin(2 pi y) (PAPER.md:444-449,
    D = I), the derivatives taken numerically by mpmath at sample nodes and times"""
    p = Problem(dim=2, n=9, c=0.7, source=2)
    o = oracle.Oracle(p)
    h = 1.0 / (p.n + 1)
    for t in (0.0, 0.13, 0.5, 0.91):
        F = o.source(t)
        for i, l in ((1, 1), (3, 7), (9, 4)):
            x, y = i * h, l * h
            want = (mp.diff(lambda s: _u51(s, x, y), t) - mp.diff(lambda s: _u51(t, s, y), x, 2)
                    - mp.diff(lambda s: _u51(t, x, s), y, 2) + p.c * _u51(t, x, y))
            assert abs(F[l - 1, i - 1] - float(want)) <= 1e-12 * 100, (t, i, l)


@pytest.mark.parametrize("G,F", [(IE, IE), (FIE, DR), (FIE, FIE)])
def test_section51_parareal_modal_closed_form(G, F):
    """P1 with the section-5.1 source: u0 = 0 and F on mode (2, 2) only, so every iterate is
    a^k_n sin(2 pi x) sin(2 pi y) with the scalar recurrence driven by
    b(t) = 2 pi cos(2 pi t) + (8 pi^2 + c) sin(2 pi t)"""
    c = 0.0
    p = Problem(dim=2, n=14, c=c, source=2, N=5, s=4, G=G, F=F, init="zero")
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    trajs, _ = o.parareal(u0, p.N, fixed=True)
    lam = modal.lambdas((2, 2), p.n, p.c, 2)
    sp = modal.ScalarParareal(lam, p.T, p.N, p.s, G, F,
                              bfun=lambda t: 2 * mp.pi * mp.cos(2 * mp.pi * t)
                              + (8 * mp.pi ** 2 + c) * mp.sin(2 * mp.pi * t))
    want = sp.run(0, p.N)
    shape = mode_shape(p.n, (2, 2))
    scale = max(np.max(np.abs(t)) for t in trajs)
    for k in range(p.N + 1):
        for n in range(p.N + 1):
            assert nrm_err(trajs[k][n], float(want[k][n]) * shape, scale) <= 1e-13, (k, n)
