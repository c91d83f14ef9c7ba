"""GPU parity of the unsplit implicit Euler propagator (PRS_IE; the Parareal/IE-IE baseline of
PAPER.md:455) against the CPU oracle (-m gpu).

The GPU solves (I - tau A) U' = U + tau F exactly in the sine basis (ie.cuh: 2 dim dense DST-I
transforms on DMMA); the oracle by band elimination of the whole system (oracle.c ie_step).
Bar as tests/test_gpu_parity.py (R13): 1e-11 of the step's / iterate's max norm.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from synth import DR, FIE, IE, Problem
from tests import modal

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_08370_b200 as prs
    prs.lib()
    yield


def prs_mod():
    import paper_2502_08370_b200 as prs
    return prs


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def nerr(gpu, cpu, *scales):
    s = max([float(np.max(np.abs(x))) for x in scales] + [1e-300])
    return float(np.max(np.abs(np.asarray(gpu) - np.asarray(cpu)))) / s


# sizes spanning one tile (64), several tiles with a ragged tail, and the degenerate n = 1
IE_STEP_CASES = [Problem(dim=2, n=n, c=c, source=src, N=4, s=3, G=IE, F=IE)
                 for n, c, src in ((1, 1.0, 1), (7, 0.0, 1), (64, 1.0, 0), (100, 1.0, 1), (130, 2.0, 1))]
IE_STEP_CASES += [Problem(dim=3, n=n, c=1.0, source=1, N=4, s=3, G=IE, F=IE) for n in (1, 5, 16)]


@pytest.mark.parametrize("p", IE_STEP_CASES, ids=lambda p: f"{p.dim}d_n{p.n}_c{p.c}_f{p.source}")
def test_ie_single_step_parity(p):
    prs = prs_mod()
    o = oracle.Oracle(p)
    ctx = prs.Context(p)
    rng = np.random.default_rng(p.n)
    for tau, t1 in ((1e-3, 0.25), (0.05, 0.5), (1.0, 1.0)):
        u = rng.standard_normal((p.n,) * p.dim)
        want = o.step(IE, tau, t1, u)
        out = torch.empty((p.n,) * p.dim, dtype=torch.float64, device="cuda")
        ctx.step(IE, tau, t1, dev(u), out)
        assert nerr(host(out), want, u, want) <= TOL, tau
    ctx.close()


IE_PARAREAL_CASES = [
    Problem(dim=2, n=48, c=1.0, source=1, N=5, s=4, G=IE, F=IE, init="phi"),
    Problem(dim=2, n=70, c=0.0, source=0, N=6, s=3, G=IE, F=IE, init="modes", seed=3),
    Problem(dim=2, n=40, c=1.0, source=1, N=4, s=5, G=FIE, F=IE, init="phi"),   # split G, exact F
    Problem(dim=2, n=40, c=1.0, source=0, N=4, s=5, G=IE, F=DR, init="modes", seed=5),
    Problem(dim=3, n=12, c=1.0, source=1, N=3, s=2, G=IE, F=IE, init="phi"),
    # DD split for F (FIE over 4 strips), exact G
    Problem(dim=2, n=32, c=1.0, split=1, dd_strips=4, dd_overlap=2, source=1, N=4, s=3, G=IE, F=FIE),
]


@pytest.mark.parametrize("p", IE_PARAREAL_CASES, ids=lambda p: p.label())
def test_ie_parareal_iterates_match_oracle_every_iteration(p):
    """every iterate k = 0..N (INIT / DELTA / CORRECT epilogues of the IE kernel), the update
    norms, and finite termination at k = N"""
    from tests.test_gpu_parity import _parareal_vs_oracle
    _parareal_vs_oracle(p)


def test_c6_shape_batched_fine_step_closed_form():
    """c6 (n = 999, the paper's h = 1e-3) on the benchmarked launch shape -- one fine step over
    all N = 20 slice states in one batch -- on random sine-mode data with F = 0, against the
    per-mode closed form 1 / (1 + delta t (c + mu_j + mu_l)) (the oracle's O(n^4) solve is out of
    reach at this size)"""
    prs = prs_mod()
    p = synth.CONFIGS["c6"].replace(source=0)
    n, B = p.n, p.N
    dt = p.T / (p.N * p.s)
    rng = np.random.default_rng(6)
    modes = [(int(j), int(l)) for j, l in rng.integers(1, n + 1, size=(12, 2))] + [(1, 1), (n, n), (1, n)]
    h = 1.0 / (n + 1)
    x = np.arange(1, n + 1) * h

    def mu(j):
        return 4.0 / h ** 2 * np.sin(j * np.pi * h / 2) ** 2
    ins, wants = [], []
    for b in range(B):
        amps = rng.standard_normal(len(modes))
        u = np.zeros((n, n))
        w = np.zeros((n, n))
        for (j, l), a in zip(modes, amps):
            shape = np.outer(np.sin(l * np.pi * x), np.sin(j * np.pi * x))
            u += a * shape
            w += a / (1.0 + dt * (p.c + mu(j) + mu(l))) * shape
        ins.append(u)
        wants.append(w)
    ctx = prs.Context(p)
    inp = dev(np.stack(ins))
    out = torch.empty_like(inp)
    ctx.step_batch(1, 0, 0, inp, out, B)
    got = host(out)
    for b in range(B):
        assert nerr(got[b], wants[b], ins[b]) <= TOL, b
    ctx.close()


def test_ie_rejects_variable_coefficients_loudly():
    prs = prs_mod()
    with pytest.raises(prs.PrsError) as ei:
        prs.Context(Problem(dim=2, n=16, coef=1, N=2, s=2, G=IE, F=IE))
    assert ei.value.code == prs.PRS_EUNSUPPORTED


def test_ie_step_needs_ie_context():
    prs = prs_mod()
    p = Problem(dim=2, n=16, N=2, s=2, G=FIE, F=FIE)
    ctx = prs.Context(p)
    x = dev(np.zeros((16, 16)))
    with pytest.raises(prs.PrsError) as ei:
        ctx.step(IE, 0.1, 0.1, x, torch.empty_like(x))
    assert ei.value.code == prs.PRS_EINVAL
    ctx.close()


# ------------------------------ the section-5.1 problem: source_kind 2 on every kernel path
S51_PARAREAL_CASES = [
    Problem(dim=2, n=40, c=0.0, source=2, N=5, s=4, G=IE, F=IE, init="zero"),
    Problem(dim=2, n=64, c=0.0, source=2, N=4, s=4, G=FIE, F=DR, init="zero"),    # per-step kernels
    Problem(dim=2, n=48, c=1.0, source=2, N=4, s=3, G=DR, F=DR, init="random"),
    Problem(dim=2, n=32, c=0.0, split=1, dd_strips=4, dd_overlap=2, source=2, N=4, s=3, G=FIE, F=FIE,
            init="zero"),
    Problem(dim=2, n=32, c=0.0, split=1, dd_strips=2, dd_overlap=4, source=2, N=4, s=3, G=IE, F=DR,
            init="zero"),
]


@pytest.mark.parametrize("p", S51_PARAREAL_CASES, ids=lambda p: p.label())
def test_section51_parareal_iterates_match_oracle(p):
    from tests.test_gpu_parity import _parareal_vs_oracle
    _parareal_vs_oracle(p)


@pytest.mark.parametrize("n", [100, 1024, 2048, 4096])
def test_section51_single_steps_long_lines(n):
    """FIE and DR steps with the section-5.1 source through the long-line kernels (xpass3 / xpass7
    + lpass) at the benchmarked line lengths, against the oracle"""
    prs = prs_mod()
    p = Problem(dim=2, n=n, c=0.0, source=2, N=4, s=3, G=FIE, F=DR)
    o = oracle.Oracle(p)
    ctx = prs.Context(p)
    # smooth data (the literal vs algebraic DR forms differ by eps tau ||A U||, R13)
    x = np.arange(1, n + 1) / (n + 1)
    u = 0.1 * np.outer(np.sin(3 * np.pi * x), np.sin(2 * np.pi * x))
    for scheme, tau, t1 in ((FIE, 1e-3, 0.3), (DR, 1e-4, 0.77)):
        want = o.step(scheme, tau, t1, u)
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
        ctx.step(scheme, tau, t1, dev(u), out)
        assert nerr(host(out), want, u, want) <= TOL, scheme
    ctx.close()


def test_section51_source_rejected_outside_2d_constant_d():
    prs = prs_mod()
    for p in (Problem(dim=3, n=8, source=2, N=2, s=2), Problem(dim=2, n=16, coef=1, source=2, N=2, s=2)):
        with pytest.raises(prs.PrsError) as ei:
            prs.Context(p)
        assert ei.value.code == prs.PRS_EINVAL
