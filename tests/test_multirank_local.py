"""The multi-rank driver on one GPU (-m gpu): P contexts of one process exchanging through the
in-process world (prs_create_local), one host thread per rank.

This runs the library's own multi-rank code -- slice partition, owner-G hand-off along the
rank chain, the stop-test all-reduce and its lagged form (NEXT-2),
converged-slice skipping, space-parallel G's band scatter / all-gather / gather
and the seeding of its band copies -- with only the transport swapped (include/prs.h; NCCL on
a multi-GPU box).  Owner-G results are bitwise independent of the rank count (SURVEY.md 8(e),
DESIGN.md R14); space-parallel G matches the oracle at every iteration.
"""
from __future__ import annotations

import threading

import numpy as np
import pytest

import oracle
import synth
from synth import DR, FIE, Problem

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


def run_ranks(p, P, body, u0=None):
    """Create P local-world contexts of problem p, run body(ctx, rank) on P threads; returns
    the per-rank results (re-raises the first failure)."""
    import paper_2502_08370_b200 as prs
    u0 = synth.initial_state(p) if u0 is None else u0
    world = prs.LocalWorld(P)
    out, errs = [None] * P, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            ctx = prs.Context(p, rank=r, world=world)
            try:
                out[r] = body(ctx, r, np.ascontiguousarray(u0))
            finally:
                ctx.close()
        except BaseException as e:  # surfaced below
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    world.close()
    if errs:
        raise errs[0][1]
    return out


def local_slices(ctx, p):
    """This rank's slice end states U_{n+1}, n over its slices (host)."""
    buf = np.empty((p.n,) * p.dim)
    res = {}
    for n in ctx.slices():
        ctx.get_slice(n + 1, buf)
        res[n + 1] = buf.copy()
    return res


def gather(results):
    full = {}
    for r in results:
        full.update(r["slices"])
    return full


def iterate_body(kmax, tol, explicit=False, cyclic=False):
    def body(ctx, r, u0):
        if cyclic:
            ctx.set_ownership(1)
        ctx.set_initial(u0)
        ctx.coarse_sweep()
        if explicit:  # prs_fine_sweep + prs_parareal_correct, unlagged
            hist = []
            for _ in range(kmax):
                ctx.fine_sweep()
                hist.append(ctx.parareal_correct())
                if hist[-1] <= tol:
                    break
            k = len(hist)
        else:
            k, hist = ctx.iterate(kmax, tol)
        return {"k": k, "hist": hist, "slices": local_slices(ctx, ctx.prob)}
    return body


OWNER_CASES = [
    # (problem, rank counts, tol)
    (Problem(dim=2, n=64, c=1.0, coef=1, N=8, s=4, G=FIE, F=DR, init="modes", seed=1), (2, 4), 0.0),
    (Problem(dim=2, n=64, c=1.0, N=6, s=5, G=DR, F=DR, init="modes", seed=2), (2, 3), 0.0),  # on-chip sweep2
    (Problem(dim=2, n=512, c=1.0, coef=1, N=8, s=3, G=FIE, F=DR, init="modes", seed=3), (2, 4), 1e-7),  # skipping
    (Problem(dim=3, n=20, c=1.0, source=1, N=6, s=3, G=FIE, F=FIE), (2,), 0.0),
    (Problem(dim=2, n=64, c=1.0, split=1, dd_strips=8, dd_overlap=4, source=1, N=6, s=3, G=FIE, F=DR), (2, 3), 0.0),
]


@pytest.mark.parametrize("p,Ps,tol", OWNER_CASES, ids=lambda x: x.label() if hasattr(x, "label") else str(x))
def test_owner_g_over_local_ranks_is_bitwise_the_single_rank_run(p, Ps, tol, monkeypatch):
    """Owner-G over P ranks -- contiguous slice blocks with the lagged and the unlagged stop
    test and the explicit fine_sweep / correct loop, and cyclic ownership (slice n on rank
    n mod P, NEXT-2) -- k, the update history and every slice end state equal the one-rank run bit
    for bit, and the one-rank run matches the oracle."""
    one = run_ranks(p, 1, iterate_body(p.N, tol))[0]
    for P in Ps:
        for mode in ("lagged", "unlagged", "explicit", "cyclic", "cyclic-explicit"):
            monkeypatch.setenv("PRS_LAG", "0" if mode == "unlagged" else "1")
            res = run_ranks(p, P, iterate_body(p.N, tol, explicit=mode.endswith("explicit"),
                                               cyclic=mode.startswith("cyclic")))
            assert all(r["k"] == one["k"] for r in res), (P, mode, [r["k"] for r in res])
            assert all(r["hist"] == one["hist"] for r in res), (P, mode)
            full = gather(res)
            assert sorted(full) == list(range(1, p.N + 1))
            for n, v in full.items():
                assert np.array_equal(v, one["slices"][n]), (P, mode, n)
    if tol == 0.0 and p.n <= 64:
        o = oracle.Oracle(p)
        u0 = synth.initial_state(p)
        trajs, upds = o.parareal(u0, p.N, fixed=True)
        scale = max(float(np.max(np.abs(t))) for t in trajs)
        for n in range(1, p.N + 1):
            assert float(np.max(np.abs(one["slices"][n] - trajs[-1][n]))) / scale <= TOL


def test_lagged_stop_discards_the_lookahead_sweep():
    """An early stop under the lagged test: the lookahead fine sweep of iteration k+1 has run
    but the trajectory is U^{k+1}; a following explicit iteration continues from it exactly as
    on one rank."""
    p = Problem(dim=2, n=64, c=1.0, coef=1, N=8, s=4, G=FIE, F=FIE, init="modes", seed=4)

    def body(ctx, r, u0):
        ctx.set_initial(u0)
        ctx.coarse_sweep()
        k, hist = ctx.iterate(p.N, 1e-6)  # (the oracle's updates: 4e-2 ... 9e-7 at k = 5)
        ctx.fine_sweep()
        extra = ctx.parareal_correct()
        return {"k": k, "hist": hist, "extra": extra, "slices": local_slices(ctx, p)}
    one = run_ranks(p, 1, body)[0]
    assert 1 < one["k"] < p.N
    res = run_ranks(p, 4, body)
    for r in res:
        assert r["k"] == one["k"] and r["hist"] == one["hist"] and r["extra"] == one["extra"]
    for n, v in gather(res).items():
        assert np.array_equal(v, one["slices"][n]), n


GPAR_CASES = [
    (Problem(dim=2, n=256, c=1.0, coef=1, N=4, s=3, G=FIE, F=DR, init="modes", seed=2), 2),
    (Problem(dim=2, n=256, c=1.0, coef=1, N=6, s=2, G=FIE, F=FIE, init="modes", seed=3), 4),
    (Problem(dim=2, n=128, c=1.0, source=1, N=4, s=4, G=FIE, F=FIE), 2),
]


@pytest.mark.parametrize("p,P", GPAR_CASES, ids=lambda x: x.label() if hasattr(x, "label") else f"P{x}")
def test_space_parallel_g_over_local_ranks_matches_oracle_and_reruns(p, P):
    """Space-parallel G over P ranks: each rank owns one row band of every coarse state; Delta
    bands scattered from the slice owners, band tuples all-gathered per G step, U / G-cache bands
    gathered back.  Every iterate and update against the oracle, twice on the
    same contexts (set_initial + coarse_sweep again): the band copies of the current iterate the
    chain's update norm reads are re-seeded after the trajectory changed."""
    o = oracle.Oracle(p)
    u0 = synth.initial_state(p)
    ctrajs, cupds = o.parareal(u0, p.N, fixed=True)

    def body(ctx, r, u0h):
        ctx.set_coarse_mode(1)
        runs = []
        for _ in range(2):
            ctx.set_initial(u0h)
            ctx.coarse_sweep()
            per_k, upds = [local_slices(ctx, p)], []
            for _k in range(p.N):
                ctx.fine_sweep()
                upds.append(ctx.parareal_correct())
                per_k.append(local_slices(ctx, p))
            runs.append((per_k, upds))
        return runs
    res = run_ranks(p, P, body)
    for run in range(2):
        for k in range(p.N + 1):
            full = {}
            for r in res:
                full.update(r[run][0][k])
            scale = max(float(np.max(np.abs(u0))), float(np.max(np.abs(ctrajs[k]))))
            for n, v in full.items():
                assert float(np.max(np.abs(v - ctrajs[k][n]))) / scale <= TOL, (run, k, n)
        for r in res:
            for k in range(p.N):
                assert abs(r[run][1][k] - cupds[k]) <= TOL * max(1.0, cupds[k]), (run, k)


def test_cyclic_ownership_balances_the_active_slices():
    """With converged-slice skipping contiguous blocks leave the first ranks idle
    while the last keeps N/P slices; cyclic ownership keeps ceil((N - k)/P) per rank.  Host-side
    check of the ownership rule the library implements (slice n on rank n mod P)."""
    N, P = 64, 8
    for k in (0, 9, 14, 40, 63):
        active = [sum(1 for n in range(r, N, P) if n >= k) for r in range(P)]
        assert max(active) - min(active) <= 1 and sum(active) == N - k
        blocks = [max(0, min(N, (r + 1) * N // P) - max(k, r * N // P)) for r in range(P)]
        if k <= N - N // P:
            assert max(blocks) == N // P  # the last block never shrinks before k > N - N/P
