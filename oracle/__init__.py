"""TEST INFRASTRUCTURE ONLY -- plain serial fp64 CPU oracle (ctypes wrapper of oracle.c).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  It shares no code with the CUDA product
path (``paper_2502_08370_b200``); the only common module is ``synth`` (seeded input
generators and config shapes, which contain none of the method's arithmetic).

Function-by-function citations are in ``oracle.c``.  Every function is pinned by a
``-m "not gpu"`` test in ``tests/test_oracle_*.py`` (closed forms, modal recurrences,
dense library solves, invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "oracle.c")]
_HDR = [os.path.join(_HERE, "oracle_problem.h")]


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, no FMA contraction, no fast-math)."""
    newest = max(os.path.getmtime(f) for f in _SRC + _HDR)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-shared", "-fPIC",
               "-pthread", "-o", _SO + ".tmp"] + _SRC + ["-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class OrcProblem(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("n", ctypes.c_int), ("c", ctypes.c_double),
                ("coef", ctypes.c_int), ("split", ctypes.c_int), ("dd_strips", ctypes.c_int),
                ("dd_overlap", ctypes.c_int), ("dd_ramp", ctypes.c_int), ("source", ctypes.c_int),
                ("T", ctypes.c_double), ("N", ctypes.c_int), ("s", ctypes.c_int),
                ("G", ctypes.c_int), ("F", ctypes.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER(OrcProblem)
        D = ctypes.POINTER(ctypes.c_double)
        I, Dd = ctypes.c_int, ctypes.c_double
        sig = {
            "orc_rho": ([P, I, Dd], Dd),
            "orc_row": ([P, I, I, I, I, D], None),
            "orc_apply": ([P, I, D, D], None),
            "orc_dense": ([P, I, D], None),
            "orc_source": ([P, Dd, D], None),
            "orc_solve": ([P, I, Dd, D, D], None),
            "orc_step": ([P, I, Dd, Dd, D, D], None),
            "orc_coarse": ([P, I, D, D], None),
            "orc_fine": ([P, I, D, D], None),
            "orc_coarse_sweep": ([P, D, D], None),
            "orc_parareal_iteration": ([P, D, D], None),
            "orc_fine_solution": ([P, D, D], None),
            "orc_nterms": ([P], I),
            "orc_set_threads": ([I], None),
        }
        for name, (args, res) in sig.items():
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = res
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def set_threads(k: int) -> None:
    """Threads for the per-slice F / G evaluations of a parareal iteration (results unchanged)."""
    lib().orc_set_threads(int(k))


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


class Oracle:
    """Oracle bound to one problem (a ``synth.Problem``)."""

    def __init__(self, prob):
        self.prob = prob
        self._p = OrcProblem(dim=prob.dim, n=prob.n, c=prob.c, coef=prob.coef, split=prob.split,
                             dd_strips=prob.dd_strips, dd_overlap=prob.dd_overlap,
                             dd_ramp=prob.dd_ramp, source=prob.source, T=prob.T, N=prob.N,
                             s=prob.s, G=prob.G, F=prob.F)
        self.L = lib()
        self.npts = prob.n ** prob.dim
        self.shape = (prob.n,) * prob.dim

    @property
    def p(self):
        return ctypes.byref(self._p)

    def _vec(self, u=None):
        if u is None:
            return np.zeros(self.shape, dtype=np.float64)
        return np.ascontiguousarray(u, dtype=np.float64).reshape(self.shape)

    def nterms(self) -> int:
        return self.L.orc_nterms(self.p)

    def rho(self, j: int, xpos: float) -> float:
        return self.L.orc_rho(self.p, j, xpos)

    def row(self, term, i, l, m=1):
        out = np.zeros(11)
        self.L.orc_row(self.p, term, i, l, m, _dp(out))
        return out

    def apply(self, term, u):
        u = self._vec(u)
        out = self._vec()
        self.L.orc_apply(self.p, term, _dp(u), _dp(out))
        return out

    def dense(self, term):
        N = self.npts
        M = np.zeros((N, N))
        self.L.orc_dense(self.p, term, _dp(M))
        return M

    def source(self, t):
        out = self._vec()
        self.L.orc_source(self.p, t, _dp(out))
        return out

    def solve(self, term, tau, r):
        r = self._vec(r)
        out = self._vec()
        self.L.orc_solve(self.p, term, tau, _dp(r), _dp(out))
        return out

    def step(self, scheme, tau, t_next, u):
        u = self._vec(u)
        out = self._vec()
        self.L.orc_step(self.p, scheme, tau, t_next, _dp(u), _dp(out))
        return out

    def coarse(self, slice_, v):
        v = self._vec(v)
        out = self._vec()
        self.L.orc_coarse(self.p, slice_, _dp(v), _dp(out))
        return out

    def fine(self, slice_, v):
        v = self._vec(v)
        out = self._vec()
        self.L.orc_fine(self.p, slice_, _dp(v), _dp(out))
        return out

    def _traj(self):
        return np.zeros((self.prob.N + 1,) + self.shape)

    def coarse_sweep(self, u0):
        u0 = self._vec(u0)
        tr = self._traj()
        self.L.orc_coarse_sweep(self.p, _dp(u0), _dp(tr))
        return tr

    def iteration(self, traj_k):
        traj_k = np.ascontiguousarray(traj_k, dtype=np.float64)
        out = self._traj()
        self.L.orc_parareal_iteration(self.p, _dp(traj_k), _dp(out))
        return out

    def fine_solution(self, u0):
        u0 = self._vec(u0)
        tr = self._traj()
        self.L.orc_fine_solution(self.p, _dp(u0), _dp(tr))
        return tr

    def parareal(self, u0, kmax, tol=0.0, fixed=False):
        """Literal parareal: returns (list of trajectories U^0..U^k, list of normalised updates).

        Stop rule (reading R7): upd_k = max|U^{k+1} - U^k| / ||U_0||_inf <= tol,
        or k = min(kmax, N_c) (finite termination).  ``fixed`` ignores tol."""
        trajs = [self.coarse_sweep(u0)]
        upds = []
        scale = float(np.max(np.abs(u0))) or 1.0
        kmax = min(kmax, self.prob.N)
        for _ in range(kmax):
            nxt = self.iteration(trajs[-1])
            upd = float(np.max(np.abs(nxt - trajs[-1]))) / scale
            trajs.append(nxt)
            upds.append(upd)
            if not np.all(np.isfinite(nxt)):
                break
            if not fixed and upd <= tol:
                break
        return trajs, upds
