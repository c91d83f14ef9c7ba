"""Seeded synthetic inputs and config shapes (shared by tests, bench, oracle and CUDA path).

This module holds NONE of the method's arithmetic: it only describes problem shapes
(BASELINE.json configs c0-c4) and draws / samples initial data U(0) = P u_0.
The source term F(t), the operators and the propagators are implemented separately by
``oracle/`` and by the CUDA library.

Random-mode initial data (BASELINE c1/c3; reading R9): 16 distinct (j, l) pairs
drawn from {1..8}^2 by a partial Fisher-Yates shuffle driven by SplitMix64(seed), amplitudes
a_jl = Z_jl / (j^2 + l^2) with Z ~ N(0,1) from Box-Muller on the same stream, and
u0(x_i, y_m) = sum a_jl sin(j pi x_i) sin(l pi y_m) sampled at the interior nodes.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

FIE, DR, IE = 0, 1, 2  # IE: unsplit implicit Euler (Parareal/IE-IE baseline, NEXT-4)
SCHEME = {"FIE": FIE, "DR": DR, "IE": IE}


@dataclasses.dataclass
class Problem:
    dim: int = 2
    n: int = 32
    c: float = 1.0
    coef: int = 0          # 0 kappa = 1, 1 kappa = 1 + 0.5 sin(2 pi x) sin(2 pi y),
                           # 2 full tensor of section 5.2 (DD only; oracle only, NEXT-3)
    split: int = 0         # 0 dimensional, 1 domain decomposition
    dd_strips: int = 8
    dd_overlap: int = 8
    dd_ramp: int = 0       # 0 linear, 1 cosine
    source: int = 0        # 0 none, 1 manufactured (u = e^{-t} prod sin(pi x_d)),
                           # 2 the section-5.1 solution u = sin(2 pi t) sin(2 pi x) sin(2 pi y) (2-D, D = I)
    T: float = 1.0
    N: int = 8
    s: int = 16
    G: int = FIE
    F: int = FIE
    init: str = "phi"      # "phi" | "modes" | "random" | "zero"
    seed: int = 0
    kmax: int = 0          # 0 -> N (finite termination)
    tol: float = 1e-10
    fixed_k: bool = False

    @property
    def npts(self) -> int:
        return self.n ** self.dim

    def replace(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)

    def label(self) -> str:
        names = {FIE: "FIE", DR: "DR", IE: "IE"}
        sp = "dd" if self.split else "dim"
        return f"{self.dim}d_n{self.n}_{sp}_{names[self.G]}-{names[self.F]}_N{self.N}_s{self.s}"


# BASELINE.json configs (0-indexed).  Readings are listed in DESIGN.md §3.
CONFIGS = {
    # c0: 2-D 32^2, manufactured e^{-t} sin sin, N = 8, s = 16, FIE-FIE, K = 8 fixed
    "c0": Problem(dim=2, n=32, c=1.0, source=1, N=8, s=16, G=FIE, F=FIE, init="phi",
                  kmax=8, fixed_k=True),
    # c1: 2-D 256^2, DR-DR, f = 0, 16 random modes, N = 32, s = 64, stop update < 1e-10
    "c1": Problem(dim=2, n=256, c=1.0, source=0, N=32, s=64, G=DR, F=DR, init="modes"),
    # c2: 3-D 128^3, FIE-FIE (x, y, z), manufactured, N = 64, s = 32
    "c2": Problem(dim=3, n=128, c=1.0, source=1, N=64, s=32, G=FIE, F=FIE, init="phi"),
    # c3: 2-D 4096^2, variable kappa, G = FIE (paper's L-stable coarse), F = DR, N = 64, s = 256
    "c3": Problem(dim=2, n=4096, c=1.0, coef=1, source=0, N=64, s=256, G=FIE, F=DR,
                  init="modes"),
    # c1p: c1 with the paper's own pairing Parareal/FIE-DR
    # (G = FIE, L-stable; F = DR)
    "c1p": Problem(dim=2, n=256, c=1.0, source=0, N=32, s=64, G=FIE, F=DR, init="modes"),
    # c4: 2-D 1024^2 DD, 8 strips, 8-cell overlap, linear ramp, manufactured, N = 32, s = 64
    "c4": Problem(dim=2, n=1024, c=1.0, split=1, dd_strips=8, dd_overlap=8, dd_ramp=0,
                  source=1, N=32, s=64, G=FIE, F=FIE, init="phi"),
    # c5: c4's DD recipe with the full diffusion tensor of PAPER.md:523-528
    # (d11 = d22 = 1/(2 + cos 3pi x cos 2pi y), d12 = 1/4), the paper's Parareal/FIE-FIE
    "c5": Problem(dim=2, n=1024, c=1.0, coef=2, split=1, dd_strips=8, dd_overlap=8, dd_ramp=0,
                  source=1, N=32, s=64, G=FIE, F=FIE, init="phi"),
    # c6: the Parareal/IE-IE baseline on the paper's section-5.1 problem
    # (PAPER.md:444-453): u = sin(2 pi t) sin(2 pi x) sin(2 pi y), D = I, c = 0 (R29),
    # h = 1e-3 (n = 999), T = 1, Delta T = 0.05 (N = 20), delta t = 2.5e-3 (s = 20), u(0) = 0
    "c6": Problem(dim=2, n=999, c=0.0, source=2, N=20, s=20, G=IE, F=IE, init="zero"),
}


# ------------------------------------------------------------------ SplitMix64
class SplitMix64:
    MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        self.state = seed & self.MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & self.MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.MASK
        return z ^ (z >> 31)

    def uniform(self) -> float:
        """(0, 1] with 53 random bits."""
        return ((self.next() >> 11) + 1) * (1.0 / 9007199254740992.0)

    def below(self, m: int) -> int:
        return self.next() % m


def mode_table(seed: int = 0, count: int = 16, jmax: int = 8):
    """Draw `count` distinct (j, l) in {1..jmax}^2 and a_jl = Z/(j^2 + l^2)."""
    rng = SplitMix64(seed)
    idx = list(range(jmax * jmax))  # ordered pair index jmax*(j-1) + (l-1)
    for k in range(count):          # partial Fisher-Yates
        r = k + rng.below(len(idx) - k)
        idx[k], idx[r] = idx[r], idx[k]
    table = []
    for k in range(count):
        j, l = idx[k] // jmax + 1, idx[k] % jmax + 1
        u1, u2 = rng.uniform(), rng.uniform()
        z = math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)
        table.append((j, l, z / (j * j + l * l)))
    return table


def _sines(n: int, j: int) -> np.ndarray:
    h = 1.0 / (n + 1)
    return np.sin(j * math.pi * h * np.arange(1, n + 1, dtype=np.float64))


def initial_state(prob: Problem) -> np.ndarray:
    """U(0) = P u_0 sampled at the interior nodes, x-fastest layout (shape (n,)*dim)."""
    n = prob.n
    if prob.init == "phi":
        s1 = _sines(n, 1)
        if prob.dim == 2:
            return np.ascontiguousarray(np.outer(s1, s1))
        return np.ascontiguousarray(s1[:, None, None] * s1[None, :, None] * s1[None, None, :])
    if prob.init == "modes":
        assert prob.dim == 2
        u = np.zeros((n, n))
        for j, l, a in mode_table(prob.seed):
            # u[y][x]: y index l-mode, x index j-mode
            u += a * np.outer(_sines(n, l), _sines(n, j))
        return u
    if prob.init == "zero":  # u(0) = sin(0) sin sin = 0 of the section-5.1 solution
        return np.zeros((n,) * prob.dim)
    if prob.init == "random":
        rng = np.random.default_rng(prob.seed)
        return rng.standard_normal((n,) * prob.dim)
    raise ValueError(prob.init)


# ------------------------------------------------------- digests of large trajectories
# (used to compare runs whose full states are too large to store: a fixed seeded set of
# sample points and +-1 random projections; pure index / sign generation, no method arithmetic)
def sample_indices(npts: int, count: int = 128, seed: int = 2502) -> np.ndarray:
    """`count` distinct flat indices into a state of npts points (first and last included)."""
    rng = SplitMix64(seed)
    picked = {0, npts - 1}
    while len(picked) < min(count, npts):
        picked.add(rng.below(npts))
    return np.array(sorted(picked), dtype=np.int64)


def projection_signs(npts: int, count: int = 4, seed: int = 8370) -> np.ndarray:
    """count x npts matrix of +-1.0 (SplitMix64 bits)."""
    rng = SplitMix64(seed)
    out = np.empty((count, npts))
    for r in range(count):
        words = np.array([rng.next() for _ in range((npts + 63) // 64)], dtype=np.uint64)
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:npts]
        out[r] = 1.0 - 2.0 * bits
    return out


def digest(states: np.ndarray, idx: np.ndarray, signs: np.ndarray) -> dict:
    """Per state of `states` (S x npts): sampled values, projections, inf norm."""
    flat = np.asarray(states, dtype=np.float64).reshape(states.shape[0], -1)
    return {"samples": flat[:, idx], "proj": flat @ signs.T, "inf": np.max(np.abs(flat), axis=1)}
