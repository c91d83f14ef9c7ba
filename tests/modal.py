"""Closed forms used to pin the oracle (test side only; never imported by product code).

* Discrete sine eigenpairs (PAPER.md:237-250 remark -- the dimensional split operators
  with constant coefficients are simultaneously diagonalised by sin(j pi x_i)):
      A_d sin(j pi x_d) = -(mu_j + c/M) sin(j pi x_d),   mu_j = (4/h^2) sin^2(j pi h / 2).
* Stability functions R_FIE, R_DR and the convergence factor
  K, evaluated in mpmath at 40 digits.
* Scalar (per-mode) FIE / DR steps with a source amplitude b(t) on the mode:
      FIE: v = a + tau b(t_{n+1});  v <- v / (1 - z_j), j = 1..M       (eq. FIE_method)
      DR : v = (1 + sum z) a + tau b;  v <- (v - z_j a) / (1 - z_j)    (eq. DR_method)
      IE : v = (a + tau b) / (1 - sum z)                               (unsplit)
  and scalar parareal on them.
"""
from __future__ import annotations

import math

import mpmath as mp

mp.mp.dps = 40


def mu(j: int, n: int):
    h = mp.mpf(1) / (n + 1)
    return 4 / h ** 2 * mp.sin(j * mp.pi * h / 2) ** 2


def lambdas(modes, n: int, c: float, M: int):
    """per-direction eigenvalues of A_d for a tuple of mode numbers"""
    return [-(mu(j, n) + mp.mpf(c) / M) for j in modes]


def r_fie(zs):
    out = mp.mpf(1)
    for z in zs:
        out /= (1 - z)
    return out


def r_dr(zs):
    return 1 + r_fie(zs) * sum(zs)


def conv_factor(zs, s, G="FIE", F="FIE"):
    R = {"FIE": r_fie, "DR": r_dr}
    rg = R[G](zs)
    rf = R[F]([z / s for z in zs]) ** s
    return abs(rf - rg) / (1 - abs(rg))


def scalar_step(scheme, a, lam, tau, b):
    zs = [tau * l for l in lam]
    if scheme == 2:  # IE, unsplit: (1 - sum z) v = a + tau b
        return (a + tau * b) / (1 - sum(zs))
    if scheme == 0:  # FIE
        v = a + tau * b
        for z in zs:
            v = v / (1 - z)
        return v
    v = (1 + sum(zs)) * a + tau * b
    for z in zs:
        v = (v - z * a) / (1 - z)
    return v


class ScalarParareal:
    """Parareal on one eigen-mode: amplitude recurrences in mpmath."""

    def __init__(self, lam, T, N, s, G, F, src_amp=0.0, bfun=None):
        self.lam = lam
        self.T, self.N, self.s, self.G, self.F = mp.mpf(T), N, s, G, F
        self.src_amp = mp.mpf(src_amp)
        self.bfun = bfun  # source amplitude b(t) on the mode (default src_amp e^{-t})

    def b(self, t):
        if self.bfun is not None:
            return self.bfun(t)
        return self.src_amp * mp.exp(-t)

    def coarse(self, n, a):
        dT = self.T / self.N
        return scalar_step(self.G, a, self.lam, dT, self.b((n + 1) * dT))

    def fine(self, n, a):
        dt = self.T / (self.N * self.s)
        for j in range(self.s):
            a = scalar_step(self.F, a, self.lam, dt, self.b((n * self.s + j + 1) * dt))
        return a

    def coarse_sweep(self, a0):
        tr = [mp.mpf(a0)]
        for n in range(self.N):
            tr.append(self.coarse(n, tr[-1]))
        return tr

    def iteration(self, tr):
        new = [tr[0]]
        for n in range(self.N):
            new.append(self.coarse(n, new[-1]) + self.fine(n, tr[n]) - self.coarse(n, tr[n]))
        return new

    def fine_solution(self, a0):
        tr = [mp.mpf(a0)]
        for n in range(self.N):
            tr.append(self.fine(n, tr[-1]))
        return tr

    def run(self, a0, K):
        trs = [self.coarse_sweep(a0)]
        for _ in range(K):
            trs.append(self.iteration(trs[-1]))
        return trs


def sines(n, j):
    h = 1.0 / (n + 1)
    return [math.sin(j * math.pi * h * i) for i in range(1, n + 1)]
