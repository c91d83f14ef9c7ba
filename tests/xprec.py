"""Extended-precision reference of one FIE / DR step (test infrastructure).

Purpose: a value close to the EXACT result of one splitting step, so that the rounding of the
oracle and of the CUDA path can each be bounded against it.  Everything is
evaluated in numpy's ``longdouble`` (x87 80-bit, eps = 2^-64 ~ 5.4e-20) straight from the
paper's formulas:

  FIE:  (I - tau A_1) V_1 = U_n + tau F_{n+1},  (I - tau A_j) V_j = V_{j-1}
  DR:  V_0 = (I + tau A) U_n + tau F_{n+1},
                           (I - tau A_j) V_j = V_{j-1} - tau A_j U_n,   U_{n+1} = V_M

with A = sum_j A_j (exact in real arithmetic, PAPER.md:63-67 / 111-134) and the split terms
written out here on the face-centred 5 / 7-point stencil (R4, R6, R15,
R16).  Each stage solve is iterative refinement: the residual b - (I - tau A_j) x is formed in
longdouble and the correction comes from a plain fp64 solve (the oracle's).  The fixed point
depends only on the longdouble residual, not on that solver, which only has to contract (its
backward error times cond(I - tau A_j) < 1).

Bound used by the tests: a backward-stable fp64 implementation of the step differs from the
exact value by a small multiple of eps64 * (|U_n| + |tau A U_n| + |tau F| + |U_{n+1}|): the
right-hand sides carry the rounding of those terms and ||(I - tau A_j)^{-1}||_inf <= 1 (the stage
matrices are M-matrices with unit row sums or more, SURVEY.md 8(c) uniqueness), so the solves
do not amplify it.  This extended-precision value's own error is ~eps80 * cond, far below it.
"""
from __future__ import annotations

import numpy as np

import oracle

LD = np.longdouble
PI = LD("3.141592653589793238462643383279502884")
EPS64 = 2.0 ** -52


class XStep:
    def __init__(self, p):
        assert p.coef in (0, 1), "5 / 7-point operators only"
        self.p = p
        self.n = p.n
        self.h = LD(1) / LD(p.n + 1)
        self.h2inv = LD(p.n + 1) * LD(p.n + 1)
        self.M = 2 if p.split else p.dim
        self.c = LD(repr(p.c)) if isinstance(p.c, float) else LD(p.c)
        self.o = oracle.Oracle(p)
        self.shape = (p.n,) * p.dim
        idx = np.arange(1, p.n + 1).astype(LD)
        self.x = idx * self.h                     # node coordinates
        self.xf = (np.arange(0, p.n + 1).astype(LD) + LD("0.5")) * self.h  # faces 1/2 .. n+1/2

    # ------------------------------------------------------------ coefficients
    def kappa(self, x, y):
        if self.p.coef == 1:
            return 1 + LD("0.5") * np.sin(2 * PI * x) * np.sin(2 * PI * y)
        return np.ones(np.broadcast(x, y).shape, dtype=LD)

    def rho0(self, pos):
        """rho_0 at 1-based positions (node i, face i + 1/2), R6: strips of w nodes,
        interface m at w m + 1/2, ramp of beta cells centred on it (linear or cosine)."""
        p = self.p
        S, w, beta = p.dd_strips, p.n // p.dd_strips, LD(p.dd_overlap)
        pos = np.asarray(pos, dtype=LD)
        out = np.empty(pos.shape, dtype=LD)
        for q, x in np.ndenumerate(pos):
            k = int(np.floor((float(x) - 0.5) / w))
            k = min(max(k, 0), S - 1)
            val = LD(1) if k % 2 == 0 else LD(0)
            for m in (k, k + 1):           # the interfaces bounding strip k
                if m < 1 or m > S - 1:
                    continue
                xl = LD(w * m) + LD("0.5") - beta / 2
                u = (x - xl) / beta
                if 0 < u < 1:
                    down = (1 - u) if p.dd_ramp == 0 else (1 + np.cos(PI * u)) / 2
                    val = down if (m - 1) % 2 == 0 else 1 - down
            out[q] = val
        return out

    # ------------------------------------------------------------ operators
    def apply(self, j, u):
        """tau-free A_j u (j < 0: the unsplit A = sum_j A_j) in longdouble."""
        if j < 0:
            return sum(self.apply(t, u) for t in range(self.M))
        u = np.asarray(u, dtype=LD)
        p = self.p
        if p.split == 1:
            return self._apply_dd(j, u)
        axis = p.dim - 1 - j  # x-fastest storage: x is the last array axis
        n = self.n
        um = np.zeros_like(u)
        up = np.zeros_like(u)
        sl = [slice(None)] * p.dim
        sl_a, sl_b = list(sl), list(sl)
        sl_a[axis], sl_b[axis] = slice(1, None), slice(None, -1)
        um[tuple(sl_a)] = u[tuple(sl_b)]   # u_{i-1}
        up[tuple(sl_b)] = u[tuple(sl_a)]   # u_{i+1}
        if p.dim == 2 and p.coef == 1:
            X, Y = self.x[None, :], self.x[:, None]
            if j == 0:
                km = self.kappa(self.xf[None, :n], Y)
                kp = self.kappa(self.xf[None, 1:], Y)
            else:
                km = self.kappa(X, self.xf[:n, None])
                kp = self.kappa(X, self.xf[1:, None])
        else:
            km = kp = LD(1)
        return (kp * (up - u) - km * (u - um)) * self.h2inv - (self.c / self.M) * u

    def _apply_dd(self, j, u):
        n = self.n
        r0n = self.rho0(np.arange(1, n + 1))
        r0f = self.rho0(np.arange(0, n + 1) + 0.5)
        rn = r0n if j == 0 else 1 - r0n
        rf = r0f if j == 0 else 1 - r0f
        X, Y = self.x[None, :], self.x[:, None]
        kxm = rf[None, :n] * self.kappa(self.xf[None, :n], Y)
        kxp = rf[None, 1:] * self.kappa(self.xf[None, 1:], Y)
        kym = rn[None, :] * self.kappa(X, self.xf[:n, None])
        kyp = rn[None, :] * self.kappa(X, self.xf[1:, None])
        z = np.zeros_like(u)
        xm, xp, ym, yp = z.copy(), z.copy(), z.copy(), z.copy()
        xm[:, 1:], xp[:, :-1] = u[:, :-1], u[:, 1:]
        ym[1:, :], yp[:-1, :] = u[:-1, :], u[1:, :]
        diff = (kxp * (xp - u) - kxm * (u - xm) + kyp * (yp - u) - kym * (u - ym)) * self.h2inv
        return diff - rn[None, :] * self.c * u

    def source(self, t):
        p = self.p
        if p.source == 0:
            return np.zeros(self.shape, dtype=LD)
        s = np.sin(PI * self.x)
        phi = np.multiply.outer(s, s) if p.dim == 2 else s[:, None, None] * s[None, :, None] * s[None, None, :]
        amp = LD(p.dim) * PI * PI + self.c - 1
        return amp * np.exp(-LD(repr(t))) * phi

    # ------------------------------------------------------------ solves / steps
    def solve(self, j, tau, b, iters=4):
        tau = LD(repr(tau))
        x = self.o.solve(j, float(tau), np.asarray(b, dtype=np.float64)).astype(LD)
        for _ in range(iters):
            r = b - (x - tau * self.apply(j, x))
            x = x + self.o.solve(j, float(tau), r.astype(np.float64)).astype(LD)
        return x

    def step(self, scheme, tau, t_next, u):
        """Returns (U_{n+1}, scale) with scale = |U_n| + |tau A U_n| + |tau F| + |U_{n+1}| (inf norms)."""
        u = np.asarray(u, dtype=LD).reshape(self.shape)
        T = LD(repr(tau))
        F = self.source(t_next)
        Au = self.apply(-1, u)
        if scheme == 0:
            v = u + T * F
            for j in range(self.M):
                v = self.solve(j, tau, v)
        else:
            v = u + T * Au + T * F
            for j in range(self.M):
                v = self.solve(j, tau, v - T * self.apply(j, u))
        nrm = lambda a: float(np.max(np.abs(a)))  # noqa: E731
        scale = nrm(u) + nrm(T * Au) + nrm(T * F) + nrm(v)
        return v, scale


def err_in_eps(got, ref, scale):
    """max |got - ref| / (eps64 * scale)."""
    d = np.max(np.abs(np.asarray(got, dtype=LD) - ref))
    return float(d) / (EPS64 * scale)
