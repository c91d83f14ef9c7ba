"""B200-native parareal with splitting propagators (arXiv 2502.08370).

Thin Python binding of the C ABI in ``include/prs.h`` (argument marshalling only).  Every
step of the method runs in the sm_100a kernels of ``libprs.so``; there is no Python or CPU
fallback: importing the binding without the built library raises.

    from paper_2502_08370_b200 import Problem, Context
    ctx = Context(problem, stream=torch.cuda.current_stream().cuda_stream)
    ctx.set_initial(u0); ctx.coarse_sweep(); k, hist = ctx.iterate(kmax, tol)
"""
from __future__ import annotations

import ctypes
import os

from ._build import SO, build  # noqa: F401

PRS_OK, PRS_EINVAL, PRS_EDIVERGED, PRS_EUNSUPPORTED, PRS_ECUDA, PRS_ENCCL = 0, 2, 3, 4, 5, 6
PRS_FIE, PRS_DR, PRS_IE = 0, 1, 2
PRS_K_XPASS, PRS_K_LPASS, PRS_K_DD, PRS_K_IE = 0, 1, 2, 3
EXPORTS = ["prs_create", "prs_nccl_unique_id", "prs_partition", "prs_set_initial",
           "prs_coarse_sweep", "prs_fine_sweep", "prs_parareal_correct", "prs_iterate",
           "prs_get_slice", "prs_step", "prs_step_batch", "prs_fine_solve", "prs_set_coarse_mode", "prs_set_pipeline", "prs_gpar_plan", "prs_set_profiling", "prs_launches", "prs_kernel_stats",
           "prs_last_error", "prs_destroy", "prs_local_world_create", "prs_local_world_destroy",
           "prs_create_local", "prs_set_ownership"]


class PrsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"prs error {code}: {msg}")
        self.code = code


class prs_problem(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("n", ctypes.c_int), ("c", ctypes.c_double),
                ("coef_kind", ctypes.c_int), ("split", ctypes.c_int), ("dd_strips", ctypes.c_int),
                ("dd_overlap", ctypes.c_int), ("dd_ramp", ctypes.c_int),
                ("source_kind", ctypes.c_int), ("T", ctypes.c_double), ("N", ctypes.c_int),
                ("s", ctypes.c_int), ("G", ctypes.c_int), ("F", ctypes.c_int)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libprs.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        so = os.environ.get("PRS_SO", SO)  # (test hook: the checked build libprs_chk.so)
        if not os.path.exists(so):
            raise ImportError(f"{SO} is missing: run paper_2502_08370_b200._build.build() "
                              "(or __graft_entry__.build()); there is no fallback path")
        L = ctypes.CDLL(so)
        V, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        PI, PD, PL = ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), \
            ctypes.POINTER(ctypes.c_longlong)
        sig = {
            "prs_create": ([ctypes.POINTER(prs_problem), I, I, V, V, ctypes.POINTER(V)], I),
            "prs_nccl_unique_id": ([V], I),
            "prs_partition": ([I, I, I, PI, PI], I),
            "prs_set_initial": ([V, V, I], I),
            "prs_coarse_sweep": ([V], I),
            "prs_fine_sweep": ([V], I),
            "prs_parareal_correct": ([V, PD], I),
            "prs_iterate": ([V, I, D, PI, PD], I),
            "prs_get_slice": ([V, I, V, I], I),
            "prs_step": ([V, I, D, D, V, V], I),
            "prs_step_batch": ([V, I, I, I, V, V, I], I),
            "prs_fine_solve": ([V, V, I, I, V, I], I),
            "prs_set_coarse_mode": ([V, I, I], I),
            "prs_set_pipeline": ([V, I], I),
            "prs_gpar_plan": ([I, I, I, I, PI, I], I),
            "prs_set_profiling": ([V, I], I),
            "prs_launches": ([V], ctypes.c_longlong),
            "prs_kernel_stats": ([V, I, PL, PD, PD], I),
            "prs_last_error": ([V], ctypes.c_char_p),
            "prs_destroy": ([V], None),
            "prs_local_world_create": ([I, ctypes.POINTER(V)], I),
            "prs_local_world_destroy": ([V], None),
            "prs_create_local": ([ctypes.POINTER(prs_problem), I, V, V, ctypes.POINTER(V)], I),
            "prs_set_ownership": ([V, I], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def to_c_problem(p) -> prs_problem:
    """Marshal a ``synth.Problem``-like object into the C struct."""
    return prs_problem(dim=p.dim, n=p.n, c=p.c, coef_kind=p.coef, split=p.split,
                       dd_strips=p.dd_strips, dd_overlap=p.dd_overlap, dd_ramp=p.dd_ramp,
                       source_kind=p.source, T=p.T, N=p.N, s=p.s, G=p.G, F=p.F)


def partition(N: int, nranks: int, rank: int):
    first, count = ctypes.c_int(), ctypes.c_int()
    rc = lib().prs_partition(N, nranks, rank, ctypes.byref(first), ctypes.byref(count))
    if rc != PRS_OK:
        raise PrsError(rc, "bad partition arguments")
    return first.value, count.value


def gpar_plan(N: int, nranks: int, rank: int, phase: int):
    """Space-parallel G band exchange of `rank` (host logic, no GPU): list of
    (kind, what, slice, band, peer, local_index) records, see include/prs.h."""
    L = lib()
    cnt = L.prs_gpar_plan(N, nranks, rank, phase, None, 0)
    if cnt < 0:
        raise PrsError(PRS_EINVAL, "bad gpar_plan arguments")
    buf = (ctypes.c_int * (6 * max(cnt, 1)))()
    L.prs_gpar_plan(N, nranks, rank, phase, buf, cnt)
    return [tuple(buf[6 * i: 6 * i + 6]) for i in range(cnt)]


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().prs_nccl_unique_id(buf)
    if rc != PRS_OK:
        raise PrsError(rc, "ncclGetUniqueId failed")
    return buf.raw


class LocalWorld:
    """prs_local_world_create: `nranks` in-process ranks on the current device (tests of the
    multi-rank driver; each rank's Context is driven by its own host thread)."""

    def __init__(self, nranks: int):
        self.L = lib()
        h = ctypes.c_void_p()
        rc = self.L.prs_local_world_create(nranks, ctypes.byref(h))
        if rc != PRS_OK:
            raise PrsError(rc, "prs_local_world_create failed")
        self.h, self.nranks = h, nranks

    def close(self):
        if getattr(self, "h", None):
            self.L.prs_local_world_destroy(self.h)
            self.h = None


class Context:
    """One prs_ctx.  Tensors passed in must be contiguous float64 CUDA tensors (or, for the
    host-buffer calls, contiguous float64 CPU tensors / numpy arrays)."""

    def __init__(self, prob, rank: int = 0, nranks: int = 1, nccl_uid: bytes | None = None,
                 stream: int | None = None, world: LocalWorld | None = None):
        self.L = lib()
        self.prob = prob
        self._cp = to_c_problem(prob)
        h = ctypes.c_void_p()
        if world is not None:
            nranks = world.nranks
            rc = self.L.prs_create_local(ctypes.byref(self._cp), rank, world.h, stream, ctypes.byref(h))
        else:
            uid = ctypes.create_string_buffer(nccl_uid, 128) if nccl_uid else None
            rc = self.L.prs_create(ctypes.byref(self._cp), rank, nranks, uid, stream, ctypes.byref(h))
        if rc != PRS_OK:
            raise PrsError(rc, "prs_create failed (see stderr)")
        self.h = h
        self.rank, self.nranks = rank, nranks
        self.first, self.count = partition(prob.N, nranks, rank)

    def _check(self, rc):
        if rc != PRS_OK:
            raise PrsError(rc, self.L.prs_last_error(self.h).decode())
        return rc

    def close(self):
        if getattr(self, "h", None):
            self.L.prs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ptr(self, x, states: int = 1, need_cuda: bool = False):
        """Pointer of a contiguous float64 buffer of `states` states (n^dim doubles each): a
        torch tensor (CUDA: on the context's device; CPU) or a numpy array.  Anything else is
        rejected here, before it can reach the ABI as a wrong-typed or wrong-sized pointer."""
        need = states * self.prob.n ** self.prob.dim
        if hasattr(x, "data_ptr"):
            import torch
            if x.dtype != torch.float64 or not x.is_contiguous() or x.numel() < need:
                raise ValueError(f"need a contiguous float64 tensor of >= {need} elements, got "
                                 f"{x.dtype} {tuple(x.shape)} contiguous={x.is_contiguous()}")
            if x.is_cuda and x.device.index != torch.cuda.current_device():
                raise ValueError(f"tensor on {x.device}, context on cuda:{torch.cuda.current_device()}")
            if need_cuda and not x.is_cuda:
                raise ValueError("this call takes device buffers (CUDA tensors)")
            return ctypes.c_void_p(x.data_ptr()), bool(x.is_cuda)
        import numpy as np
        if need_cuda:
            raise ValueError("this call takes device buffers (CUDA tensors)")
        if not isinstance(x, np.ndarray) or x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"] \
                or x.size < need:
            raise ValueError(f"need a C-contiguous float64 array of >= {need} elements")
        return ctypes.c_void_p(x.ctypes.data), False

    def set_initial(self, u0):
        p, dev = self._ptr(u0)
        self._check(self.L.prs_set_initial(self.h, p, int(dev)))

    def coarse_sweep(self):
        self._check(self.L.prs_coarse_sweep(self.h))

    def fine_sweep(self):
        self._check(self.L.prs_fine_sweep(self.h))

    def parareal_correct(self) -> float:
        upd = ctypes.c_double()
        self._check(self.L.prs_parareal_correct(self.h, ctypes.byref(upd)))
        return upd.value

    def iterate(self, kmax: int, tol: float):
        k = ctypes.c_int()
        hist = (ctypes.c_double * max(kmax, 1))()
        rc = self.L.prs_iterate(self.h, kmax, tol, ctypes.byref(k), hist)
        self._check(rc)
        return k.value, [hist[i] for i in range(k.value)]

    def get_slice(self, n: int, out):
        p, dev = self._ptr(out)
        self._check(self.L.prs_get_slice(self.h, n, p, int(dev)))
        return out

    def step(self, scheme: int, tau: float, t_next: float, inp, out):
        pi, _ = self._ptr(inp, need_cuda=True)
        po, _ = self._ptr(out, need_cuda=True)
        self._check(self.L.prs_step(self.h, scheme, tau, t_next, pi, po))
        return out

    def step_batch(self, which: int, slice0: int, j: int, inp, out, B: int):
        pi, _ = self._ptr(inp, B, need_cuda=True)
        po, _ = self._ptr(out, B, need_cuda=True)
        self._check(self.L.prs_step_batch(self.h, which, slice0, j, pi, po, B))
        return out

    def fine_solve(self, u0, out, nslices: int | None = None):
        """Sequential fine solution: nslices * s fine steps from u0 (default: all N slices)."""
        pi, di = self._ptr(u0)
        po, do = self._ptr(out)
        ns = self.prob.N if nslices is None else nslices
        self._check(self.L.prs_fine_solve(self.h, pi, int(di), ns, po, int(do)))
        return out

    def set_coarse_mode(self, mode: int, bands: int = 0):
        """0: owner-G chain; 1: space-parallel G over P row bands (P = nranks, or `bands`
        virtual bands on one rank)."""
        self._check(self.L.prs_set_coarse_mode(self.h, mode, bands))

    def set_ownership(self, mode: int):
        """0: contiguous slice blocks; 1: cyclic (slice n on rank n mod P), see include/prs.h."""
        self._check(self.L.prs_set_ownership(self.h, mode))
        self.cyclic = mode == 1 and self.nranks > 1
        if self.cyclic:
            self.first, self.count = self.rank, len(range(self.rank, self.prob.N, self.nranks))
        else:
            self.first, self.count = partition(self.prob.N, self.nranks, self.rank)

    def slices(self):
        """Global indices of this rank's slices."""
        if getattr(self, "cyclic", False):
            return list(range(self.rank, self.prob.N, self.nranks))
        return list(range(self.first, self.first + self.count))

    def set_pipeline(self, blocks: int):
        """Pipelined parareal for iterate(): `blocks` slice blocks (0: off)."""
        self._check(self.L.prs_set_pipeline(self.h, blocks))

    def set_profiling(self, on: bool):
        self._check(self.L.prs_set_profiling(self.h, int(on)))

    def launches(self) -> int:
        return int(self.L.prs_launches(self.h))

    def kernel_stats(self, kind: int):
        n, ms, by = ctypes.c_longlong(), ctypes.c_double(), ctypes.c_double()
        self._check(self.L.prs_kernel_stats(self.h, kind, ctypes.byref(n), ctypes.byref(ms),
                                            ctypes.byref(by)))
        return n.value, ms.value, by.value
