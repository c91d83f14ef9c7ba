"""Multi-process host logic of the slice-sharded driver, world_size 2 over gloo on CPU.

The NCCL data path itself needs several GPUs; what is checked here is everything around it
that runs on the host: the slice partition every rank derives independently, the NCCL
unique-id marshalling through torch.distributed, and the owner-G schedule of §6 of
DESIGN.md (rank p receives U^{k+1}_{first} from p-1, runs its local coarse chain with the
correction, sends its last state to p+1, then a max all-reduce of the update) executed with
the CPU oracle's propagators over gloo, which must reproduce the serial parareal bit for bit
(result invariance across rank counts).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from synth import DR, FIE, Problem


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(rank, world, port, fn, q, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world, *args)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def spawn(fn, world=2, args=()):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


# ------------------------------------------------------------------ workers
def _partition_worker(rank, world, N):
    import paper_2502_08370_b200 as prs
    first, count = prs.partition(N, world, rank)
    allp = [None] * world
    dist.all_gather_object(allp, (first, count))
    return allp


def _uid_worker(rank, world):
    import paper_2502_08370_b200 as prs
    obj = [prs.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def _schedule_worker(rank, world, prob_kw, K):
    """Owner-G parareal over gloo with oracle propagators (reference model of the driver)."""
    import oracle
    import paper_2502_08370_b200 as prs
    p = Problem(**prob_kw)
    o = oracle.Oracle(p)
    first, count = prs.partition(p.N, world, rank)
    u0 = synth.initial_state(p)
    shape = u0.shape
    # local trajectory: [0] incoming state U_first, [i] = U_{first+i}
    traj = np.zeros((count + 1,) + shape)
    gcache = np.zeros((count,) + shape)

    def recv_in():
        t = torch.zeros(shape, dtype=torch.float64)
        dist.recv(t, src=rank - 1)
        traj[0] = t.numpy()

    def send_out():
        dist.send(torch.from_numpy(np.ascontiguousarray(traj[count])), dst=rank + 1)

    # coarse sweep
    if rank == 0:
        traj[0] = u0
    else:
        recv_in()
    for i in range(count):
        g = o.coarse(first + i, traj[i])
        traj[i + 1] = g
        gcache[i] = g
    if rank < world - 1:
        send_out()
    hist = []
    for _ in range(K):
        delta = np.stack([o.fine(first + i, traj[i]) - gcache[i] for i in range(count)])
        if rank > 0:
            recv_in()
        upd = 0.0
        for i in range(count):
            g = o.coarse(first + i, traj[i])
            new = g + delta[i]
            upd = max(upd, float(np.max(np.abs(new - traj[i + 1]))))
            gcache[i] = g
            traj[i + 1] = new
        if rank < world - 1:
            send_out()
        t = torch.tensor([upd], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        hist.append(float(t.item()) / float(np.max(np.abs(u0))))
    return first, traj[1:].copy(), hist


# -------------------------------------------------------------------- tests
@pytest.mark.parametrize("N", [8, 64, 7])
def test_partition_agrees_across_ranks(N):
    out = spawn(_partition_worker, 2, (N,))
    parts = out[0]
    assert parts == out[1]
    assert parts[0][0] == 0 and parts[0][0] + parts[0][1] == parts[1][0]
    assert parts[1][0] + parts[1][1] == N


def test_nccl_unique_id_broadcast():
    out = spawn(_uid_worker, 2)
    assert isinstance(out[0], bytes) and len(out[0]) == 128
    assert out[0] == out[1]


@pytest.mark.parametrize("kw", [
    dict(dim=2, n=12, N=6, s=3, G=FIE, F=FIE, source=1),
    dict(dim=2, n=12, N=5, s=3, G=FIE, F=DR, coef=1, init="modes"),
    dict(dim=2, n=16, N=4, s=2, split=1, dd_strips=4, dd_overlap=2, G=DR, F=FIE, source=1),
])
def test_owner_g_schedule_reproduces_serial_parareal(kw):
    import oracle
    K = 3
    out = spawn(_schedule_worker, 2, (kw, K))
    p = Problem(**kw)
    u0 = synth.initial_state(p)
    trajs, upds = oracle.Oracle(p).parareal(u0, K, fixed=True)
    full = np.zeros_like(trajs[-1])
    full[0] = u0
    for r in (0, 1):
        first, local, hist = out[r]
        full[first + 1:first + 1 + len(local)] = local
        # update norms identical on every rank (max all-reduce) and equal to the serial ones
        # (g + Delta vs the oracle's (g + F) - G: rounding of iterate-sized values)
        assert np.allclose(hist, upds, rtol=0.0, atol=1e-14)
    assert out[0][2] == out[1][2]
    scale = max(float(np.max(np.abs(t))) for t in trajs)
    assert float(np.max(np.abs(full - trajs[-1]))) / scale <= 1e-14


# ------------------------------------------- space-parallel G: band exchange plan
def _gpar_plan_worker(rank, world, N, L):
    """Execute this rank's prs_gpar_plan (the ops prs_parareal_correct issues to NCCL) with
    gloo point-to-point on tagged CPU data; return what landed where."""
    import paper_2502_08370_b200 as prs
    P = world
    first, count = prs.partition(N, P, rank)
    code = lambda sl, band, kind: float(1000 * sl + 10 * band + kind)  # noqa: E731
    delta = torch.stack([torch.stack([torch.full((L,), code(first + i, p, 1)) for p in range(P)])
                         for i in range(count)])
    traj = torch.full((count + 1, P, L), -1.0)
    gcache = torch.full((count, P, L), -1.0)
    gb_d = torch.full((N, L), -1.0)
    gb_u = torch.stack([torch.full((L,), code(sl, rank, 2)) for sl in range(N + 1)])
    gb_gc = torch.stack([torch.full((L,), code(sl, rank, 3)) for sl in range(N)])
    # the owner's U^k end states (local index 1..count), tagged 4, for the seed phase
    trajk = torch.stack([torch.stack([torch.full((L,), code(first + i, p, 4)) for p in range(P)])
                         for i in range(count + 1)])
    seeded = torch.full((N + 1, L), -1.0)
    for phase in (2, 0, 1):
        reqs = []
        for kind, what, sl, band, peer, lidx in prs.gpar_plan(N, P, rank, phase):
            if phase == 2:
                assert what == 1
                src, dst = (trajk[lidx, band] if kind != 1 else None), seeded[sl + 1]
            elif phase == 0:
                src, dst = (delta[lidx, band] if kind != 1 else None), gb_d[sl]
            else:
                src = gb_u[sl + 1] if what == 1 else gb_gc[sl]
                dst = (traj if what == 1 else gcache)[lidx, band] if kind != 0 else None
            if kind == 2:
                dst.copy_(src)
            elif kind == 0:
                reqs.append(dist.isend(src.contiguous(), peer))
            else:
                buf = torch.empty(L)
                reqs.append((dist.irecv(buf, peer), buf, dst))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                r[2].copy_(r[1])
            else:
                r.wait()
    return {"first": first, "count": count, "gb_d": gb_d[:, 0].tolist(), "seeded": seeded[:, 0].tolist(),
            "traj": traj[:, :, 0].tolist(), "gcache": gcache[:, :, 0].tolist()}


@pytest.mark.parametrize("world,N", [(2, 8), (3, 7), (4, 8)])
def test_space_parallel_g_exchange_plan(world, N):
    """SURVEY 8(e) space-parallel G: the seed phase gives every rank its band of the current
    iterate U^k_1..U^k_N, Delta bands reach their band ranks and every owner gets back all P
    bands of its U_{n+1}, its incoming U_first and its G cache (the exact op list
    prs_parareal_correct issues to the transport, run over gloo)."""
    import paper_2502_08370_b200 as prs
    prs.build()  # no-op when libprs.so is current (host logic only: no GPU needed)
    prs.lib()
    out = spawn(_gpar_plan_worker, world=world, args=(N, 3))
    for rank in range(world):
        o = out[rank]
        assert not isinstance(o, str), o
        first, count = o["first"], o["count"]
        assert o["gb_d"] == [1000.0 * sl + 10 * rank + 1 for sl in range(N)]
        # seed: this rank's band of every U^k_{n+1}, n = 0..N-1, from the slice owners
        assert o["seeded"][1:] == [1000.0 * (sl + 1) + 10 * rank + 4 for sl in range(N)]
        for i in range(1, count + 1):
            assert o["traj"][i] == [1000.0 * (first + i) + 10 * p + 2 for p in range(world)]
        if rank > 0:
            assert o["traj"][0] == [1000.0 * first + 10 * p + 2 for p in range(world)]
        for i in range(count):
            assert o["gcache"][i] == [1000.0 * (first + i) + 10 * p + 3 for p in range(world)]
