"""N>1 host logic on CPU with gloo (world size 2 and 4).

The distributed path sends, per refresh phase and peer, the concatenation of
the boxes of the library's exchange plan (sf_exchange_plan; the same plan the
CUDA driver packs, ships over NCCL and unpacks).  Here every rank holds its
padded block in the reference layout (field.hpp:31-52) as a numpy array, packs
and unpacks per that plan and ships the messages with torch.distributed
send/recv over gloo in the plan's posting order.  After the three axis phases
every ghost must equal the global array at the wrapped coordinate -- the
reference's own check, tests/test_grid.cpp:195-252.  The residual reduction
is checked as the driver does it: allreduce(max) of IEEE bit patterns.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1201_2118_b200 as sfb
from paper_1201_2118_b200 import _lib


def plan(ext, world, ghost, periodic, rank, mask, axis):
    lib = sfb.lib()
    e = (C.c_int64 * 3)(*ext)
    per = (C.c_int * 3)(*[1 if p else 0 for p in periodic])
    n = C.c_int()
    _lib.check(lib.sf_exchange_plan(e, world, ghost, per, rank, mask, axis, 0, None, C.byref(n)))
    out = (C.c_int64 * (15 * max(1, n.value)))()
    _lib.check(lib.sf_exchange_plan(e, world, ghost, per, rank, mask, axis, n.value, out, C.byref(n)))
    rows = [list(out[15 * i: 15 * i + 15]) for i in range(n.value)]
    return [dict(kind=r[0], peer=r[1], field=r[2], axis=r[3], side=r[4], lo=r[5:8], dims=r[8:11],
                 dlo=r[11:14], count=r[14]) for r in rows]


def cell_tag(i, j, k):  # tests/test_grid.cpp:22-26
    return i + 1000.0 * j + 1000000.0 * k


def box_view(a, g, lo, dims):
    return a[lo[2] + g: lo[2] + g + dims[2], lo[1] + g: lo[1] + g + dims[1], lo[0] + g: lo[0] + g + dims[0]]


def exchange_on_rank(rank, world, ext, ghost, periodic, faces_only):
    d = sfb.decompose(ext, world, ghost, periodic)
    lo, dims = d.lo[rank], d.size(rank)
    g = ghost
    a = np.full((dims[2] + 2 * g, dims[1] + 2 * g, dims[0] + 2 * g), np.nan)
    kk, jj, ii = np.meshgrid(np.arange(dims[2]), np.arange(dims[1]), np.arange(dims[0]), indexing="ij")
    a[g:-g, g:-g, g:-g] = cell_tag(ii + lo[0], jj + lo[1], kk + lo[2])
    for axis in ([-1] if faces_only else [0, 1, 2]):
        P = plan(ext, world, ghost, periodic, rank, 1, axis)
        for p in P:
            if p["kind"] == 2:  # copy inside this rank (periodic self-wrap)
                box_view(a, g, p["dlo"], p["dims"])[...] = box_view(a, g, p["lo"], p["dims"])
        sends, recvs = {}, {}
        for p in P:
            if p["kind"] == 0:
                sends.setdefault(p["peer"], []).append(p)
            elif p["kind"] == 1:
                recvs.setdefault(p["peer"], []).append(p)
        ops, rbufs = [], {}
        for peer in sorted(sends):
            buf = np.concatenate([box_view(a, g, p["lo"], p["dims"]).reshape(-1) for p in sends[peer]])
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(buf.copy()), peer))
        for peer in sorted(recvs):
            rbufs[peer] = torch.empty(sum(p["count"] for p in recvs[peer]), dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, rbufs[peer], peer))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for peer, buf in rbufs.items():
            off = 0
            for p in recvs[peer]:
                n = p["count"]
                box_view(a, g, p["lo"], p["dims"])[...] = buf[off: off + n].numpy().reshape(p["dims"][::-1])
                off += n
    return a, lo, dims


def check_ghosts(a, lo, dims, ext, g, periodic, d, rank, faces_only):
    bad = 0
    for k in range(-g, dims[2] + g):
        for j in range(-g, dims[1] + g):
            for i in range(-g, dims[0] + g):
                c = (i, j, k)
                out = [x < 0 or x >= dims[t] for t, x in enumerate(c)]
                if not any(out):
                    continue
                if faces_only and sum(out) > 1:
                    continue  # the fused loop exchanges faces only
                # is every out-of-block axis a processor (or wrapped) face?
                proc = True
                self_wrap = False
                for t in range(3):
                    if out[t]:
                        side = 0 if c[t] < 0 else 1
                        nb = d.neighbor(rank, t, side)
                        if nb < 0:
                            proc = False
                        self_wrap = self_wrap or nb == rank
                v = a[k + g, j + g, i + g]
                if faces_only and self_wrap:
                    continue  # the half-sweep kernel writes periodic self-wraps itself
                if not proc:
                    bad += 0 if np.isnan(v) else 1  # physical ghosts are not ours to fill here
                    continue
                gc = [(lo[t] + c[t]) % ext[t] for t in range(3)]
                if v != cell_tag(*gc):
                    bad += 1
    return bad


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for ext, ghost, periodic, faces_only in cases:
            d = sfb.decompose(ext, world, ghost, periodic)
            a, lo, dims = exchange_on_rank(rank, world, ext, ghost, periodic, faces_only)
            results.append(check_ghosts(a, lo, dims, ext, ghost, periodic, d, rank, faces_only))
        # residual: allreduce(max) of |x| bit patterns (the driver's NCCL call)
        def vals_of(r):
            v = np.abs(np.random.default_rng(r).standard_normal(64))
            if r == world - 1:
                v[7] = np.nan
            return v
        bits = torch.from_numpy(vals_of(rank).view(np.int64).copy())
        dist.all_reduce(bits, op=dist.ReduceOp.MAX)
        got = bits.numpy().view(np.float64)
        want = np.max(np.stack([vals_of(r) for r in range(world)]), axis=0)  # NaN-sticky
        results.append(int(np.array_equal(got, want, equal_nan=True)))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(world, cases):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


CASES = [
    ((12, 10, 9), 1, (True, True, True), False),
    ((12, 10, 9), 2, (True, False, True), False),
    ((11, 8, 7), 1, (False, False, False), False),
    ((12, 10, 9), 1, (True, True, True), True),
    ((11, 8, 7), 1, (False, False, False), True),
    # the temporal pass's per-pass exchange: 2 deep, no periodic axis
    ((14, 12, 10), 2, (False, False, False), False),
]


def test_two_ranks_exchange_every_ghost_like_the_global_oracle():
    out = run_world(2, CASES)
    for rank, res in out.items():
        assert res[:-1] == [0] * len(CASES), (rank, res)
        assert res[-1] == 1  # NaN-sticky max over ranks


def test_four_ranks_with_shared_periodic_faces():
    # (2,2,1) process grid: both x faces of a rank face the same peer when periodic
    out = run_world(4, CASES[:2] + CASES[3:4] + CASES[5:6])
    for rank, res in out.items():
        assert res[:-1] == [0, 0, 0, 0], (rank, res)


def test_plan_counts_match_between_peers():
    ext, g = (13, 9, 8), 2
    for world, per in [(2, (True, True, True)), (4, (True, False, True)), (8, (False, False, False))]:
        for axis in (-1, 0, 1, 2):
            sent, recv = {}, {}
            for r in range(world):
                for p in plan(ext, world, g, per, r, 0b10011, axis):
                    if p["kind"] == 0:
                        sent.setdefault((r, p["peer"]), []).append(p["count"])
                    elif p["kind"] == 1:
                        recv.setdefault((p["peer"], r), []).append(p["count"])
            assert sent.keys() == recv.keys()
            for k in sent:
                assert sent[k] == recv[k], (world, axis, k)


# ---- the temporal pass's direct-store exchange (sf_direct_plan) -------------------
def direct_plan(ext, world, ghost, periodic, rank):
    lib = sfb.lib()
    e = (C.c_int64 * 3)(*ext)
    per = (C.c_int * 3)(*[1 if p else 0 for p in periodic])
    n = C.c_int()
    out = (C.c_int64 * (14 * 26))()
    _lib.check(lib.sf_direct_plan(e, world, ghost, per, rank, 26, out, C.byref(n)))
    rows = [list(out[14 * i: 14 * i + 14]) for i in range(n.value)]
    return [dict(peer=r[0], d=r[1:4], lo=r[4:7], dims=r[7:10], dlo=r[10:13], count=r[13]) for r in rows]


def direct_exchange_on_rank(rank, world, ext, ghost, periodic):
    """The driver's direct stores (k_tasks type 4) restated: every box of this
    rank's plan goes straight into the peer's ghost shell; here the boxes of
    one peer travel as one gloo message in plan order, and the receiver places
    them with the sender's plan (the device stores need no message at all)."""
    d = sfb.decompose(ext, world, ghost, periodic)
    lo, dims = d.lo[rank], d.size(rank)
    g = ghost
    a = np.full((dims[2] + 2 * g, dims[1] + 2 * g, dims[0] + 2 * g), np.nan)
    kk, jj, ii = np.meshgrid(np.arange(dims[2]), np.arange(dims[1]), np.arange(dims[0]), indexing="ij")
    a[g:-g, g:-g, g:-g] = cell_tag(ii + lo[0], jj + lo[1], kk + lo[2])
    mine = direct_plan(ext, world, ghost, periodic, rank)
    sends = {}
    for b in mine:
        sends.setdefault(b["peer"], []).append(box_view(a, g, b["lo"], b["dims"]).reshape(-1).copy())
    incoming = {}
    for p in range(world):
        if p == rank:
            continue
        boxes = [b for b in direct_plan(ext, world, ghost, periodic, p) if b["peer"] == rank]
        if boxes:
            incoming[p] = boxes
    reqs, bufs = [], {}
    for p, parts in sends.items():
        reqs.append(dist.isend(torch.from_numpy(np.concatenate(parts)), dst=p))
    for p, boxes in incoming.items():
        bufs[p] = torch.empty(sum(b["count"] for b in boxes), dtype=torch.float64)
        reqs.append(dist.irecv(bufs[p], src=p))
    for r in reqs:
        r.wait()
    for p, boxes in incoming.items():
        flat, at = bufs[p].numpy(), 0
        for b in boxes:
            box_view(a, g, b["dlo"], b["dims"])[...] = flat[at:at + b["count"]].reshape(b["dims"][::-1])
            at += b["count"]
    return a, lo, dims


def _worker_direct(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        results = []
        for ext, ghost, periodic in cases:
            d = sfb.decompose(ext, world, ghost, periodic)
            a, lo, dims = direct_exchange_on_rank(rank, world, ext, ghost, periodic)
            # the same ghosts as the three exchange-only axis phases deliver
            results.append(check_ghosts(a, lo, dims, ext, ghost, periodic, d, rank, False))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


def run_world_direct(world, cases):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_direct, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


# every periodic axis split over >= 2 ranks (the temporal pass's precondition:
# no self-wrap); 2-deep and 3-deep shells, uneven blocks
DIRECT_CASES = [
    ((14, 12, 10), 2, (False, False, False)),
    ((15, 11, 9), 2, (True, False, False)),
    ((13, 12, 11), 3, (False, False, False)),
]


def test_direct_store_plan_fills_the_ghosts_of_the_exchange_phases_two_ranks():
    out = run_world_direct(2, DIRECT_CASES)
    for rank, res in out.items():
        assert res == [0] * len(DIRECT_CASES), (rank, res)


def test_direct_store_plan_with_edges_and_corners_four_ranks():
    # (2,2,1): edge neighbours (diagonals), and with periodic x and y both x
    # (and y) faces of a rank face the same peer
    out = run_world_direct(4, DIRECT_CASES[:1] + [((14, 12, 10), 2, (True, True, False))])
    for rank, res in out.items():
        assert res == [0, 0], (rank, res)


def test_direct_store_plan_is_symmetric_between_peers():
    # what rank r stores into peer p is exactly what p's ghost boxes expect:
    # same count per direction, and opposite directions pair up
    for world, ext, per in [(2, (14, 12, 10), (True, False, False)), (4, (14, 12, 10), (False, False, False)),
                            (8, (12, 12, 12), (True, True, True))]:
        plans = {r: direct_plan(ext, world, 2, per, r) for r in range(world)}
        for r, P in plans.items():
            for b in P:
                back = [c for c in plans[b["peer"]] if c["peer"] == r and c["d"] == [-x for x in b["d"]]]
                assert back and back[0]["count"] == b["count"], (world, r, b)


def _worker_transport(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1201_2118_b200.sim import _TorchHostTransport
        t = _TorchHostTransport()
        # call through the C function pointers the library receives
        ag = C.cast(C.cast(t.c.allgather, C.c_void_p), _lib.ALLGATHER_FN)
        bar = C.cast(C.cast(t.c.barrier, C.c_void_p), _lib.BARRIER_FN)
        send = (C.c_uint64 * 3)(rank, 100 + rank, 2 ** 63 + rank)
        recv = (C.c_uint64 * (3 * world))()
        rc1 = ag(None, C.cast(send, C.c_void_p), C.cast(recv, C.c_void_p), 24)
        rc2 = bar(None)
        want = [v for r in range(world) for v in (r, 100 + r, 2 ** 63 + r)]
        q.put((rank, [rc1, rc2, list(recv) == want]))
    finally:
        dist.destroy_process_group()


def test_host_transport_callbacks_over_gloo():
    # the allgather / barrier callbacks of the CUDA-IPC transport
    # (sf_host_transport) as the library calls them: rank-ordered bytes
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_transport, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(3))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in out.items():
        assert res == [0, 0, True], (rank, res)
