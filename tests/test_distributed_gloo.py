"""Row-sharded orchestration on CPU: 2 ranks over gloo == 1 process.

The engine (_engine.py) is run with the test-only numpy backend and the
product communicator (distributed.TorchComm) over a gloo process group, so
the sharding, the all-reduce points and their order are exercised exactly
as on NVLink; only the per-rank arithmetic is numpy instead of libskp.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from np_backend import NumpyBackend
from oracle import skp_oracle as o
from paper_2605_09755_b200 import _engine
from paper_2605_09755_b200.distributed import TorchComm, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _NpComm:
    """Adapter: numpy arrays all-reduced through torch.distributed (gloo)."""

    def __init__(self, comm: TorchComm):
        self.comm, self.rank, self.world = comm, comm.rank, comm.world

    def allreduce_(self, a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        self.comm.allreduce_(t)
        return t.numpy()


def _problem(m=240, n=120, l=60, r2=12, seed=7):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, 40)))
    v, _ = np.linalg.qr(rng.standard_normal((n, 40)))
    a = (u * (0.8 ** np.arange(40))) @ v.T + 1e-6 * rng.standard_normal((m, n))
    sk = o.CountSketch("countsketch", n, l, o.substream(seed, 0), s=4)
    atil = sk.apply_right(a)
    omega = o.draw_omega(l, r2, o.substream(seed, 1))
    return a, atil, omega


def _worker(rank, world, port, q, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, atil, omega = _problem()
        row0, rows = shard_rows(a.shape[0], world, rank)
        comm = _NpComm(TorchComm())
        be = NumpyBackend()
        y = _engine.power_iterate(be, comm, atil[row0:row0 + rows], omega, q, True,
                                  rows_total=a.shape[0])
        qb = _engine.orthonormalize(be, comm, y, rows_total=a.shape[0])
        u, s, v = _engine.randsvd(be, comm, a[row0:row0 + rows], qb)
        out[rank] = (row0, qb, s, v)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q", [0, 2])
def test_two_rank_rsvd_matches_single_process(q):
    a, atil, omega = _problem()
    be = NumpyBackend()
    y = _engine.power_iterate(be, _engine.LOCAL, atil, omega, q, True)
    q1 = _engine.orthonormalize(be, _engine.LOCAL, y)
    _, s1, v1 = _engine.randsvd(be, _engine.LOCAL, a, q1)
    # the single-process engine agrees with the reference restatement (span)
    q_ref = o.orthonormalize(o.power_iterate(atil, omega, q))
    np.testing.assert_allclose(q1 @ q1.T, q_ref @ q_ref.T, atol=1e-8)

    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    qs = [out[r] for r in range(2)]
    q2 = np.vstack([qs[0][1], qs[1][1]])
    np.testing.assert_allclose(q2 @ q2.T, q1 @ q1.T, atol=1e-8)
    np.testing.assert_allclose(qs[0][2], s1, rtol=1e-10)
    np.testing.assert_allclose(qs[0][2], qs[1][2], rtol=0, atol=0)


def test_shard_rows_partition():
    for m in (1, 7, 262144, 1000003):
        for w in (1, 2, 3, 4, 8):
            parts = [shard_rows(m, w, r) for r in range(w)]
            assert parts[0][0] == 0
            assert sum(p[1] for p in parts) == m
            for (a0, ar), (b0, _) in zip(parts, parts[1:]):
                assert a0 + ar == b0
            assert max(p[1] for p in parts) - min(p[1] for p in parts) <= 1


def _pad_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        base = torch.full((5, 8), float(rank + 1))
        view = base[:, :6]                      # row-padded view, like _ops.empty2d
        TorchComm().allreduce_(view)
        out[rank] = view.clone().numpy()
    finally:
        dist.destroy_process_group()


def test_allreduce_padded_views():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_pad_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in range(2):
        np.testing.assert_array_equal(out[r], np.full((5, 6), 3.0))
