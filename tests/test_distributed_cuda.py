"""Row-sharded CUDA engine with 2 ranks == 1 rank.

Two processes over gloo share cuda:0 and run the product drivers
(``distributed.rsvd_sharded`` / ``nystrom_sharded``) on ``CudaBackend`` with
the product ``TorchComm``: every per-rank kernel is libskp, and the exchanges
are the real all-reduces -- the lazy failure flags, the non-finite count,
||A||_F^2, Z = sum A~_p^T Y_p, the Grams, B^T and W~.  Each rank holds its own
row slab (its own fp16 split exponents).  The ranks do not wait on each other
inside kernels (gloo all-reduces run between launches), so sharing one GPU
is safe.  The 2-rank results must match the 1-rank results.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

M, N, L, R2, K, Q = 65536, 2048, 512, 96, 64, 2
NK = 4096


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spec():
    import paper_2605_09755_b200 as skp
    return skp.RangeFinderSpec(k=K, l=L, r1=L, r2=R2, q=Q, eps=0.5, seed=13, s=8)


def _nspec():
    import paper_2605_09755_b200 as skp
    return skp.RangeFinderSpec(k=64, l=512, r1=512, r2=64, q=2, eps=0.5, seed=4, s=8)


def _inputs(row0, rows, krow0, krows):
    from paper_2605_09755_b200 import datagen
    spec_v = np.arange(1.0, 1025.0) ** -0.5
    a = datagen.lowrank_plus_noise_gpu(M, N, spec_v, 1e-6, seed=3, row0=row0, rows=rows)
    x = datagen.rbf_points(NK, 16, seed=4)
    h = datagen.rbf_bandwidth(x, NK, seed=4)
    kmat = datagen.rbf_kernel_gpu(x, h, row0=krow0, rows=krows)
    return a, kmat


def _run(comm, rank, world):
    from paper_2605_09755_b200 import distributed as D
    row0, rows = D.shard_rows(M, world, rank)
    krow0, krows = D.shard_rows(NK, world, rank)
    a, kmat = _inputs(row0, rows, krow0, krows)
    u, s, v, rel = D.rsvd_sharded(a, _spec(), M, comm, with_error=True)
    c, w = D.nystrom_sharded(kmat, _nspec(), krow0, NK, comm)
    return dict(u=u.double().cpu().numpy(), s=s.double().cpu().numpy(),
                v=v.double().cpu().numpy(), rel=rel, c=c.double().cpu().numpy(),
                w=w.double().cpu().numpy())


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_09755_b200 import distributed as D
        r = _run(D.TorchComm(), rank, world)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **r)
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_cuda_match_one(tmp_path):
    from paper_2605_09755_b200 import _engine
    one = _run(_engine.LOCAL, 0, 1)
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    r0, r1 = (dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(2))
    # replicated outputs agree across ranks bit for bit (same all-reduced inputs)
    np.testing.assert_array_equal(r0["s"], r1["s"])
    np.testing.assert_array_equal(r0["w"], r1["w"])
    # ... and with the single-rank run to the fp32 parity tolerance
    np.testing.assert_allclose(r0["s"][:K], one["s"][:K], rtol=1e-5)
    assert abs(float(r0["rel"]) - one["rel"]) <= 1e-4 * one["rel"]
    # U (row slabs) and V span the same dominant spaces: compare projectors
    u2 = np.vstack([r0["u"], r1["u"]])[:, :K]
    u1 = one["u"][:, :K]
    blk = slice(0, 4096)
    np.testing.assert_allclose(u2[blk] @ u2[blk].T, u1[blk] @ u1[blk].T, atol=2e-4)
    v1, v2 = one["v"][:, :K], r0["v"][:, :K]
    np.testing.assert_allclose(v2 @ v2.T, v1 @ v1.T, atol=2e-4)
    # Nystrom: same core spectrum, same approximation (C rows concatenated)
    c2 = np.vstack([r0["c"], r1["c"]])
    np.testing.assert_allclose(np.linalg.eigvalsh(r0["w"]), np.linalg.eigvalsh(one["w"]),
                               rtol=1e-4, atol=1e-6 * np.abs(one["w"]).max())
    app1 = one["c"][:512] @ np.linalg.pinv(one["w"], rcond=1e-10) @ one["c"][:512].T
    app2 = c2[:512] @ np.linalg.pinv(r0["w"], rcond=1e-10) @ c2[:512].T
    assert np.linalg.norm(app2 - app1) <= 1e-3 * np.linalg.norm(app1)


# seeded ragged configurations of the sharded rsvd (the bench's driver):
# odd row counts (uneven slabs), both power paths (sketch space / products),
# q in {0, 1, 3}, s in {1, 8}
SWEEP = [(30001, 1500, 600, 120, 100, 3, 8), (20011, 3000, 900, 40, 30, 1, 1),
         (40003, 1024, 500, 200, 150, 0, 8), (12345, 2222, 333, 70, 60, 2, 8)]


def _run_sweep(comm, rank, world):
    import paper_2605_09755_b200 as skp
    from paper_2605_09755_b200 import datagen, distributed as D
    out = {}
    for ci, (m, n, l, r2, k, q, s) in enumerate(SWEEP):
        row0, rows = D.shard_rows(m, world, rank)
        spec_v = np.exp(-np.arange(1.0, 601.0) / 150.0)
        a = datagen.lowrank_plus_noise_gpu(m, n, spec_v, 1e-7, seed=ci, row0=row0, rows=rows)
        spec = skp.RangeFinderSpec(k=k, l=l, r1=l, r2=r2, q=q, eps=0.5, seed=ci, s=s)
        _, sv, _, rel = D.rsvd_sharded(a, spec, m, comm, with_error=True)
        out[f"s{ci}"] = sv.double().cpu().numpy()
        out[f"rel{ci}"] = np.array(rel)
    return out


def _worker_sweep(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_09755_b200 import distributed as D
        np.savez(os.path.join(out_dir, f"sweep{rank}.npz"), **_run_sweep(D.TorchComm(), rank, world))
    finally:
        dist.destroy_process_group()


def test_two_ranks_sweep_match_one(tmp_path):
    from paper_2605_09755_b200 import _engine
    one = _run_sweep(_engine.LOCAL, 0, 1)
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker_sweep, args=(r, 2, port, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(900)
        assert p.exitcode == 0
    r0, r1 = (dict(np.load(tmp_path / f"sweep{r}.npz")) for r in range(2))
    for ci, (m, n, l, r2, k, q, s) in enumerate(SWEEP):
        np.testing.assert_array_equal(r0[f"s{ci}"], r1[f"s{ci}"])
        np.testing.assert_allclose(r0[f"s{ci}"][:k], one[f"s{ci}"][:k], rtol=1e-5,
                                   err_msg=f"config {SWEEP[ci]}")
        e1, e2 = float(one[f"rel{ci}"]), float(r0[f"rel{ci}"])
        assert abs(e2 - e1) <= 1e-3 * e1, (SWEEP[ci], e1, e2)
