"""Multi-rank path of the distributed solver on CPU: the library's
decomposition and exchange schedule (csrc/dist.cu; modelled per rank in
tests/dist_cpu_model.py with the oracle's kernels) over the gloo backend at
world size 1, 2 and 4, against the single-process oracle; plus the host
helpers of paper_2508_02613_b200.dist (partition, unique-id broadcast)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
N3 = (8, 16, 8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(n):
    rng = np.random.default_rng(5)
    return rng.uniform(0.05, 2.0, n), np.array([1.0, -0.5, 0.3, 0.2, -0.1, 0.4])


def _worker(rank, world, port, n, kind, out_q):
    sys.path.insert(0, REPO)
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_cpu_model import RankModel
        from paper_2508_02613_b200 import dist as Dm
        # the unique-id broadcast of Comm.nccl_from_torch (any backend)
        idb = Dm.broadcast_unique_id(lambda: bytes(range(128)))
        assert idb == bytes(range(128))
        rho, eb = _problem(n)
        lo, hi = Dm.slab_rows(n[1], world, rank)
        m = RankModel(n, (1.0, 1.0, 1.0), rho[:, lo:hi].copy(), 2.0 / 3.0, 0.5, kind, world, rank)
        f = m.rhs(eb)
        it, hist, term, x = m.pcg(f, 1e-10, 999)
        out_q.put((rank, it, hist, term, x, f, m.dinv))
    finally:
        dist.destroy_process_group()


def _run(world, n, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(res, key=lambda t: t[0])


@pytest.mark.parametrize("world,kind", [(1, "green-jacobi"), (2, "green-jacobi"), (2, "green"),
                                        (4, "green-jacobi")])
def test_dist_model_matches_single_process(world, kind):
    sys.path.insert(0, REPO)
    from oracle import jfft_oracle as X
    n = N3
    rho, eb = _problem(n)
    c = X.isotropic_stiffness(3, 2.0 / 3.0, 0.5)
    h = X.pixel_size(n, (1.0, 1.0, 1.0))
    blocks = X.assemble_green(n, (1.0, 1.0, 1.0), c)
    inv = X.assemble_jacobi(rho, c, h)
    f = X.assemble_rhs(rho, c, h, eb)
    it, hist, term, x = X.pcg(rho, c, h, f, kind, blocks, inv, eta=1e-10)
    res = _run(world, n, kind)
    L1 = n[1] // world
    xs = np.concatenate([r[4] for r in res], axis=2)
    fs = np.concatenate([r[5] for r in res], axis=2)
    assert np.abs(fs - f).max() <= 1e-13 * np.abs(f).max()
    for rank, it_r, hist_r, term_r, _, _, dinv in res:
        assert it_r == it and term_r == term
        assert np.abs(np.array(hist_r) - hist).max() <= 1e-12 * hist[0]
        if dinv is not None:
            assert np.abs(dinv - inv[:, :, rank * L1:(rank + 1) * L1]).max() <= 1e-14 * inv.max()
    # all ranks agree bitwise on the recurrence scalars
    assert all(r[2] == res[0][2] for r in res)
    assert np.abs(xs - x).max() <= 1e-9 * np.abs(x).max()


def test_partition_helpers():
    sys.path.insert(0, REPO)
    from paper_2508_02613_b200 import dist as Dm
    assert [Dm.slab_rows(1024, 8, r) for r in (0, 7)] == [(0, 128), (896, 1024)]
    rows = [Dm.k0_rows(1024, 8, r) for r in range(8)]
    assert rows[0] == (0, 64) and rows[-1] == (448, 513)
    assert sum(hi - lo for lo, hi in rows) == 513
    f = np.arange(2 * 4 * 8 * 2.0).reshape(2, 4, 8, 2)
    assert np.array_equal(Dm.join(Dm.split(f, 4, axis=2), axis=2), f)
    with pytest.raises(ValueError):
        Dm.slab_rows(100, 8, 0)
    with pytest.raises(ValueError):
        Dm.k0_rows(24, 8, 0)
