"""The multi-GPU host logic (paper_2508_02613_b200.slab: slab partition, halo
exchange, all-to-all FFT transposes, rank-ordered reductions) on CPU with the
gloo backend at world size 2 and 4, against the single-process oracle."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(n):
    rng = np.random.default_rng(5)
    rho = rng.uniform(0.05, 2.0, n)
    return rho, np.array([1.0, -0.5, 0.3, 0.2, -0.1, 0.4])


def _worker(rank, world, port, n, kind, out_q):
    sys.path.insert(0, REPO)
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import jfft_oracle as X
        from paper_2508_02613_b200.slab import SlabLayout, SlabPCG
        from slab_cpu_backend import CpuBackend
        lengths = (1.0, 1.0, 1.0)
        rho, eb = _problem(n)
        lay = SlabLayout(n, lengths, world, rank)
        sl = slice(lay.plane0, lay.plane0 + lay.L0)
        c = X.isotropic_stiffness(3, 2.0 / 3.0, 0.5)
        h = X.pixel_size(n, lengths)
        rhs = X.assemble_rhs(rho, c, h, eb)
        solver = SlabPCG(lay, CpuBackend(), torch.from_numpy(rho[sl].copy()), 2.0 / 3.0, 0.5,
                         kind=kind)
        f_local = solver.assemble_rhs(eb).numpy()
        assert np.abs(f_local - rhs[:, sl]).max() <= 1e-13 * np.abs(rhs).max()
        it, hist, term, x, _ = solver.solve(torch.from_numpy(rhs[:, sl].copy()), eta=1e-10)
        dinv = solver.dinv.numpy() if solver.dinv is not None else None
        out_q.put((rank, it, hist, term, x.numpy(), dinv))
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


@pytest.mark.parametrize("world,kind", [(2, "green-jacobi"), (2, "green"), (4, "green-jacobi"),
                                        (2, "jacobi")])
def test_slab_pcg_matches_single_process(world, kind):
    sys.path.insert(0, REPO)
    from oracle import jfft_oracle as X
    n = (8, 8, 8)
    rho, eb = _problem(n)
    c = X.isotropic_stiffness(3, 2.0 / 3.0, 0.5)
    h = X.pixel_size(n, (1.0, 1.0, 1.0))
    blocks = X.assemble_green(n, (1.0, 1.0, 1.0), c)
    inv = X.assemble_jacobi(rho, c, h)
    f = X.assemble_rhs(rho, c, h, eb)
    it, hist, term, x = X.pcg(rho, c, h, f, kind, blocks, inv, eta=1e-10)
    res = _run(world, n, kind)
    L0 = n[0] // world
    xs = np.concatenate([r[4] for r in res], axis=1)
    for rank, it_r, hist_r, term_r, _, dinv in res:
        assert it_r == it and term_r == term
        assert np.abs(np.array(hist_r) - hist).max() <= 1e-12 * hist[0]
        if dinv is not None:
            assert np.abs(dinv - inv[:, rank * L0:(rank + 1) * L0]).max() <= 1e-14 * inv.max()
    # all ranks agree bitwise on the recurrence scalars
    assert all(r[2] == res[0][2] for r in res)
    assert np.abs(xs - x).max() <= 1e-9 * np.abs(x).max()
