"""Slab-decomposed 3-D PCG over P ranks through libjfftb200.

The whole iteration runs inside the library (csrc/dist.cu): per rank the
fused stencil / FFT / block-solve passes, between them the three exchange
steps of the path -- a halo row of p per side for the stencil, an all-to-all
of the half spectra after the axis-0 transform and back before the last
inverse one, and all-gathers of per-rank partial sums -- with every PCG
scalar on the device (no host synchronisation inside an iteration).  This
module is the host side: communicator set-up, the slab partition and the
reference-shaped ``pcg`` call (solver.py:64-140 semantics and report).

Partition (rank r of P, n1 % P == 0): real space rows [r L1, (r+1) L1) of
axis 1, L1 = n1 / P; k space axis-0 frequency rows
[r n0 / (2P), (r+1) n0 / (2P)) (the last rank also holds the Nyquist row
n0 / 2).

Communicators: ``Comm.nccl_from_torch()`` (one process per GPU; rank 0's
NCCL unique id is broadcast over torch.distributed, NCCL itself is driven by
the library on the solver's stream) or ``Comm.local(P)`` (all P ranks in
this process on one device, for testing the decomposition on one GPU).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .solver import CONVERGED, ITERATION_CAP, SolveReport

KINDS = {"green": N.PC_GREEN, "green-jacobi": N.PC_GREEN_JACOBI}


def slab_rows(n1: int, world: int, rank: int) -> tuple[int, int]:
    """Axis-1 rows [lo, hi) of rank ``rank``'s real-space slab."""
    if n1 % world:
        raise ValueError(f"n1 = {n1} does not split into {world} slabs")
    L1 = n1 // world
    return rank * L1, (rank + 1) * L1


def k0_rows(n0: int, world: int, rank: int) -> tuple[int, int]:
    """Axis-0 frequency rows [lo, hi) of rank ``rank``'s spectral slab."""
    if (n0 // 2) % world:
        raise ValueError(f"n0 / 2 = {n0 // 2} does not split into {world} slabs")
    per = n0 // 2 // world
    return rank * per, (rank + 1) * per + (1 if rank == world - 1 else 0)


def split(field: np.ndarray, world: int, axis: int) -> list[np.ndarray]:
    """Per-rank slabs of a global field along axis ``axis`` (the axis-1 of the
    grid: 1 for a scalar field, 2 for a vector field)."""
    return [np.ascontiguousarray(a) for a in np.split(field, world, axis=axis)]


def join(slabs, axis: int) -> np.ndarray:
    return np.concatenate(list(slabs), axis=axis)


def broadcast_unique_id(make_id, group=None) -> bytes:
    """Rank 0 makes the 128-byte id (``make_id()``), every rank returns it
    (torch.distributed object broadcast; works over gloo and NCCL)."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    N.check(N.load().jfftb_comm_unique_id(buf))
    return buf.raw


class Comm(N._Handle):
    _destroy = "jfftb_comm_destroy"

    def __init__(self, ptr, world: int, rank: int, local: bool, device: int):
        super().__init__(ptr)
        self.world, self.rank, self.local, self.device = world, rank, local, device

    @classmethod
    def local_ranks(cls, world: int, device: int | None = None) -> "Comm":
        dev = N.device_id() if device is None else device
        out = C.c_void_p()
        N.check(N.load().jfftb_comm_create_local(world, dev, C.byref(out)))
        return cls(out, world, 0, True, dev)

    @classmethod
    def nccl(cls, id128: bytes, rank: int, world: int, device: int) -> "Comm":
        out = C.c_void_p()
        N.check(N.load().jfftb_comm_create_nccl(id128, rank, world, device, C.byref(out)))
        return cls(out, world, rank, False, device)

    @classmethod
    def nccl_from_torch(cls, group=None, device: int | None = None) -> "Comm":
        """One rank per process of the initialised torch.distributed group."""
        import torch
        import torch.distributed as dist
        dev = torch.cuda.current_device() if device is None else device
        idb = broadcast_unique_id(unique_id, group)
        return cls.nccl(idb, dist.get_rank(group), dist.get_world_size(group), dev)


@dataclass
class DistInfo:
    world: int
    L1: int
    local_ranks: int
    first_rank: int
    k0lo: int
    kcnt: int
    slab_nodes: int
    loopback: bool


class DistSolver(N._Handle):
    """Operator + Green(-Jacobi) preconditioner + PCG on the slabs of this
    process.  ``rho``: the local density slabs (n0, L1, n2) -- one for an
    NCCL communicator, all P stacked on a new leading axis for the loopback;
    NumPy (host) or a CUDA tensor (device)."""

    _destroy = "jfftb_dist_destroy"

    def __init__(self, comm: Comm, n, lengths, rho, lam: float, mu: float,
                 lam_ref: float | None = None, mu_ref: float | None = None,
                 kind: str = "green-jacobi"):
        if kind not in KINDS:
            raise ValueError(f"distributed solves support {sorted(KINDS)}, not {kind!r}")
        n = tuple(int(k) for k in n)
        lengths = tuple(float(x) for x in lengths)
        lam_ref = lam if lam_ref is None else lam_ref
        mu_ref = mu if mu_ref is None else mu_ref
        where, ptr, self._keep = _pointer(rho)
        out = C.c_void_p()
        N.check(N.load().jfftb_dist_create(comm.ptr, (C.c_int64 * 3)(*n), (C.c_double * 3)(*lengths),
                                           ptr, where, float(lam), float(mu), float(lam_ref),
                                           float(mu_ref), KINDS[kind], C.byref(out)))
        super().__init__(out)
        self._keep = None
        self.comm, self.n, self.lengths, self.kind = comm, n, lengths, kind
        info = (C.c_int64 * 8)()
        N.check(N.load().jfftb_dist_info(self.ptr, info))
        self.info = DistInfo(*[int(v) for v in info[:7]], bool(info[7]))
        L1 = self.info.L1
        self.slab_shape = (3, n[0], L1, n[2])
        self.local_shape = ((comm.world,) if comm.local else ()) + self.slab_shape

    def _out(self, like=None):
        if like is not None and not isinstance(like, np.ndarray):
            import torch
            return torch.empty(self.local_shape, dtype=torch.float64, device=like.device)
        return np.empty(self.local_shape)

    def assemble_rhs(self, eps_bar, device=None):
        eb = np.ascontiguousarray(eps_bar, dtype=np.float64)
        if eb.shape != (6,):
            raise ValueError("macroscopic strain must have shape (6,)")
        out = self._out(device)
        where, ptr, keep = _pointer(out)
        N.check(N.load().jfftb_dist_assemble_rhs(self.ptr, N.dptr(eb), ptr, where))
        del keep
        return out

    def jacobi_inv_sqrt(self):
        out = self._out()
        N.check(N.load().jfftb_dist_jacobi_export(self.ptr, N.vptr(out), N.HOST))
        return out

    def pcg(self, rhs, eta: float = 1e-6, max_iter: int = 999, x_out=None) -> SolveReport:
        """solver.py:64-140 on the slabs; the report's solution holds this
        process's slabs (``local_shape``)."""
        where, rptr, rkeep = _pointer(rhs)
        if x_out is None:
            x_out = self._out(rhs if where == N.DEVICE else None)
        xwhere, xptr, xkeep = _pointer(x_out)
        if xwhere != where or xkeep is not x_out:
            raise ValueError("x_out must be a contiguous float64 array in the rhs's memory space")
        hist = np.empty(max_iter + 1)
        it, term, wall = C.c_int(), C.c_int(), C.c_double()
        N.check(N.load().jfftb_dist_pcg(self.ptr, rptr, where, float(eta), int(max_iter), xptr,
                                        N.dptr(hist), C.byref(it), C.byref(term), C.byref(wall)),
                N.SolverAbortError)
        k = it.value
        return SolveReport(k, hist[:k + 1].tolist(),
                           CONVERGED if term.value == 0 else ITERATION_CAP, wall.value, x_out)


def _pointer(a):
    """(where, void pointer, keep-alive) of a NumPy array or CUDA tensor."""
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        return N.HOST, N.vptr(a), a
    import torch
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise ValueError("device arrays must be contiguous float64 tensors")
        torch.cuda.current_stream(a.device).synchronize()
        return N.DEVICE, C.c_void_p(a.data_ptr()), a
    raise TypeError(f"unsupported array type {type(a)}")
