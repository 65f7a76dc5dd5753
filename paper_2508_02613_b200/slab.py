"""Slab-decomposed 3-D PCG over P ranks.

One process per GPU; rank r owns node planes [r L0, (r+1) L0) of axis 0
(L0 = n0 / P) of every vector field.  Per iteration the path has three real
exchange steps, each a collective here:

* halo exchange of one p-plane per side for the stencil (send/recv pairs);
* an all-to-all transpose inside each distributed FFT: the local 2-D
  transform (axes 1, 2) of the slab is redistributed so that every rank holds
  all of axis 0 for an axis-1 frequency slab [r L1, (r+1) L1), L1 = n1 / P,
  where the axis-0 transform and the Green block solve run locally;
* all-gather of per-rank partial dot products, summed in rank order on every
  rank, so alpha / beta / the termination value are bitwise identical across
  ranks and independent of reduction-tree shape.

The recurrence is solver.py:64-140 exactly (absolute <r, G r> <= eta, history,
cap, abort on NaN / curvature <= 0, final mean subtraction).

Local compute goes through a backend: ``DeviceBackend`` (libjfftb200 stencil on
a halo-extended slab, libjfftb200 block solve on the frequency slab, cuFFT via
torch.fft for the local transforms, NCCL) or, in the multi-process CPU tests
only, ``tests/slab_cpu_backend.py`` (NumPy oracle kernels, gloo).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import torch
import torch.distributed as dist

CONVERGED = "converged"
ITERATION_CAP = "iteration-cap"


class SolverAbortError(RuntimeError):
    pass


@dataclass(frozen=True)
class SlabLayout:
    n: tuple          # global (n0, n1, n2)
    lengths: tuple
    world: int
    rank: int

    def __post_init__(self):
        n0, n1, _ = self.n
        if n0 % self.world or n1 % self.world:
            raise ValueError(f"grid {self.n} does not split into {self.world} slabs")

    @property
    def L0(self):
        return self.n[0] // self.world

    @property
    def L1(self):
        return self.n[1] // self.world

    @property
    def plane0(self):
        return self.rank * self.L0

    @property
    def N(self):
        return self.n[0] * self.n[1] * self.n[2]

    @property
    def nh(self):
        return self.n[2] // 2 + 1


class SlabComm:
    """The three exchange patterns over torch.distributed (NCCL or gloo)."""

    def __init__(self, layout: SlabLayout, group=None):
        self.lay = layout
        self.group = group

    def _p2p(self, ops):
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def halo(self, ext: torch.Tensor) -> None:
        """ext: (c, L0 + 2, n1, n2); fill planes 0 and L0 + 1 from the
        neighbouring slabs (periodic)."""
        lay = self.lay
        L0 = lay.L0
        if lay.world == 1:
            ext[:, 0].copy_(ext[:, L0])
            ext[:, L0 + 1].copy_(ext[:, 1])
            return
        prev, nxt = (lay.rank - 1) % lay.world, (lay.rank + 1) % lay.world
        first = ext[:, 1].contiguous()
        last = ext[:, L0].contiguous()
        from_prev = torch.empty_like(first)
        from_next = torch.empty_like(first)
        # NCCL ignores tags and matches the sends and receives between one
        # pair of ranks in posting order; at world 2 (prev == nxt) the order
        # below pairs last -> from_prev and first -> from_next on both ranks
        ops = [dist.P2POp(dist.isend, last, nxt, self.group, tag=2),
               dist.P2POp(dist.isend, first, prev, self.group, tag=1),
               dist.P2POp(dist.irecv, from_prev, prev, self.group, tag=2),
               dist.P2POp(dist.irecv, from_next, nxt, self.group, tag=1)]
        self._p2p(ops)
        ext[:, 0].copy_(from_prev)
        ext[:, L0 + 1].copy_(from_next)

    def all_to_all(self, send: torch.Tensor) -> torch.Tensor:
        """send: (P, ...) contiguous, chunk j goes to rank j; returns (P, ...)
        with chunk i received from rank i."""
        if self.lay.world == 1:
            return send
        real = torch.view_as_real(send) if send.is_complex() else send
        recv = torch.empty_like(real)
        dist.all_to_all_single(recv, real.contiguous(), group=self.group)
        return torch.view_as_complex(recv) if send.is_complex() else recv

    def allsum(self, values) -> list:
        """Deterministic sum over ranks of a few scalars (rank order)."""
        t = torch.tensor(list(values), dtype=torch.float64)
        if self.lay.world == 1:
            return [float(v) for v in t]
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = t.to(dev)
        out = [torch.empty_like(t) for _ in range(self.lay.world)]
        dist.all_gather(out, t, group=self.group)
        acc = out[0].clone()
        for o in out[1:]:
            acc += o
        return [float(v) for v in acc.cpu()]


class SlabPCG:
    """Distributed PCG for one operator / preconditioner on a slab layout.

    rho_local: (L0, n1, n2) density planes of this rank (torch tensor on the
    backend's device); kind: "none" | "green" | "jacobi" | "green-jacobi".
    """

    def __init__(self, layout: SlabLayout, backend, rho_local: torch.Tensor, lam: float,
                 mu: float, kind: str = "green-jacobi", comm: SlabComm | None = None):
        self.lay, self.be, self.kind = layout, backend, kind
        self.comm = comm or SlabComm(layout)
        L0, (n0, n1, n2) = layout.L0, layout.n
        dev = backend.device
        rho_ext = torch.empty((1, L0 + 2, n1, n2), dtype=torch.float64, device=dev)
        rho_ext[0, 1:L0 + 1].copy_(rho_local)
        self.comm.halo(rho_ext)
        backend.setup(layout, rho_ext[0], lam, mu)
        self.p_ext = torch.zeros((3, L0 + 2, n1, n2), dtype=torch.float64, device=dev)
        self.kp_ext = torch.zeros_like(self.p_ext)
        self.dinv = None
        if kind in ("jacobi", "green-jacobi"):
            self.dinv = self._jacobi()

    # -- pieces ----------------------------------------------------------------
    def assemble_rhs(self, eps_bar) -> torch.Tensor:
        """operators.py:61-76 on the slab: f = -B^T W rho C E (local planes)."""
        L0 = self.lay.L0
        self.be.rhs(eps_bar, self.kp_ext)
        return self.kp_ext[:, 1:L0 + 1].clone()

    def apply_K(self, p: torch.Tensor) -> torch.Tensor:
        """K p for a local (3, L0, n1, n2) field (halo exchange + local stencil)."""
        L0 = self.lay.L0
        self.p_ext[:, 1:L0 + 1].copy_(p)
        self.comm.halo(self.p_ext)
        self.be.stencil(self.p_ext, self.kp_ext)
        return self.kp_ext[:, 1:L0 + 1]

    def _jacobi(self) -> torch.Tensor:
        """preconditioners.py:97-119 on the slab: d * 2^d comb probes (parity
        of the GLOBAL plane index along axis 0)."""
        lay = self.lay
        L0, (n0, n1, n2) = lay.L0, lay.n
        if any(k % 2 for k in lay.n):
            raise ValueError("diagonal probing requires an even node count")
        dev = self.be.device
        i0 = (torch.arange(L0, device=dev) + lay.plane0) % 2
        i1 = torch.arange(n1, device=dev) % 2
        i2 = torch.arange(n2, device=dev) % 2
        diag = torch.empty((3, L0, n1, n2), dtype=torch.float64, device=dev)
        for alpha in range(3):
            for o0 in (0, 1):
                for o1 in (0, 1):
                    for o2 in (0, 1):
                        mask = ((i0 == o0)[:, None, None] & (i1 == o1)[None, :, None]
                                & (i2 == o2)[None, None, :])
                        comb = torch.zeros((3, L0, n1, n2), dtype=torch.float64, device=dev)
                        comb[alpha][mask] = 1.0
                        resp = self.apply_K(comb)
                        diag[alpha][mask] = resp[alpha][mask]
        bad = float(((diag < 0) | ~torch.isfinite(diag)).any())
        if self.comm.allsum([bad])[0] > 0:
            raise ValueError("probed diagonal has negative or non-finite entries")
        diag[diag == 0.0] = 1.0
        return 1.0 / torch.sqrt(diag)

    def fft_forward(self, u: torch.Tensor) -> torch.Tensor:
        """(c, L0, n1, n2) real -> (c, n0, L1, n2/2+1) complex, axis-1 slab."""
        lay = self.lay
        c, L0, P, L1, nh = u.shape[0], lay.L0, lay.world, lay.L1, lay.nh
        a = self.be.rfft2(u)                                         # (c, L0, n1, nh)
        send = a.reshape(c, L0, P, L1, nh).permute(2, 0, 1, 3, 4).contiguous()
        recv = self.comm.all_to_all(send)                            # (P, c, L0, L1, nh)
        t = recv.permute(1, 0, 2, 3, 4).reshape(c, lay.n[0], L1, nh)
        # the block solve works in place on the (c, n0, L1, nh) C-order layout
        return self.be.fft_axis0(t, inverse=False).contiguous()

    def fft_inverse(self, spec: torch.Tensor) -> torch.Tensor:
        """Inverse of fft_forward, unnormalised (1/N is in the block solve)."""
        lay = self.lay
        c, L0, P, L1, nh = spec.shape[0], lay.L0, lay.world, lay.L1, lay.nh
        t = self.be.fft_axis0(spec, inverse=True)                    # (c, n0, L1, nh)
        send = t.reshape(c, P, L0, L1, nh).permute(1, 0, 2, 3, 4).contiguous()
        recv = self.comm.all_to_all(send)                            # (P, c, L0, L1, nh)
        a = recv.permute(1, 2, 0, 3, 4).reshape(c, L0, lay.n[1], nh)
        return self.be.irfft2(a, lay.n[1:])

    def precondition(self, r: torch.Tensor):
        """z = M r, plus the slab sums of <r, G r> and <r, z> (solver.py:124-132)."""
        kind = self.kind
        if kind == "green-jacobi":
            s = self.dinv * r
            spec = torch.cat([self.fft_forward(r), self.fft_forward(s)], dim=0)
            qr, qs = self.be.green_apply("green-jacobi", spec)
            z = self.dinv * self.fft_inverse(spec[3:])
            return z, qr, qs
        spec = self.fft_forward(r)
        qr, _ = self.be.green_apply("green", spec)
        if kind == "green":
            return self.fft_inverse(spec), qr, qr
        z = r.clone() if kind == "none" else self.dinv * (self.dinv * r)
        return z, qr, self.be.dot(r, z)

    # -- the recurrence (solver.py:64-140) ------------------------------------
    def solve(self, rhs: torch.Tensor, eta: float = 1e-6, max_iter: int = 999):
        start = time.perf_counter()
        comm = self.comm

        def checked(v, what):
            if not math.isfinite(v):
                raise SolverAbortError(f"{what} became non-finite in PCG")
            return v

        x = torch.zeros_like(rhs)
        r = rhs.clone()
        z, qr, qz = self.precondition(r)
        g2, rz = comm.allsum([qr, qz])
        g2 = checked(g2, "residual Green norm")
        hist = [g2]
        if g2 <= eta:
            return 0, hist, CONVERGED, x, time.perf_counter() - start
        rz = checked(rz, "preconditioned residual product")
        p = z.clone()
        it, term = 0, ITERATION_CAP
        while it < max_iter:
            kp = self.apply_K(p)
            curv = checked(comm.allsum([self.be.dot(p, kp)])[0], "search-direction curvature")
            if curv <= 0.0:
                raise SolverAbortError(f"non-positive curvature {curv:.3e} in PCG")
            alpha = rz / curv
            x.add_(p, alpha=alpha)
            r.sub_(kp, alpha=alpha)
            it += 1
            z, qr, qz = self.precondition(r)
            g2, rz_new = comm.allsum([qr, qz])
            g2 = checked(g2, "residual Green norm")
            hist.append(g2)
            if g2 <= eta:
                term = CONVERGED
                break
            rz_new = checked(rz_new, "preconditioned residual product")
            beta = rz_new / rz
            p.mul_(beta).add_(z)
            rz = rz_new
        sums = comm.allsum([float(x[c].sum()) for c in range(3)])
        for c in range(3):
            x[c] -= sums[c] / self.lay.N
        return it, hist, term, x, time.perf_counter() - start


class DeviceBackend:
    """libjfftb200 kernels on this rank's GPU (cuFFT via torch.fft for the
    local 2-D and axis-0 transforms)."""

    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)

    def setup(self, lay: SlabLayout, rho_ext: torch.Tensor, lam: float, mu: float):
        from . import _native as N
        n0, n1, n2 = lay.n
        L0 = lay.L0
        l0 = lay.lengths[0] * (L0 + 2) / n0  # same pixel size on the extended slab
        self._N = N
        self.grid_ext = N.GridHandle(3, (L0 + 2, n1, n2), (l0, lay.lengths[1], lay.lengths[2]),
                                     device=self.device.index)
        self.grid_ext.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        self.rho_ext = rho_ext.contiguous()
        self.op_ext = N.OpHandle(self.grid_ext, self.rho_ext.data_ptr(), lam, mu, where=N.DEVICE)
        self.grid_full = N.GridHandle(3, lay.n, lay.lengths, device=self.device.index)
        self.grid_full.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        self.green = N.GreenSlabHandle(self.grid_full, lam, mu, lay.rank * lay.L1, lay.L1)

    def stencil(self, p_ext: torch.Tensor, out_ext: torch.Tensor):
        N = self._N
        N.check(N.load().jfftb_apply_system(self.op_ext.ptr, p_ext.data_ptr(), out_ext.data_ptr(),
                                            N.DEVICE))

    def rhs(self, eps_bar, out_ext: torch.Tensor):
        import numpy as np
        N = self._N
        e = np.ascontiguousarray(eps_bar, dtype=np.float64)
        N.check(N.load().jfftb_assemble_rhs(self.op_ext.ptr, N.dptr(e), out_ext.data_ptr(),
                                            N.DEVICE))

    def rfft2(self, u):
        return torch.fft.rfft2(u, dim=(-2, -1))

    def irfft2(self, a, s):
        return torch.fft.irfft2(a, s=tuple(s), dim=(-2, -1), norm="forward")

    def fft_axis0(self, t, inverse):
        return torch.fft.ifft(t, dim=1, norm="forward") if inverse else torch.fft.fft(t, dim=1)

    def green_apply(self, kind, spec):
        N = self._N
        if not spec.is_contiguous():
            raise ValueError("the slab block solve needs a C-contiguous spectrum")
        qr, qs = self.green.apply(N.KIND_CODES[kind], spec.data_ptr())
        return qr, qs

    def dot(self, a, b) -> float:
        return float(torch.dot(a.reshape(-1), b.reshape(-1)))
