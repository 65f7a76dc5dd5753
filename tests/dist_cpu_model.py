"""CPU model of the library's distributed PCG (csrc/dist.cu) for the
multi-process gloo tests -- TEST INFRASTRUCTURE ONLY.

It runs, per rank, exactly the decomposition and exchange schedule of
dist.cu with NumPy kernels from the oracle:

* real space: axis-1 rows [r L1, (r+1) L1) of every field; the stencil reads
  a halo-extended slab (rows r L1 - 1 .. (r+1) L1) filled by exchanging one
  row of p with each neighbour (posting order: last row up, first row down,
  then receive from below and above -- the order dist.cu uses so NCCL's
  per-pair matching pairs them right, also at world 2);
* pass A: axis-0 real-to-complex transform of r' and s = D^-1/2 r' on the
  local columns; all-to-all of the axis-0 frequency rows (rank q gets rows
  paralleling dist.py.k0_rows), kept as one segment per source rank;
* passes B / C: axis-1 and axis-2 transforms of the k0-slab, the Green block
  solve with G(k) taken from the oracle's numpy-layout blocks (G(-k) =
  conj G(k) for the other half), Parseval sums weighted 1 on k0 in {0, n0/2}
  and 2 elsewhere; inverse transforms; all-to-all back; axis-0 C2R (pass I);
* scalars: each rank's partial sums are all-gathered and summed in rank
  order on every rank.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from oracle import jfft_oracle as X


def k0_rows(n0, world, rank):
    per = n0 // 2 // world
    return rank * per, (rank + 1) * per + (1 if rank == world - 1 else 0)


class RankModel:
    def __init__(self, n, lengths, rho_slab, lam, mu, kind, world, rank):
        self.n, self.world, self.rank, self.kind = tuple(n), world, rank, kind
        n0, n1, n2 = self.n
        self.L1 = n1 // world
        self.c = X.isotropic_stiffness(3, lam, mu)
        self.h = X.pixel_size(self.n, lengths)
        self.rho_ext = self.halo(rho_slab[None])[0]
        self.k0lo, self.k0hi = k0_rows(n0, world, rank)
        full = X.assemble_green(self.n, lengths, self.c)  # (n0, n1, n2/2+1, 3, 3)
        k0 = np.arange(self.k0lo, self.k0hi)
        k1 = np.arange(n1)
        k2 = np.arange(n2)
        # G(k0, k1, k2) for every k2: the stored half has k2 <= n2/2
        lo = k2 <= n2 // 2
        G = np.empty((len(k0), n1, n2, 3, 3), dtype=complex)
        G[:, :, lo] = full[k0][:, :, k2[lo]]
        m0, m1, m2 = (-k0) % n0, (-k1) % n1, (-k2[~lo]) % n2
        G[:, :, ~lo] = np.conj(full[m0][:, m1][:, :, m2])
        self.G = G
        self.w = np.where((k0 == 0) | (2 * k0 == n0), 1.0, 2.0)[:, None, None]
        self.dinv = None
        if kind == "green-jacobi":
            self.dinv = self.jacobi()

    # ---- exchanges ----------------------------------------------------------
    def halo(self, f):
        """(c, n0, L1, n2) -> (c, n0, L1 + 2, n2) with the neighbours' rows."""
        lo, hi = (self.rank - 1) % self.world, (self.rank + 1) % self.world
        first = np.ascontiguousarray(f[:, :, 0])
        last = np.ascontiguousarray(f[:, :, -1])
        if self.world == 1:
            from_lo, from_hi = last, first
        else:
            from_lo, from_hi = np.empty_like(first), np.empty_like(first)
            t = [torch.from_numpy(a) for a in (last, first, from_lo, from_hi)]
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, t[0], hi),
                                           dist.P2POp(dist.isend, t[1], lo),
                                           dist.P2POp(dist.irecv, t[2], lo),
                                           dist.P2POp(dist.irecv, t[3], hi)])
            for r in reqs:
                r.wait()
        return np.concatenate([from_lo[:, :, None], f, from_hi[:, :, None]], axis=2)

    def allsum(self, vals):
        t = torch.tensor(list(vals), dtype=torch.float64)
        if self.world == 1:
            return t.numpy()
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t)
        acc = out[0].clone()
        for o in out[1:]:
            acc += o
        return acc.numpy()

    def alltoall_fwd(self, spec):
        """(F, n0/2+1, L1, n2) local columns -> (F, kcnt, n1, n2) k0-slab."""
        W = self.world
        chunks = [np.ascontiguousarray(spec[:, slice(*k0_rows(self.n[0], W, q))]) for q in range(W)]
        recv = self._alltoall(chunks, lambda q: (spec.shape[0], self.k0hi - self.k0lo,
                                                 self.L1, self.n[2]))
        return np.concatenate(recv, axis=2)  # segments of L1 rows in rank order

    def alltoall_bwd(self, z):
        """(F, kcnt, n1, n2) -> (F, n0/2+1, L1, n2)."""
        W = self.world
        chunks = [np.ascontiguousarray(z[:, :, q * self.L1:(q + 1) * self.L1]) for q in range(W)]
        recv = self._alltoall(chunks, lambda q: (z.shape[0],) + (
            k0_rows(self.n[0], W, q)[1] - k0_rows(self.n[0], W, q)[0], self.L1, self.n[2]))
        return np.concatenate(recv, axis=1)

    def _alltoall(self, chunks, shape_of):
        if self.world == 1:
            return chunks
        recv = [np.empty(shape_of(q), dtype=complex) for q in range(self.world)]
        ops = []
        for q in range(self.world):
            if q == self.rank:
                recv[q][...] = chunks[q]
                continue
            ops.append(dist.P2POp(dist.isend, torch.view_as_real(torch.from_numpy(chunks[q])), q))
            ops.append(dist.P2POp(dist.irecv, torch.view_as_real(torch.from_numpy(recv[q])), q))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        return recv

    # ---- local kernels ------------------------------------------------------
    def K(self, p):
        return X.apply_K(self.rho_ext, self.c, self.h, self.halo(p))[:, :, 1:-1]

    def rhs(self, eb):
        return X.assemble_rhs(self.rho_ext, self.c, self.h, np.asarray(eb, float))[:, :, 1:-1]

    def jacobi(self):
        n0, n1, n2 = self.n
        diag = np.empty((3, n0, self.L1, n2))
        rows = np.arange(self.rank * self.L1 - 1, (self.rank + 1) * self.L1 + 1) % n1
        for a in range(3):
            for o0 in (0, 1):
                for o1 in (0, 1):
                    for o2 in (0, 1):
                        comb = np.zeros((3, n0, self.L1 + 2, n2))
                        m = ((np.arange(n0)[:, None, None] % 2 == o0) & (rows[None, :, None] % 2 == o1)
                             & (np.arange(n2)[None, None, :] % 2 == o2))
                        comb[a][m] = 1.0
                        resp = X.apply_K(self.rho_ext, self.c, self.h, comb)[:, :, 1:-1]
                        sel = m[:, 1:-1]
                        diag[a][sel] = resp[a][sel]
        if np.any(diag < 0) or not np.all(np.isfinite(diag)):
            raise ValueError("probed diagonal has negative or non-finite entries")
        diag[diag == 0.0] = 1.0
        return 1.0 / np.sqrt(diag)

    def precond(self, r):
        """(z, <r, G r>, <r, z>) -- the fused passes A..I of one iteration."""
        n0 = self.n[0]
        Nt = float(np.prod(self.n))
        gj = self.kind == "green-jacobi"
        fields = [r, self.dinv * r] if gj else [r]
        spec = np.fft.rfft(np.concatenate(fields), axis=1)           # pass A (axis 0)
        sl = self.alltoall_fwd(spec)                                  # -> k0-slab
        sl = np.fft.fft(np.fft.fft(sl, axis=2), axis=3)               # passes B, C
        rh = sl[:3]
        q0 = np.einsum("kyzab,bkyz->akyz", self.G, rh)
        quad_r = float(np.sum(self.w * np.real(np.conj(rh) * q0).sum(axis=0))) / Nt
        src = sl[3:] if gj else rh
        zh = np.einsum("kyzab,bkyz->akyz", self.G, src) / Nt
        quad_s = float(np.sum(self.w * np.real(np.conj(src) * zh).sum(axis=0)))
        zh = np.fft.ifft(np.fft.ifft(zh, axis=3), axis=2) * (self.n[1] * self.n[2])
        back = self.alltoall_bwd(zh)                                  # -> local columns
        z = np.fft.irfft(back, n=n0, axis=1) * n0                     # pass I (unnormalised)
        if gj:
            z = self.dinv * z
        return z, quad_r, quad_s

    def pcg(self, rhs, eta, max_iter):
        x = np.zeros_like(rhs)
        r = rhs.copy()
        z, qr, qs = self.precond(r)
        g2, rz = self.allsum([qr, qs])
        hist = [g2]
        if g2 <= eta:
            return 0, hist, "converged", self.sub_mean(x)
        p = z.copy()
        it, term = 0, "iteration-cap"
        while it < max_iter:
            kp = self.K(p)
            curv = self.allsum([float(np.sum(p * kp))])[0]
            if not curv > 0:
                raise RuntimeError("non-positive curvature")
            alpha = rz / curv
            x += alpha * p
            r -= alpha * kp
            it += 1
            z, qr, qs = self.precond(r)
            g2, rz_new = self.allsum([qr, qs])
            hist.append(g2)
            if g2 <= eta:
                term = "converged"
                break
            p = (rz_new / rz) * p + z
            rz = rz_new
        return it, hist, term, self.sub_mean(x)

    def sub_mean(self, x):
        s = self.allsum(x.sum(axis=(1, 2, 3)))
        return x - (s / float(np.prod(self.n)))[:, None, None, None]
