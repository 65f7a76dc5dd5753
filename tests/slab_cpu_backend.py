"""CPU backend for paper_2508_02613_b200.slab (multi-process gloo tests only):
the same local operations as DeviceBackend, computed with the NumPy oracle."""

import numpy as np
import torch

from oracle import jfft_oracle as X


class CpuBackend:
    device = torch.device("cpu")

    def setup(self, lay, rho_ext, lam, mu):
        n0, n1, n2 = lay.n
        self.lay = lay
        self.c = X.isotropic_stiffness(3, lam, mu)
        self.h = X.pixel_size(lay.n, lay.lengths)
        self.rho_ext = rho_ext.numpy().copy()
        full = X.assemble_green(lay.n, lay.lengths, self.c)      # (n0, n1, nh, 3, 3)
        lo = lay.rank * lay.L1
        self.blocks = full[:, lo:lo + lay.L1]
        nh = lay.nh
        k2 = np.arange(nh)
        self.w = np.where((k2 == 0) | (2 * k2 == n2), 1.0, 2.0)

    def stencil(self, p_ext, out_ext):
        # periodic over the extended slab: the interior planes see only their
        # true neighbours (halo planes), so they are exact
        out_ext.copy_(torch.from_numpy(X.apply_K(self.rho_ext, self.c, self.h, p_ext.numpy())))

    def rhs(self, eps_bar, out_ext):
        out_ext.copy_(torch.from_numpy(X.assemble_rhs(self.rho_ext, self.c, self.h,
                                                      np.asarray(eps_bar, dtype=float))))

    def rfft2(self, u):
        return torch.fft.rfft2(u, dim=(-2, -1))

    def irfft2(self, a, s):
        return torch.fft.irfft2(a, s=tuple(s), dim=(-2, -1), norm="forward")

    def fft_axis0(self, t, inverse):
        return torch.fft.ifft(t, dim=1, norm="forward") if inverse else torch.fft.fft(t, dim=1)

    def _quad(self, s):
        z = np.einsum("xyzab,bxyz->axyz", self.blocks, s)
        q = (np.conj(s) * z).real.sum(axis=0)
        return z, float((q * self.w[None, None, :]).sum()) / self.lay.N

    def green_apply(self, kind, spec):
        a = spec.numpy()  # shares memory with the tensor
        if kind == "green-jacobi":
            _, qr = self._quad(a[:3])
            z, qs = self._quad(a[3:])
            a[3:] = z / self.lay.N
            return qr, qs
        z, q = self._quad(a[:3])
        a[:3] = z / self.lay.N
        return q, q

    def dot(self, a, b):
        return float(np.vdot(a.numpy(), b.numpy()))
