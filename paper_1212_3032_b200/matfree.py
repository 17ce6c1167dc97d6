"""Matrix-free system operator (north-star item 2).

``MatrixFreeOperator(assembler, omega, bcs)`` is a callable ``v -> A v``
for the reference's operator seam ``gmres(apply_a=callable)``
(linsolve.py:73-77).  Each application recomputes every element pair on
the GPU (``ewb_matfree_apply``) with the dense assembler's quadrature
ladder, so the (N,N) matrix is never stored — the path for meshes whose
dense operator exceeds HBM (BASELINE cfg5: 245,760 DOF, 966 GB dense).

The column mixing follows ``apply_bcs`` (assembly.py:293-296):
    A v = T (mask_N v) - U (mask_D v),   b = U (mask_N p) - T (mask_D p)
and ``apply_multi`` applies A to any number of vectors, up to 5 per pass
over the element pairs (the SEM product Y = A X plus b share one
evaluation of the kernels for K <= 4).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .assembly import DIRICHLET, Assembler, BoundaryConditionSet


def _torch():
    import torch

    return torch


class MatrixFreeOperator:
    MAX_K = 5

    def __init__(self, assembler: Assembler, omega: complex,
                 bcs: BoundaryConditionSet | None = None):
        torch = _torch()
        self.asm = assembler
        self.omega = complex(omega)
        if self.omega == 0:
            raise ValueError("omega == 0 takes the static (dense) path")
        n = assembler.n
        self.n = n
        kinds = (np.zeros(n, dtype=np.uint8) if bcs is None
                 else np.ascontiguousarray(bcs.flat_kind(), dtype=np.uint8))
        self.kinds = kinds
        self.kinds_dev = torch.from_numpy(kinds).cuda()
        dmask = torch.from_numpy(kinds == DIRICHLET).cuda()
        self.all_neumann = not bool((kinds == DIRICHLET).any())
        self._mask_d = dmask
        self._ws = None
        self.pinv = None
        self.applications = 0

    def _workspace(self, K):
        torch = _torch()
        need = int(_lib.load().ewb_matfree_workspace_bytes(self.asm.ctx, K))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device="cuda")
        return self._ws

    # y_k = T vt_k + U vu_k, passes of up to MAX_K vectors
    def _apply_tu(self, vt, vu, want_pinv: bool = False, masks=None):
        torch = _torch()
        K = int(vt.shape[0])
        if K < 1:
            raise ValueError("no vectors to apply")
        if K > self.MAX_K:
            parts = [self._apply_tu(vt[c:c + self.MAX_K],
                                    vu[c:c + self.MAX_K] if vu is not None else None,
                                    want_pinv and c == 0)
                     for c in range(0, K, self.MAX_K)]
            return torch.cat(parts)
        lib = _lib.load()
        ws = self._workspace(K)
        y = torch.empty((K, self.n), dtype=torch.complex128, device="cuda")
        pinv = None
        if want_pinv:
            if self.pinv is None:
                self.pinv = torch.empty((self.n // 3, 3, 3), dtype=torch.complex128, device="cuda")
            pinv = self.pinv
        full = (1 << K) - 1
        t_mask, u_mask = masks if masks is not None else (full, full)
        _lib.check(lib.ewb_matfree_apply_masked(
            self.asm.ctx, self.omega.real, self.omega.imag, _lib.ptr(vt),
            _lib.ptr(vu) if vu is not None else None, K, t_mask, u_mask, _lib.ptr(y),
            _lib.ptr(self.kinds_dev), _lib.ptr(pinv) if pinv is not None else None,
            _lib.ptr(ws), ws.numel(), None, _lib.stream_handle()), "ewb_matfree_apply")
        self.applications += 1
        return y

    def apply_gated(self, vt_ptr: int, vu_ptr, w_ptr: int, gate_ptr: int):
        """w = T vt + U vu (device pointers, one vector), skipped on the
        device when *gate == 0 (the operator GMRES's queued iterations)."""
        lib = _lib.load()
        ws = self._workspace(1)
        _lib.check(lib.ewb_matfree_apply(
            self.asm.ctx, self.omega.real, self.omega.imag, vt_ptr, vu_ptr, 1, w_ptr, None, None,
            _lib.ptr(ws), ws.numel(), gate_ptr, _lib.stream_handle()), "ewb_matfree_apply")

    def _split(self, V):
        """(vt, vu) for A: vt = mask_N v, vu = -mask_D v."""
        torch = _torch()
        if self.all_neumann:
            return V.contiguous(), None
        zero = torch.zeros((), dtype=V.dtype, device=V.device)
        vt = torch.where(self._mask_d, zero, V).contiguous()
        vu = torch.where(self._mask_d, -V, zero).contiguous()
        return vt, vu

    def apply_multi(self, V, want_pinv: bool = False):
        """A V for V (K, n) device, K <= 5, in one pass over all element pairs."""
        vt, vu = self._split(V)
        return self._apply_tu(vt, vu, want_pinv)

    def __call__(self, v):
        torch = _torch()
        v = v.to(device="cuda", dtype=torch.complex128).reshape(1, -1)
        return self.apply_multi(v)[0]

    def rhs_and_apply(self, p, V=None, want_pinv: bool = True):
        """b = U mask_N p - T mask_D p, plus A V (rows of V) in the same pass."""
        torch = _torch()
        p = p.to(device="cuda", dtype=torch.complex128).reshape(1, -1)
        zero = torch.zeros((), dtype=p.dtype, device=p.device)
        bt = torch.where(self._mask_d, -p, zero)
        bu = torch.where(self._mask_d, zero, p)
        if V is None:
            y = self._apply_tu(bt.contiguous(), bu.contiguous(), want_pinv)
            return y[0], None
        vt, vu = self._split(V)
        masks = None
        if vu is None:
            # all-Neumann: the history columns have no U part and b no T part
            vu = torch.zeros_like(vt)
            k = int(V.shape[0])
            if k + 1 <= self.MAX_K:
                masks = ((1 << k) - 1, 1 << k)
        y = self._apply_tu(torch.cat([vt, bt]).contiguous(), torch.cat([vu, bu]).contiguous(),
                           want_pinv, masks)
        return y[-1], y[:-1]

    def block_preconditioner(self):
        from .linsolve import BlockDiagPreconditioner

        if self.pinv is None:
            torch = _torch()
            self.apply_multi(torch.zeros((1, self.n), dtype=torch.complex128, device="cuda"),
                             want_pinv=True)
        return BlockDiagPreconditioner(self.pinv)
