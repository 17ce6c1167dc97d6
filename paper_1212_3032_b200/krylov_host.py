"""GMRES / SEM for operator callables (the matrix-free seam, linsolve.py:73-77).

The reference's algorithm (right preconditioning, MGS Arnoldi, complex
Givens with real cosine, exit decided on the literal residual b - A x;
linsolve.py:107-210) with every vector, coefficient and decision on the
device: ``ewb_opgmres_phase`` kernels hold the whole solver state in HBM
(``ewb_op_head`` + Hessenberg/Givens arrays), the operator is applied by
its own launches between them, and the host only enqueues.  Operator
applications carry a device gate word, so a chunk of iterations is queued
ahead and the ones past convergence do no work; the host reads the
4-byte ``done`` word once per chunk (one synchronisation per solve at the
sizes of cfg5, not one per iteration).

A generic Python callable cannot be gated: it is called once per
iteration after reading the gate word (the seam accepts any callable; the
B200 hot path is ``MatrixFreeOperator``).

SEM (linsolve.py:213-242) for an operator: Y = A X from one multi-vector
application, then the device CGS2 QR / rank filter / solve of
``ewb_sem_from_products`` (the dense path's ``k_sem``).
"""

from __future__ import annotations

import ctypes
import logging

from . import _lib

log = logging.getLogger(__name__)


def _torch():
    import torch

    return torch


class OpHead(ctypes.Structure):
    """``ewb_op_head`` (include/ewbem_b200.h)."""

    _fields_ = [(nm, ctypes.c_int32) for nm in
                ("in_cycle", "lit_pending", "done", "converged", "iterations", "j", "m", "used",
                 "cycle_open", "n_hist", "applications", "pad")] + \
               [(nm, ctypes.c_double) for nm in
                ("norm_b", "rnorm", "residual", "init_residual", "final_residual")]


class OpSolver:
    """Device workspace + enqueue logic of one operator GMRES (reusable)."""

    CHUNK = 8   # Arnoldi steps queued between two reads of the `done` word

    def __init__(self, n: int, restart: int, maxiter: int):
        torch = _torch()
        lib = _lib.require_cuda()
        self.lib = lib
        self.n, self.restart, self.maxiter = n, restart, maxiter
        nbytes = int(lib.ewb_opgmres_workspace_bytes(n, restart))
        if nbytes < 0:
            raise ValueError("restart must be in [1, 128]")
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        from .linsolve import gmres_hist_cap

        self.hist_cap = gmres_hist_cap(maxiter, restart)
        self.hist = torch.zeros(self.hist_cap, dtype=torch.float64, device="cuda")
        ptrs = [ctypes.c_void_p() for _ in range(4)]
        gates = [ctypes.POINTER(ctypes.c_int32)() for _ in range(2)]
        _lib.check(lib.ewb_opgmres_buffers(_lib.ptr(self.ws), n, restart,
                                           *[ctypes.byref(p) for p in ptrs],
                                           *[ctypes.byref(g) for g in gates]),
                   "ewb_opgmres_buffers")
        self.z_ptr, self.vt_ptr, self.vu_ptr, self.w_ptr = (p.value for p in ptrs)
        self.gate_cycle = ctypes.cast(gates[0], ctypes.c_void_p).value
        self.gate_lit = ctypes.cast(gates[1], ctypes.c_void_p).value
        self.head_host = torch.empty(ctypes.sizeof(OpHead), dtype=torch.uint8, pin_memory=True)
        self.done_host = torch.empty(4, dtype=torch.uint8, pin_memory=True)
        base = _lib.ptr(self.ws)
        off = OpHead.done.offset
        self.ws_done = self.ws[off:off + 4]
        self.ws_head = self.ws[:ctypes.sizeof(OpHead)]
        self.z = self._view(self.z_ptr - base)
        self.w = self._view(self.w_ptr - base)

    def _view(self, off):
        return self.ws[off:off + 16 * self.n].view(_torch().complex128)

    def _phase(self, ph, b, x, has_x0, ax0, pinv, kinds, split_u, tol):
        _lib.check(self.lib.ewb_opgmres_phase(
            ph, _lib.ptr(self.ws), self.ws.numel(), _lib.ptr(b), _lib.ptr(x), int(has_x0),
            _lib.ptr(ax0) if ax0 is not None else None,
            _lib.ptr(pinv) if pinv is not None else None,
            _lib.ptr(kinds) if kinds is not None else None, int(split_u), self.n, float(tol),
            self.restart, self.maxiter, _lib.ptr(self.hist), self.hist_cap,
            _lib.stream_handle()), "ewb_opgmres_phase")

    def head(self) -> OpHead:
        self.head_host.copy_(self.ws_head)
        return OpHead.from_buffer_copy(self.head_host.numpy().tobytes())

    def solve(self, op, b, x, has_x0, tol, pinv, ax0=None):
        """x <- GMRES solution of op x = b; returns the final ewb_op_head."""
        gated = hasattr(op, "apply_gated")
        kinds = op.kinds_dev if gated and not op.all_neumann else None
        split_u = kinds is not None
        args = (b, x, has_x0, ax0, pinv, kinds, split_u, tol)

        def apply(gate):
            if gated:
                op.apply_gated(self.vt_ptr, self.vu_ptr if split_u else None, self.w_ptr, gate)
            else:   # a plain callable: decide on the host
                self.done_host.copy_(self.ws[OpHead.in_cycle.offset if gate == self.gate_cycle
                                             else OpHead.lit_pending.offset:][:4])
                if int(self.done_host.view(_torch().int32)[0]):
                    self.w.copy_(op(self.z))

        self._phase(0, *args)
        apply(self.gate_lit)
        self._phase(3, *args)
        chunk = self.CHUNK if gated else 1
        while True:
            self.done_host.copy_(self.ws_done)
            if int(self.done_host.view(_torch().int32)[0]):
                break
            for _ in range(chunk):
                apply(self.gate_cycle)
                self._phase(1, *args)
            self._phase(2, *args)
            apply(self.gate_lit)
            self._phase(3, *args)
        return self.head()


_SOLVERS: dict = {}


def gmres_operator(apply_a, b, x0, tol, restart, maxiter, precond, ax0=None):
    """Operator GMRES on the device.  ``ax0``: A x0 when the caller already
    has it (SEM's (A X) s): the initial residual then costs no application
    unless it already meets tol."""
    from .linsolve import BlockDiagPreconditioner, SolveStats

    torch = _torch()
    n = int(b.shape[0])
    pinv = None
    if precond is not None:
        if not isinstance(precond, BlockDiagPreconditioner):
            raise TypeError("precond must be a BlockDiagPreconditioner on the device path")
        pinv = precond.pinv
    key = (n, restart, maxiter)
    solver = _SOLVERS.get(key)
    if solver is None:
        _SOLVERS.clear()   # one live workspace (cfg5: V and W are 236 MB each)
        solver = _SOLVERS[key] = OpSolver(n, restart, maxiter)
    b = b.to(device="cuda", dtype=torch.complex128).contiguous()
    x = (torch.zeros(n, dtype=torch.complex128, device="cuda") if x0 is None
         else x0.to(device="cuda", dtype=torch.complex128).clone())
    if ax0 is not None:
        ax0 = ax0.to(device="cuda", dtype=torch.complex128).contiguous()
    head = solver.solve(apply_a, b, x, x0 is not None, tol, pinv, ax0)
    st = SolveStats(iterations=head.iterations, init_residual=head.init_residual,
                    final_residual=head.final_residual, converged=bool(head.converged),
                    matvecs=head.applications)
    nh = min(head.n_hist, solver.hist_cap)
    st.residual_history = solver.hist[:nh].cpu().tolist() if nh else []
    if not st.converged:
        log.warning("GMRES stalled at residual %.3e after %d iterations",
                    st.final_residual, st.iterations)
    return x, st


_SEM_WS: dict = {}


def sem_operator(apply_a, b, xcols, rank_tol, Y=None, return_ax0=False):
    """SEM guess for an operator: Y = A X in one multi-vector application
    (unless given), then the device QR / rank filter / solve.  With
    ``return_ax0`` also returns A x0 = Y s (no extra application)."""
    torch = _torch()
    lib = _lib.require_cuda()
    xcols = xcols.contiguous()
    K, n = int(xcols.shape[0]), int(xcols.shape[1])
    if Y is None:
        Y = (apply_a.apply_multi(xcols) if hasattr(apply_a, "apply_multi")
             else torch.stack([apply_a(xcols[i]) for i in range(K)]))
    Y = Y.contiguous()
    nbytes = int(lib.ewb_sem_workspace_bytes(n, K))
    ws = _SEM_WS.get("ws")
    if ws is None or ws.numel() < nbytes:
        ws = _SEM_WS["ws"] = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        _SEM_WS["res"] = torch.zeros(16, dtype=torch.uint8, device="cuda")
    x0 = torch.empty(n, dtype=torch.complex128, device="cuda")
    ax0 = torch.empty(n, dtype=torch.complex128, device="cuda") if return_ax0 else None
    bd = b.to(device="cuda", dtype=torch.complex128).contiguous()
    _lib.check(lib.ewb_sem_from_products(
        _lib.ptr(bd), _lib.ptr(xcols), _lib.ptr(Y), K, n, float(rank_tol), _lib.ptr(x0),
        _lib.ptr(ax0) if ax0 is not None else None, _lib.ptr(ws), ws.numel(),
        _lib.ptr(_SEM_WS["res"]), _lib.stream_handle()), "ewb_sem_from_products")
    return (x0, ax0) if return_ax0 else x0
