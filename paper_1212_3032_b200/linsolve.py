"""Krylov solves on the B200 (mirror of reference ``linsolve.py``).

* ``gmres(apply_a, b, x0, tol, restart, maxiter, precond)`` — for a dense
  matrix the whole restarted, right-preconditioned GMRES (MGS + complex
  Givens, true-residual restart test; linsolve.py:107-210) runs as ONE
  cooperative kernel launch (``ewb_gmres``).  A callable ``apply_a`` (the
  matrix-free seam, linsolve.py:73-77) runs the same algorithm with the
  operator launched per iteration and the Arnoldi vectors on the device.
* ``block_diag_precond(A)`` — inverse 3x3 diagonal blocks on the device.
* ``sem_initial_guess(history, apply_a, b)`` — Y = A X in one pass, QR with
  the rank filter, x0 = X R^{-1} Q^H b (linsolve.py:213-242).
* ``SolutionHistory`` keeps the newest-first ring buffer in HBM.

Arrays are CUDA tensors; numpy inputs are uploaded once.
"""

from __future__ import annotations

import ctypes
import logging
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib

log = logging.getLogger(__name__)


def _torch():
    import torch

    return torch


@dataclass
class SolveStats:
    """Per-solve record (linsolve.py:28-48)."""

    k: int = -1
    omega: complex = 0.0
    iterations: int = 0
    init_residual: float = 0.0
    final_residual: float = 0.0
    seconds: float = 0.0
    converged: bool = True
    residual_history: list = field(default_factory=list, repr=False)
    matvecs: int = 0   # device extra: passes over A inside the solve

    CSV_HEADER = "k,omega_re,omega_im,iterations,init_residual,final_residual,seconds"

    def csv_row(self) -> str:
        omega = complex(self.omega)
        return (f"{self.k},{omega.real!r},{omega.imag!r},{self.iterations},"
                f"{float(self.init_residual)!r},{float(self.final_residual)!r},"
                f"{float(self.seconds)!r}")


def _dev(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.complex128).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=complex))).cuda()


class SolutionHistory:
    """Newest-first ring of the last ``capacity`` solutions, kept in HBM."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("history capacity must be >= 1")
        self.capacity = capacity
        self._buf = None   # (capacity, n) complex128, row 0 newest
        self._len = 0

    def push(self, x) -> None:
        torch = _torch()
        x = _dev(x).reshape(-1)
        if self._buf is None or self._buf.shape[1] != x.shape[0]:
            self._buf = torch.zeros((self.capacity, x.shape[0]), dtype=torch.complex128,
                                    device="cuda")
            self._len = 0
        if self.capacity > 1:
            self._buf[1:] = self._buf[:-1].clone()
        self._buf[0] = x
        self._len = min(self._len + 1, self.capacity)

    def __len__(self) -> int:
        return self._len

    def columns(self):
        """(K, n) device tensor, row c = c-th newest solution (contiguous)."""
        if not self._len:
            raise ValueError("empty solution history")
        return self._buf[: self._len]

    def matrix(self):
        """(n, K) like the reference (newest first), as a device tensor."""
        return self.columns().T


class BlockDiagPreconditioner:
    """v -> P^{-1} v with P the 3x3 diagonal blocks of A (linsolve.py:80-104)."""

    def __init__(self, pinv):
        self.pinv = pinv  # (n/3, 3, 3) complex128 cuda

    def __call__(self, v):
        torch = _torch()
        v = _dev(v)
        nb = self.pinv.shape[0]
        return torch.einsum("bij,bj->bi", self.pinv, v.reshape(nb, 3)).reshape(-1)


def block_diag_precond(a_mat) -> BlockDiagPreconditioner:
    torch = _torch()
    lib = _lib.require_cuda()
    a = _dev(a_mat)
    n = a.shape[0]
    if a.dim() != 2 or a.shape != (n, n) or n % 3:
        raise ValueError("matrix must be square with size divisible by 3")
    pinv = torch.empty((n // 3, 3, 3), dtype=torch.complex128, device="cuda")
    sing = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(lib.ewb_blockdiag_inverse(_lib.ptr(a), n, _lib.ptr(pinv), _lib.ptr(sing),
                                         _lib.stream_handle()), "ewb_blockdiag_inverse")
    ns = int(sing.item())
    if ns:
        log.warning("%d singular 3x3 diagonal blocks; identity fallback", ns)
    return BlockDiagPreconditioner(pinv)


class _Workspace:
    """Cached device scratch for ewb_gmres / ewb_sem_guess."""

    def __init__(self):
        self.buf = None
        self.hist = None
        self.res = None

    def get(self, nbytes: int):
        torch = _torch()
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        return self.buf

    def hist_buf(self, cap: int):
        torch = _torch()
        if self.hist is None or self.hist.numel() < cap:
            self.hist = torch.empty(cap, dtype=torch.float64, device="cuda")
        return self.hist

    def result(self):
        torch = _torch()
        if self.res is None:
            self.res = torch.zeros(64, dtype=torch.uint8, device="cuda")
        return self.res


_WS = _Workspace()


def gmres_device(a, b, x, has_x0: bool, tol: float, restart: int, maxiter: int, pinv=None,
                 ws: _Workspace | None = None, stats: SolveStats | None = None,
                 sync: bool = True, ax0=None, res=None, hist=None):
    """Dense GMRES on device tensors; x (n,) is in/out.  Returns SolveStats.

    ax0: optional device A x0 (e.g. from :func:`sem_device`), saving the
    initial residual's pass over A.  res / hist: optional caller-owned result
    (64 B) and history buffers, so several solves can be queued without a
    host read-back in between (``sync=False``)."""
    lib = _lib.load()
    ws = ws or _WS
    n = int(b.shape[0])
    nbytes = int(lib.ewb_gmres_workspace_bytes(n, restart))
    buf = ws.get(nbytes)
    cap = gmres_hist_cap(maxiter, restart)
    hist = ws.hist_buf(cap) if hist is None else hist
    cap = min(cap, hist.numel())
    res = ws.result() if res is None else res
    _lib.check(lib.ewb_gmres(_lib.ptr(a), _lib.ptr(b), _lib.ptr(pinv) if pinv is not None else None,
                             _lib.ptr(x), int(bool(has_x0)),
                             _lib.ptr(ax0) if (ax0 is not None and has_x0) else None,
                             n, float(tol), int(restart),
                             int(maxiter), _lib.ptr(buf), buf.numel(), _lib.ptr(hist), cap,
                             _lib.ptr(res), _lib.stream_handle()), "ewb_gmres")
    st = stats or SolveStats()
    if sync:
        _fill_stats(st, res, hist)
    return st


_CONC_WS: list = []


def gmres_device_concurrent(As, bs, xs, tol: float, restart: int, maxiter: int, pinvs=None,
                            ress=None, hists=None, sync: bool = True):
    """Independent dense GMRES solves (SEM off: the frequencies of a sweep do
    not depend on each other) run side by side, each on its own stream with
    ~1/m of the SMs (ewb_set_solver_ctas), instead of one after another with
    the whole GPU.  Each solve then streams A at its SMs' share of the HBM
    bandwidth while its per-step reductions and grid barriers overlap the
    other solves' streaming, so small systems, whose passes are short next
    to the per-step overhead, gain most.  Same algorithm and results per
    system as ``gmres_device`` up to the grid-size dependent grouping of the
    dot-product partials (rounding)."""
    torch = _torch()
    lib = _lib.load()
    m = len(bs)
    if m == 0:
        return []
    while len(_CONC_WS) < m:
        _CONC_WS.append(_Workspace())
    full = int(lib.ewb_solver_ctas())
    per = max(1, full // m)
    main = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in range(m)]
    stats = [SolveStats() for _ in range(m)]
    _lib.check(lib.ewb_set_solver_ctas(per))
    try:
        for i in range(m):
            streams[i].wait_stream(main)
            with torch.cuda.stream(streams[i]):
                gmres_device(As[i], bs[i], xs[i], False, tol, restart, maxiter,
                             None if pinvs is None else pinvs[i], ws=_CONC_WS[i],
                             stats=stats[i], sync=False,
                             res=None if ress is None else ress[i],
                             hist=None if hists is None else hists[i])
    finally:
        _lib.check(lib.ewb_set_solver_ctas(full))   # the caller's budget back
    for st_ in streams:
        main.wait_stream(st_)
    if sync:
        for i in range(m):
            _fill_stats(stats[i], _CONC_WS[i].result() if ress is None else ress[i],
                        _CONC_WS[i].hist_buf(1) if hists is None else hists[i])
    return stats


def gmres_hist_cap(maxiter: int, restart: int) -> int:
    """Residual-history slots one solve can write (init + per iteration + per cycle)."""
    return maxiter + 2 + maxiter // max(restart, 1) + 2


def _fill_stats(st: SolveStats, res, hist):
    r = res[:32].cpu().numpy().view(np.uint8)
    out = _lib.GmresResult.from_buffer_copy(r.tobytes())
    st.iterations = out.iterations
    st.init_residual = out.init_residual
    st.final_residual = out.final_residual
    st.converged = bool(out.converged)
    st.matvecs = out.matvecs
    nh = min(out.n_hist, hist.numel())
    st.residual_history = hist[:nh].cpu().tolist() if nh else []
    return st


def gmres(apply_a, b, x0=None, tol: float = 1e-5, restart: int = 60, maxiter: int = 1000,
          precond=None):
    """Restarted right-preconditioned GMRES (linsolve.py:107-210) on the GPU.

    Returns (x, SolveStats) with x a CUDA tensor.
    """
    torch = _torch()
    t0 = time.perf_counter()
    if not 0.0 < tol < 1.0:
        raise ValueError(f"tol must be in (0, 1), got {tol}")
    _lib.require_cuda()
    bd = _dev(b).reshape(-1)
    n = bd.shape[0]
    pinv = None
    if precond is not None:
        if isinstance(precond, BlockDiagPreconditioner):
            pinv = precond.pinv
        elif not callable(apply_a) or hasattr(apply_a, "matvec_device"):
            raise TypeError("precond must come from block_diag_precond() on the device path")
    if callable(apply_a) and not _is_matrix(apply_a):
        from .krylov_host import gmres_operator

        x, st = gmres_operator(apply_a, bd, x0, tol, restart, maxiter, precond)
        st.seconds = time.perf_counter() - t0
        return x, st
    a = _dev(apply_a)
    if a.shape != (n, n):
        raise ValueError("matrix/vector size mismatch")
    x = torch.zeros(n, dtype=torch.complex128, device="cuda") if x0 is None else _dev(x0).clone()
    st = gmres_device(a, bd, x, x0 is not None, tol, restart, maxiter, pinv)
    if not st.converged:
        log.warning("GMRES stalled at residual %.3e after %d iterations",
                    st.final_residual, st.iterations)
    st.seconds = time.perf_counter() - t0
    return x, st


def _is_matrix(a) -> bool:
    torch = _torch()
    return isinstance(a, (np.ndarray, torch.Tensor))


class SemWorkspace:
    def __init__(self):
        self.buf = None
        self.res = None

    def get(self, nbytes):
        torch = _torch()
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        if self.res is None:
            self.res = torch.zeros(16, dtype=torch.uint8, device="cuda")
        return self.buf, self.res


_SEM_WS = SemWorkspace()


def sem_device(a, b, xcols, rank_tol: float, x0_out, ws: SemWorkspace | None = None,
               ax0_out=None):
    """x0_out <- SEM guess for dense a (device); xcols (K, n) newest first.
    ax0_out (optional): receives A x0 from the same products."""
    lib = _lib.load()
    ws = ws or _SEM_WS
    K, n = int(xcols.shape[0]), int(xcols.shape[1])
    nbytes = int(lib.ewb_sem_workspace_bytes(n, K))
    buf, res = ws.get(nbytes)
    _lib.check(lib.ewb_sem_guess(_lib.ptr(a), _lib.ptr(b), _lib.ptr(xcols), K, n,
                                 float(rank_tol), _lib.ptr(x0_out),
                                 _lib.ptr(ax0_out) if ax0_out is not None else None,
                                 _lib.ptr(buf), buf.numel(),
                                 _lib.ptr(res), _lib.stream_handle()), "ewb_sem_guess")
    return res


def sem_initial_guess(history: SolutionHistory, apply_a, b, rank_tol: float = 1e-10):
    """Least-squares extrapolated initial guess (linsolve.py:213-242)."""
    torch = _torch()
    _lib.require_cuda()
    xcols = history.columns().contiguous()
    bd = _dev(b).reshape(-1)
    if callable(apply_a) and not _is_matrix(apply_a):
        from .krylov_host import sem_operator

        return sem_operator(apply_a, bd, xcols, rank_tol)
    a = _dev(apply_a)
    x0 = torch.empty_like(bd)
    sem_device(a, bd, xcols, rank_tol, x0)
    return x0
