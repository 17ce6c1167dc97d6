"""GMRES / SEM for operator callables (the matrix-free seam, linsolve.py:73-77).

Same algorithm as the reference (right preconditioning, MGS Arnoldi,
complex Givens with real cosine, true-residual restart test;
linsolve.py:107-210) with every vector on the device: the operator is
one expensive launch per iteration (ewb_matfree_apply), the Arnoldi
dot/axpy run on device tensors with the coefficients kept on the device,
and the (j+2)-entry Hessenberg column is read back once per iteration for
the Givens update — the only host synchronisation in the loop.
"""

from __future__ import annotations

import logging
import os

import numpy as np

log = logging.getLogger(__name__)


def _torch():
    import torch

    return torch


def gmres_operator(apply_a, b, x0, tol, restart, maxiter, precond, ax0=None):
    """``ax0``: A x0 when the caller already has it (SEM's (A X) s), so the
    initial residual costs no operator application (the dense path's ax0,
    DESIGN.md §8); otherwise r0 = b - A x0 as linsolve.py:144."""
    from .linsolve import SolveStats

    torch = _torch()
    pc = precond if precond is not None else (lambda v: v)
    n = b.shape[0]
    nb = float(torch.linalg.vector_norm(b))
    st = SolveStats()
    if nb == 0.0:
        return torch.zeros(n, dtype=torch.complex128, device="cuda"), st
    x = (torch.zeros(n, dtype=torch.complex128, device="cuda") if x0 is None
         else x0.to(device="cuda", dtype=torch.complex128).clone())
    if ax0 is not None and x0 is not None:
        r = b - ax0
    else:
        r = b - apply_a(x) if bool((x != 0).any()) else b.clone()
    rnorm = float(torch.linalg.vector_norm(r))
    res = rnorm / nb
    st.init_residual = res
    st.residual_history.append(res)
    its = 0
    true_pass = os.environ.get("EWB_TRUE_RESIDUAL_PASS") == "1"
    while res > tol and its < maxiter:
        m = min(restart, maxiter - its)
        V = torch.empty((m + 1, n), dtype=torch.complex128, device="cuda")
        # the cycle's operator products A P^{-1} v_j, kept so that the true
        # residual at the end needs no further application (as ewb_gmres)
        W = None if true_pass else torch.empty((m, n), dtype=torch.complex128, device="cuda")
        r_start = r
        H = np.zeros((m + 1, m), dtype=complex)
        cs = np.zeros(m, dtype=complex)
        sn = np.zeros(m, dtype=complex)
        beta = rnorm
        V[0] = r / beta
        g = np.zeros(m + 1, dtype=complex)
        g[0] = beta
        used = 0
        for j in range(m):
            w = apply_a(pc(V[j])).clone()
            if W is not None:
                W[j] = w
            hcol = torch.empty(j + 2, dtype=torch.complex128, device="cuda")
            for i in range(j + 1):
                h = torch.vdot(V[i], w)
                hcol[i] = h
                w -= h * V[i]
            hn = torch.linalg.vector_norm(w)
            hcol[j + 1] = hn
            col = hcol.cpu().numpy()
            H[: j + 2, j] = col
            if col[j + 1].real > 0:
                V[j + 1] = w / hn
            for i in range(j):
                top = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + np.conj(cs[i]) * H[i + 1, j]
                H[i, j] = top
            den = np.sqrt(abs(H[j, j]) ** 2 + abs(H[j + 1, j]) ** 2)
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            elif H[j, j] == 0.0:
                cs[j], sn[j] = 0.0, 1.0
            else:
                cs[j] = abs(H[j, j]) / den
                sn[j] = (H[j, j] / abs(H[j, j])) * np.conj(H[j + 1, j]) / den
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            used = j + 1
            est = abs(g[j + 1]) / nb
            st.residual_history.append(est)
            if est <= tol:
                break
        y = np.zeros(used, dtype=complex)
        for i in range(used - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:used] @ y[i + 1:used]) / H[i, i]
        yd = torch.from_numpy(y).cuda()
        x = x + pc(V[:used].T @ yd)
        # true residual (linsolve.py:200-201): b - A x_new equals
        # r_start - sum_j y_j A P^{-1} v_j to rounding
        r = b - apply_a(x) if W is None else r_start - W[:used].T @ yd
        rnorm = float(torch.linalg.vector_norm(r))
        res = rnorm / nb
    st.iterations = its
    st.final_residual = res
    st.converged = res <= tol
    if not st.converged:
        log.warning("GMRES stalled at residual %.3e after %d iterations", res, its)
    return x, st


def sem_operator(apply_a, b, xcols, rank_tol, Y=None, return_ax0=False):
    """SEM guess for an operator; Y = A X computed in one multi-vector pass.
    With ``return_ax0`` also returns A x0 = Y s (no extra application)."""
    torch = _torch()
    K = xcols.shape[0]
    if Y is None:
        if hasattr(apply_a, "apply_multi"):
            Y = apply_a.apply_multi(xcols)
        else:
            Y = torch.stack([apply_a(xcols[i]) for i in range(K)])
    Yt = Y.T  # (n, K)
    keep = np.arange(K)
    for _ in range(2):
        q, r = torch.linalg.qr(Yt[:, keep])
        dg = torch.abs(torch.diagonal(r)).cpu().numpy()
        good = dg >= rank_tol * dg.max() if dg.max() > 0 else dg > 0
        if good.all():
            s = torch.linalg.solve(r, q.conj().T @ b)
            x0 = (xcols[keep].T @ s).to(torch.complex128)
            return (x0, (Yt[:, keep] @ s).to(torch.complex128)) if return_ax0 else x0
        keep = keep[good]
        if keep.size == 0:
            break
    return (xcols[0].clone(), Y[0].clone()) if return_ax0 else xcols[0].clone()
