"""Multi-core CPU run of the reference algorithm — TEST / BASELINE INFRASTRUCTURE ONLY.

Used only by ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``)
and by tests, never by the product.  It runs the same per-column work as
``ewbem_oracle.DenseOracle`` (the reference ``Assembler``,
assembly.py:122-254) and the same ``apply_bcs`` / ``block_diag_precond`` /
``sem_initial_guess`` / ``gmres`` (assembly.py:263-297, linsolve.py:80-242),
with the columns dealt to W forked worker processes so a measured CPU time
uses every host core (the reference itself is single-process per frequency;
its fork pool, driver.py:113-122, parallelises over frequencies only when
solution extrapolation is off).

Layout: T, U (n_e,3,n_e,3) and A (N,N) complex128 live in anonymous shared
memory mapped before the fork; worker c owns the element columns
[c n_e/W, (c+1) n_e/W) for the geometry prep, static pass, dynamic assembly
and the BC column swap.  The parent sums the static row-sum partials in
worker order and runs the BLAS parts (b, SEM products, GMRES) with all
BLAS threads.
"""

from __future__ import annotations

import mmap
import multiprocessing as mp
import os
import time

import numpy as np

from . import ewbem_oracle as O


def _shared(shape, dtype):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = mmap.mmap(-1, max(n, 1), flags=mmap.MAP_SHARED)
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape), buf


class _Worker:
    """State of one forked worker: its columns' pair data (assembly.py:142-171)."""

    def __init__(self, par, cols):
        self.p, self.cols = par, cols
        self.data = []
        self.rowsums = None

    def prep(self):
        p = self.p
        g, xc = p.g, p.g["centroids"]
        far, mid = O.rule_g3(), O.rule_g7()
        near_cache = {}
        tier = O.tiers_for_rows(xc, g["diameters"], np.arange(p.n_e), self.cols)
        for jj, j in enumerate(self.cols):
            vj = g["corners"][j]
            groups = []
            for tid, rule in ((0, far), (1, mid)):
                rows = np.flatnonzero(tier[:, jj] == tid)
                rows = rows[rows != j]
                if rows.size:
                    groups.append((rows, rule))
            nr = np.flatnonzero(tier[:, jj] == 2)
            nr = nr[nr != j]
            if nr.size:
                lv = O.near_level(O.surface_distance(xc[nr], vj) / g["diameters"][j])
                for lvl in np.unique(lv):
                    if lvl not in near_cache:
                        near_cache[lvl] = O.rule_refine(O.rule_g7(), int(lvl))
                    groups.append((nr[lv == lvl], near_cache[lvl]))
            buckets = []
            for rows, (bary, wts) in groups:
                r, d, dn = O.pair_geom(xc[rows], bary @ vj, g["normals"][j])
                buckets.append((rows, wts * g["areas"][j], r, d, dn))
            ys, ws = O.self_points(vj)
            r, d, dn = O.pair_geom(xc[j][None, :], ys, g["normals"][j])
            self.data.append((j, buckets, (ws, r, d, dn)))
        return None

    def static(self):                               # assembly.py:193-205
        p = self.p
        part = np.zeros((p.n_e, 3, 3))
        for j, buckets, _ in self.data:
            for rows, w, r, d, dn in buckets:
                _, tb = O.blocks_static(r, d, dn, w, p.g["normals"][j], p.med)
                part[rows] += tb
        return part

    def set_rowsums(self, rs):
        self.rowsums = rs

    def tu(self, omega):                            # assembly.py:219-254
        p = self.p
        tm, um = p.tm, p.um
        ok = True
        for j, buckets, (ws, r, d, dn) in self.data:
            nj = p.g["normals"][j]
            for rows, w, rr, dd, ddn in buckets:
                ub, tb = O.blocks_dynamic(rr, dd, ddn, w, nj, p.med, omega)
                um[rows, :, j, :] = ub
                tm[rows, :, j, :] = tb
            ud, td = O.blocks_dynamic(r, d, dn, ws, nj, p.med, omega)
            _, ts = O.blocks_static(r, d, dn, ws, nj, p.med)
            um[j, :, j, :] = ud[0]
            tm[j, :, j, :] = -self.rowsums[j] + (td[0] - ts[0])
            ok = ok and bool(np.isfinite(tm[:, :, j, :]).all() and np.isfinite(um[:, :, j, :]).all())
        return ok

    def bcs(self, dmask):                           # assembly.py:293-294 (own columns)
        p = self.p
        n = 3 * p.n_e
        t2, u2 = p.tm.reshape(n, n), p.um.reshape(n, n)
        for j in self.cols:
            for c in range(3):
                q = 3 * j + c
                p.a[:, q] = -u2[:, q] if dmask[q] else t2[:, q]
        return None


def _serve(conn, par, cols, nthreads):
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(nthreads)
    except Exception:
        pass
    w = _Worker(par, cols)
    while True:
        msg = conn.recv()
        if msg is None:
            break
        name, args = msg
        t0 = time.perf_counter()
        out = getattr(w, name)(*args)
        conn.send((out, time.perf_counter() - t0))


class ParallelOracle:
    """The reference per-frequency path on W host processes (timing baseline)."""

    def __init__(self, vertices, triangles, med: O.Medium, workers: int | None = None):
        self.g = O.element_geometry(vertices, triangles)
        self.med = med
        self.n_e = len(triangles)
        n = 3 * self.n_e
        self.workers = max(1, min(workers or os.cpu_count() or 1, self.n_e))
        self.tm, self._b1 = _shared((self.n_e, 3, self.n_e, 3), np.complex128)
        self.um, self._b2 = _shared((self.n_e, 3, self.n_e, 3), np.complex128)
        self.a, self._b3 = _shared((n, n), np.complex128)
        ctx = mp.get_context("fork")
        bounds = np.linspace(0, self.n_e, self.workers + 1).astype(int)
        self.conns, self.procs = [], []
        for c in range(self.workers):
            here, there = ctx.Pipe()
            cols = np.arange(bounds[c], bounds[c + 1])
            pr = ctx.Process(target=_serve, args=(there, self, cols, 1), daemon=True)
            pr.start()
            self.conns.append(here)
            self.procs.append(pr)
        self.seconds = {}
        t0 = time.perf_counter()
        self._all("prep")
        t1 = time.perf_counter()
        parts = self._all("static")
        self.rowsums = np.zeros((self.n_e, 3, 3))
        for part in parts:
            self.rowsums += part
        self._all("set_rowsums", self.rowsums)
        self.seconds["prep_s"] = t1 - t0
        self.seconds["static_s"] = time.perf_counter() - t1

    def _all(self, name, *args):
        for c in self.conns:
            c.send((name, args))
        return [c.recv()[0] for c in self.conns]

    def tu(self, omega):
        if not all(self._all("tu", complex(omega))):
            raise FloatingPointError(f"non-finite entries assembled at omega = {omega}")
        n = 3 * self.n_e
        return self.tm.reshape(n, n), self.um.reshape(n, n)

    def system(self, omega, kinds, prescribed):
        """apply_bcs (assembly.py:263-297) with the column swap on the workers."""
        t_mat, u_mat = self.tu(omega)
        kinds = np.asarray(kinds).reshape(-1)
        dmask = kinds == O.DIRICHLET
        self._all("bcs", dmask)
        p = np.asarray(prescribed, dtype=complex)
        nm = ~dmask
        b = u_mat[:, nm] @ p[nm]
        b -= t_mat[:, dmask] @ p[dmask]
        return self.a, b

    def solve_frequency(self, omega, kinds, prescribed, history=None, tol=1e-8, restart=60,
                        maxiter=1000):
        """One complete frequency of run_sweep (driver.py:128-153): assembly,
        BCs, SEM guess, block preconditioner, GMRES.  Returns (x, stats, parts)."""
        parts = {}
        t0 = time.perf_counter()
        a_mat, b = self.system(omega, kinds, prescribed)
        t1 = time.perf_counter()
        x0 = O.sem_guess(history, a_mat, b) if history is not None and len(history) else None
        t2 = time.perf_counter()
        pc, _ = O.block_precond(a_mat)
        x, st = O.gmres(a_mat, b, x0=x0, tol=tol, restart=restart, maxiter=maxiter, precond=pc)
        t3 = time.perf_counter()
        parts.update(assembly_bcs_s=t1 - t0, sem_s=t2 - t1, precond_gmres_s=t3 - t2,
                     total_s=t3 - t0)
        return x, st, parts

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for pr in self.procs:
            pr.join(timeout=10)
            if pr.is_alive():
                pr.terminate()
        self.conns, self.procs = [], []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sweep_seconds(cfg_arrays, workers=None, frequencies=None):
    """Time the reference sweep loop (driver.py:92-176) on the host.

    ``cfg_arrays``: dict(vertices, triangles, med, kinds, dof_signal,
    signal_samples, period, n_omega, kappa, sem_depth, sem, tol, restart,
    maxiter).  ``frequencies``: solve k = 0..f-1 only (None = all).
    Returns dict(setup_s, per_freq_s [list], its [list], workers)."""
    c = cfg_arrays
    t0 = time.perf_counter()
    eta = O.eta_from_kappa(c["kappa"], c["period"])
    om = O.frequency_grid(c["period"], c["n_omega"], eta)
    nf = len(om) if frequencies is None else min(len(om), frequencies)
    spectra = np.stack([O.forward_spectrum(s, c["period"], eta)[:len(om)]
                        for s in c["signal_samples"]])
    par = ParallelOracle(c["vertices"], c["triangles"], c["med"], workers)
    setup = time.perf_counter() - t0
    hist = O.History(c["sem_depth"]) if c["sem"] else None
    per, its, parts = [], [], []
    try:
        for k in range(nf):
            t1 = time.perf_counter()
            p = spectra[np.asarray(c["dof_signal"]), k]
            x, st, pt = par.solve_frequency(om[k], c["kinds"], p, hist, c["tol"], c["restart"],
                                            c["maxiter"])
            if hist is not None:
                hist.push(x)
            per.append(time.perf_counter() - t1)
            its.append(st.iterations)
            parts.append(pt)
    finally:
        par.close()
    return dict(setup_s=setup, prep_s=par.seconds["prep_s"], static_s=par.seconds["static_s"],
                per_freq_s=per, its=its, parts=parts, workers=par.workers)
