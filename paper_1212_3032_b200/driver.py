"""Frequency sweep on one B200 (mirror of reference ``driver.py:92-176``).

``run_sweep(cfg) -> SweepResult`` keeps the reference's sequencing exactly
(ascending k, SEM history pushed after each solve, probes, NaN poisoning of
every history when any solve fails, manifest) while every per-frequency
array stays in HBM.  The device loop lives in :class:`DeviceSweep`:

    per group of nb (default 16) consecutive k:
            ewb_assemble_system_multi (assembly + BCs + b + P^{-1} of all nb
                                  frequencies in one pass over the element
                                  pairs; no T/U)
    per k:  ewb_sem_guess         (if history: Y = A X, QR, x0)
            ewb_gmres             (the whole restarted solve, one launch)
            one small read-back   (fault flags + iteration count + residuals)
    end:    ewb_window_idft       (conjugate fill + window + IDFT for the
                                   probe columns, or all DOFs)

With SEM off and torch.distributed initialised with world > 1, the
frequencies are dealt round-robin to the ranks (the reference's fork pool,
driver.py:113-122, as replicas on separate GPUs) and the per-frequency
results are all-gathered once at the end.
"""

from __future__ import annotations

import ctypes
import logging
import math
import os
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from .assembly import DIRICHLET, NEUMANN, Assembler
from .linsolve import SolveStats, block_diag_precond, gmres_device, sem_device
from .transform import (check_residue, eta_from_kappa, forward_mft_batch, frequency_grid,
                        windowed_inverse_device)

log = logging.getLogger(__name__)


class SweepError(RuntimeError):
    """A frequency solve failed in a way that invalidates the sweep."""


@dataclass
class SweepResult:
    times: np.ndarray
    histories: dict
    half_spectra: dict
    stats: list
    manifest: dict
    failed_frequencies: list = field(default_factory=list)
    full_field: object = None          # optional (N, n_dofs) device histories

    @property
    def total_iterations(self) -> int:
        return sum(s.iterations for s in self.stats)


def shard_frequencies(n_freq: int, rank: int, world: int) -> list:
    """Round-robin frequency ownership (balanced: low and high k mixed)."""
    return list(range(rank, n_freq, world))


def _dist():
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist
    except Exception:
        pass
    return None


def gather_frequency_results(local: dict, n_freq: int, width: int, dist=None):
    """All-gather {k: (values (width,) complex, stats 6-tuple)} from every rank.

    Returns (values (n_freq, width) complex ndarray, meta (n_freq, 6)).
    Host-side bookkeeping, exercised with the gloo backend in the tests.
    """
    import torch

    dist = dist or _dist()
    world = dist.get_world_size() if dist else 1
    vals = np.zeros((n_freq, width), dtype=complex)
    meta = np.zeros((n_freq, 6))
    owned = np.zeros(n_freq)
    for k, (v, st) in local.items():
        vals[k] = v
        meta[k] = st
        owned[k] = 1
    if world > 1:
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.from_numpy(np.concatenate([vals.view(np.float64), meta,
                                             owned[:, None]], axis=1)).to(dev)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        total = sum(p.cpu().numpy() for p in parts)
        w2 = 2 * width
        vals = np.ascontiguousarray(total[:, :w2]).view(complex)
        meta = total[:, w2:w2 + 6]
        owned = total[:, -1]
    if not np.all(owned == 1):
        raise SweepError("frequency ownership is not a partition of the sweep")
    return vals, meta


MAX_SEM_DEPTH = 8   # SEM history columns the device QR holds (kMaxSem)


def n_hist_passes(K: int) -> int:
    """Passes over A of one SEM product Y = A X (up to 4 columns per pass)."""
    return (K + 3) // 4 if K > 0 else 0


class DeviceSweep:
    """The per-frequency loop with every array resident in HBM.

    Construction uploads the per-run inputs (BC kinds, the prescribed
    spectra of every frequency); ``run()`` performs the sweep and returns
    device tensors.  ``timing=True`` brackets the assembly and solver
    launches of every frequency with CUDA events (phase split for the
    roofline report).
    """

    def __init__(self, cfg, assembler: Assembler | None = None,
                 frequencies: list | None = None, assembly_batch: int | None = None):
        import torch

        _lib.require_cuda()
        if cfg.sem_enabled and cfg.sem_depth > MAX_SEM_DEPTH:
            # rejected before any assembly or solve (the reference accepts any
            # depth; the device SEM keeps up to 8 history columns)
            raise ValueError(f"sem_depth {cfg.sem_depth} > {MAX_SEM_DEPTH} is not supported "
                             "on the device path")
        self.cfg = cfg
        self.eta = eta_from_kappa(cfg.kappa, cfg.period)
        self.omegas = frequency_grid(cfg.period, cfg.n_omega, self.eta)
        self.n_freq = len(self.omegas)
        self.h2d_bytes = 0
        spectra = forward_mft_batch(cfg.signals, cfg.period, cfg.n_omega, self.eta, self.n_freq)
        self.asm = assembler or Assembler(cfg.mesh, cfg.material)
        if assembler is None:
            m = cfg.mesh
            self.h2d_bytes += 8 * (m.centroids.size + m.normals.size + m.areas.size
                                   + m.diameters.size + 9 * m.n_elements)
        n = cfg.mesh.n_dofs
        self.n = n
        self.kinds = np.ascontiguousarray(cfg.bcs.flat_kind(), dtype=np.uint8)
        sig = cfg.bcs.flat_signal().astype(np.int64)
        spec_t = np.ascontiguousarray(spectra.T)                    # (n_freq, n_signals)
        spec_dev = torch.from_numpy(spec_t).cuda()
        sig_dev = torch.from_numpy(sig).cuda()
        self.h2d_bytes += spec_t.nbytes + sig.nbytes + self.kinds.nbytes
        self.P = spec_dev[:, sig_dev].contiguous()                  # (n_freq, n) prescribed
        self.frequencies = list(range(self.n_freq)) if frequencies is None else list(frequencies)
        self.sol = torch.zeros((self.n_freq, n), dtype=torch.complex128, device="cuda")
        self.x = torch.zeros(n, dtype=torch.complex128, device="cuda")
        self.hist = torch.zeros((cfg.sem_depth, n), dtype=torch.complex128, device="cuda")
        self.system = None
        self.batch = None
        self.assembly_batch = assembly_batch
        self.d2h_bytes = 0

    def _p_rows(self, ks):
        """Prescribed spectra of frequencies ks as an (nf, N) device view/copy."""
        return (self.P[ks[0]:ks[-1] + 1] if ks == list(range(ks[0], ks[-1] + 1))
                else self.P[ks].contiguous())

    def batch_size(self) -> int:
        """Frequencies assembled per pass over the element pairs.

        ``assembly_batch`` (constructor) or ``EWB_ASSEMBLY_BATCH`` (default 16),
        capped at 16 and by free HBM: the batch holds nb dense N x N systems
        (cfg2: 3.77 GB each) and may take at most half of the free memory."""
        import torch

        nb = self.assembly_batch
        if nb is None:
            nb = int(os.environ.get("EWB_ASSEMBLY_BATCH", "16"))
        nb = max(1, min(int(nb), 32, len(self.frequencies)))
        if nb > 1 and self.batch is None:
            free, _ = torch.cuda.mem_get_info()
            per = 16 * self.n * self.n + 16 * 4 * self.n
            nb = max(1, min(nb, int(0.65 * free // per)))
        return nb

    def run_matrix_free(self):
        """Matrix-free sweep (north-star item 2): the operator is recomputed in
        every application, nothing of size N^2 is stored.  Per frequency the
        right-hand side, the SEM product Y = A X and the block preconditioner
        come from ONE pass over all element pairs (ewb_matfree_apply with K+1
        vectors); GMRES then applies the operator once per iteration."""
        import torch

        from .krylov_host import gmres_operator, sem_operator
        from .linsolve import BlockDiagPreconditioner
        from .matfree import MatrixFreeOperator

        cfg = self.cfg
        stats = {}
        n_hist = 0
        K = cfg.sem_depth
        self.hist.zero_()
        self.phase = {"applications": 0, "solves": 0, "seconds": 0.0}
        for k in self.frequencies:
            omega = complex(self.omegas[k])
            t0 = time.perf_counter()
            try:
                if omega == 0:
                    raise ValueError("omega == 0 (kappa = 0) needs the dense static path")
                op = MatrixFreeOperator(self.asm, omega, cfg.bcs)
                use_sem = cfg.sem_enabled and n_hist > 0
                hist = self.hist[:n_hist] if use_sem else None
                b, Y = op.rhs_and_apply(self.P[k], hist, want_pinv=True)
                pc = BlockDiagPreconditioner(op.pinv)
                x0, ax0 = (sem_operator(op, b, hist, 1e-10, Y=Y, return_ax0=True) if use_sem
                           else (None, None))
                x, st = gmres_operator(op, b, x0, cfg.tol, cfg.restart, cfg.maxiter, pc,
                                       ax0=ax0)
                nf, sg = ctypes.c_int32(), ctypes.c_int32()
                _lib.check(self.asm._lib.ewb_ctx_flags(self.asm.ctx, ctypes.byref(nf),
                                                       ctypes.byref(sg), _lib.stream_handle()))
                if nf.value:
                    raise FloatingPointError(f"non-finite operator entries at omega = {omega}")
            except SweepError:
                raise
            except Exception as exc:
                raise SweepError(f"frequency index {k} (omega={omega:.6g}): {exc}") from exc
            torch.cuda.synchronize()
            st.k, st.omega = k, omega
            st.seconds = time.perf_counter() - t0
            st.matvecs += op.applications   # GMRES's applications + the b / SEM passes
            stats[k] = st
            self.phase["applications"] += st.matvecs
            self.phase["solves"] += 1
            self.phase["seconds"] += st.seconds
            self.sol[k] = x
            if cfg.sem_enabled:
                self.hist[1:] = self.hist[:-1].clone()
                self.hist[0] = x
                n_hist = min(n_hist + 1, K)
            log.info("k=%d its=%d applications=%d %.2fs", k, st.iterations, st.matvecs,
                     st.seconds)
        return stats

    def run(self, timing: bool = False):
        """Sweep the owned frequencies; returns {k: SolveStats}.

        Every launch of the sweep is queued without a host read-back: the
        fault flags, GMRES results and residual histories of each frequency
        land in per-frequency device slots that are read once at the end
        (the first non-finite frequency then raises, as in driver.py:141-145).
        SEM also returns A x0, so GMRES starts without a pass over A."""
        import torch

        from .linsolve import gmres_hist_cap

        if getattr(self, "matrix_free", False):
            return self.run_matrix_free()
        cfg = self.cfg
        asm = self.asm
        lib = asm._lib
        stats = {}
        ev = []
        n_hist = 0
        K = cfg.sem_depth
        self.hist.zero_()
        self.phase = {"assembly_ms": 0.0, "solve_ms": 0.0, "matvecs": 0, "solves": 0}
        t_host0 = time.perf_counter()
        nf = len(self.frequencies)
        cap = gmres_hist_cap(cfg.maxiter, cfg.restart)
        res_all = torch.zeros((nf, 64), dtype=torch.uint8, device="cuda")
        hist_all = torch.zeros((nf, cap), dtype=torch.float64, device="cuda")
        flags_all = torch.zeros((nf, 4), dtype=torch.int32, device="cuda")
        ax0 = torch.empty(self.n, dtype=torch.complex128, device="cuda")
        nb = self.batch_size()
        asm_ev = []
        # groups: up to nb consecutive frequencies assembled in one pass over
        # the element pairs (omega == 0, the static path, always alone)
        groups = []
        i0 = 0
        while i0 < nf:
            g_ = [i0]
            if complex(self.omegas[self.frequencies[i0]]) != 0:
                while (len(g_) < nb and i0 + len(g_) < nf
                       and complex(self.omegas[self.frequencies[i0 + len(g_)]]) != 0):
                    g_.append(i0 + len(g_))
            groups.append(g_)
            i0 += len(g_)
        conc_env = os.environ.get("EWB_CONCURRENT_SOLVES", "auto")
        concurrent = (not cfg.sem_enabled
                      and (conc_env == "1" or (conc_env == "auto" and self.n < 12000)))
        full_ctas = int(lib.ewb_solver_ctas())
        for gi, group in enumerate(groups):
            ks = [self.frequencies[i] for i in group]
            idx = group[0]
            try:
                e_a = torch.cuda.Event(enable_timing=True)
                e_b = torch.cuda.Event(enable_timing=True)
                e_a.record()
                if complex(self.omegas[ks[0]]) != 0:
                    self.batch = asm.assemble_system_multi(
                        [self.omegas[k] for k in ks], cfg.bcs, self._p_rows(ks), out=self.batch,
                        flags=flags_all[group[0]:group[-1] + 1], check=False)
                    out = self.batch
                    members = [out.member(f) for f in range(len(group))]
                else:
                    omega = complex(self.omegas[ks[0]])
                    sysm = asm.assemble_system(omega, cfg.bcs, self.P[ks[0]], check=False)
                    sysm.pinv = block_diag_precond(sysm.A).pinv   # static path (kappa = 0)
                    _lib.check(lib.ewb_ctx_flags_async(asm.ctx, _lib.ptr(flags_all[group[0]]),
                                                       _lib.stream_handle()),
                               "ewb_ctx_flags_async")
                    members = [sysm]
                e_b.record()
                asm_ev.append((e_a, e_b))
            except SweepError:
                raise
            except Exception as exc:
                _lib.check(lib.ewb_set_solver_ctas(full_ctas))
                omega = complex(self.omegas[ks[0]])
                raise SweepError(f"frequency index {ks[0]} (omega={omega:.6g}): {exc}") from exc
            if concurrent and len(group) > 1:
                # independent members (no SEM chain): solved side by side
                # (measured: 1.4-1.8x faster at N = 3840-4096, 1.06-1.1x at
                # 7680-8192, 4 % slower at 15360-16384, hence the size cut)
                from .linsolve import gmres_device_concurrent

                try:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    gmres_device_concurrent([m.A for m in members], [m.b for m in members],
                                            [self.sol[k] for k in ks], cfg.tol, cfg.restart,
                                            cfg.maxiter, [m.pinv for m in members],
                                            ress=[res_all[i] for i in group],
                                            hists=[hist_all[i] for i in group], sync=False)
                    e1.record()
                except Exception as exc:
                    omega = complex(self.omegas[ks[0]])
                    raise SweepError(f"frequency index {ks[0]} (omega={omega:.6g}): {exc}") from exc
                for j_, (i, k) in enumerate(zip(group, ks)):
                    ev.append((i, k, complex(self.omegas[k]), e0, e1, 0, len(group), j_ == 0))
                continue
            for i, k, sysm in zip(group, ks, members):
                omega = complex(self.omegas[k])
                try:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    use_sem = cfg.sem_enabled and n_hist > 0
                    if use_sem:
                        sem_device(sysm.A, sysm.b, self.hist[:n_hist], 1e-10, self.x, ax0_out=ax0)
                    gmres_device(sysm.A, sysm.b, self.x, use_sem, cfg.tol, cfg.restart,
                                 cfg.maxiter, sysm.pinv, sync=False,
                                 ax0=ax0 if use_sem else None, res=res_all[i], hist=hist_all[i])
                    e1.record()
                except SweepError:
                    raise
                except Exception as exc:
                    _lib.check(lib.ewb_set_solver_ctas(full_ctas))
                    raise SweepError(f"frequency index {k} (omega={omega:.6g}): {exc}") from exc
                ev.append((i, k, omega, e0, e1, n_hist if use_sem else 0, 1, True))
                self.sol[k] = self.x
                if cfg.sem_enabled:
                    self.hist[1:] = self.hist[:-1].clone()
                    self.hist[0] = self.x
                    n_hist = min(n_hist + 1, K)
            _lib.check(lib.ewb_set_solver_ctas(full_ctas))   # the caller's budget back
        t_host1 = time.perf_counter()
        torch.cuda.synchronize()
        t_host2 = time.perf_counter()
        flags = flags_all.cpu().numpy()
        res_host = res_all.cpu().numpy()
        # residual histories: one read-back of the used columns for every frequency
        nh_max = max([min(_lib.GmresResult.from_buffer_copy(res_host[e[0], :32].tobytes()).n_hist,
                          cap) for e in ev] + [0])
        hist_host = hist_all[:, :nh_max].cpu().numpy()
        self.d2h_bytes += flags_all.numel() * 4 + res_all.numel() + hist_host.nbytes
        if timing:
            for e_a, e_b in asm_ev:
                self.phase["assembly_ms"] += e_a.elapsed_time(e_b)
        for idx, k, omega, e0, e1, sem_cols, share, first in ev:
            if flags[idx, 0]:
                raise SweepError(f"frequency index {k} (omega={omega:.6g}): non-finite entries "
                                 f"assembled at omega = {omega}")
            if flags[idx, 1]:
                log.warning("%d singular 3x3 diagonal blocks; identity fallback", flags[idx, 1])
            out = _lib.GmresResult.from_buffer_copy(res_host[idx, :32].tobytes())
            st = SolveStats(k=k, omega=omega, iterations=out.iterations,
                            init_residual=out.init_residual, final_residual=out.final_residual,
                            converged=bool(out.converged), matvecs=out.matvecs)
            nh = min(out.n_hist, cap)
            st.residual_history = hist_host[idx, :nh].tolist() if nh else []
            if not st.converged:
                log.warning("GMRES stalled at residual %.3e after %d iterations (k=%d)",
                            st.final_residual, st.iterations, k)
            st.seconds = e0.elapsed_time(e1) * 1e-3 / share   # concurrent group: its mean
            stats[k] = st
            if timing:
                if first:
                    self.phase["solve_ms"] += e0.elapsed_time(e1)
            # passes over A: the solver's own count + SEM's Y = A X pass(es)
            self.phase["matvecs"] += st.matvecs + (n_hist_passes(sem_cols) if sem_cols else 0)
            self.phase["solves"] += 1
        # host-side split (enqueue / wait for the device / result processing)
        self.phase["host_enqueue_ms"] = (t_host1 - t_host0) * 1e3
        self.phase["host_wait_ms"] = (t_host2 - t_host1) * 1e3
        self.phase["host_post_ms"] = (time.perf_counter() - t_host2) * 1e3
        return stats

    def probe_half(self, probes):
        import torch

        cols = []
        for p in probes:
            unknown = (self.kinds[p.dof] == NEUMANN) if p.quantity == "displacement" else \
                (self.kinds[p.dof] == DIRICHLET)
            cols.append(self.sol[:, p.dof] if unknown else self.P[:, p.dof])
        if not cols:
            return torch.zeros((self.n_freq, 0), dtype=torch.complex128, device="cuda")
        return torch.stack(cols, dim=1).contiguous()

    def displacement_field(self):
        """u for every DOF at every frequency: (n_freq, n) device."""
        import torch

        neu = torch.from_numpy(self.kinds == NEUMANN).cuda()
        return torch.where(neu[None, :], self.sol, self.P)


def run_sweep(cfg, full_field: bool = False, assembler: Assembler | None = None,
              distributed: bool = True, _sweep_out: list | None = None,
              matrix_free: bool | None = None) -> SweepResult:
    """Run the transient analysis described by ``cfg`` on the GPU.

    ``matrix_free=None`` picks the matrix-free operator automatically when the
    dense (N, N) complex matrix would not fit comfortably in HBM (> 40 % of
    the free device memory)."""
    import torch

    t_begin = time.perf_counter()
    dist = _dist() if distributed else None
    world = dist.get_world_size() if dist else 1
    rank = dist.get_rank() if dist else 0
    parallel = world > 1 and not cfg.sem_enabled
    if world > 1 and cfg.sem_enabled:
        log.info("solution extrapolation is sequential; every rank runs the whole sweep")
    eta = eta_from_kappa(cfg.kappa, cfg.period)
    n_freq = cfg.n_omega // 2 + 1
    mine = shard_frequencies(n_freq, rank, world) if parallel else None
    ds = DeviceSweep(cfg, assembler, mine)
    if matrix_free is None:
        free, _ = torch.cuda.mem_get_info()
        matrix_free = 16.0 * cfg.mesh.n_dofs ** 2 > 0.4 * free
    ds.matrix_free = bool(matrix_free)
    log.info("sweep: %d elements, %d frequencies, eta=%.4g 1/s", cfg.mesh.n_elements, n_freq, eta)
    stats_local = ds.run()
    probes = list(cfg.probes)
    probe_half = ds.probe_half(probes)
    stats_list = [None] * n_freq
    if parallel:
        local = {k: (probe_half[k].cpu().numpy(),
                     (stats_local[k].iterations, stats_local[k].init_residual,
                      stats_local[k].final_residual, stats_local[k].seconds,
                      float(stats_local[k].converged), 0.0)) for k in ds.frequencies}
        vals, meta = gather_frequency_results(local, n_freq, len(probes), dist)
        probe_half = torch.from_numpy(vals).cuda()
        for k in range(n_freq):
            it, i0, f0, sec, conv, _ = meta[k]
            stats_list[k] = SolveStats(k=k, omega=complex(ds.omegas[k]), iterations=int(it),
                                       init_residual=float(i0), final_residual=float(f0),
                                       seconds=float(sec), converged=bool(conv))
    else:
        for k in ds.frequencies:
            stats_list[k] = stats_local[k]
    failed = [s.k for s in stats_list if not s.converged]
    if failed:
        log.error("non-converged frequencies: %s", failed)
    times = np.arange(cfg.n_omega) * (cfg.period / cfg.n_omega)
    histories, half_spectra = {}, {}
    if probes:
        series, residue = windowed_inverse_device(probe_half, cfg.window, eta, cfg.period)
        series_h = series.cpu().numpy()
        residue_h = residue.cpu().numpy()
        half_h = probe_half.cpu().numpy()
        ds.d2h_bytes += series_h.nbytes + residue_h.nbytes + half_h.nbytes
        for i, p in enumerate(probes):
            half_spectra[p.name] = half_h[:, i].copy()
            check_residue(float(residue_h[i]))
            s = series_h[:, i].copy()
            histories[p.name] = np.full_like(s, np.nan) if failed else s
    field_hist = None
    if full_field:
        field_hist, _ = windowed_inverse_device(ds.displacement_field(), cfg.window, eta,
                                                cfg.period)
    manifest = build_manifest(cfg, eta, time.perf_counter() - t_begin, failed)
    if _sweep_out is not None:
        _sweep_out.append(ds)
    return SweepResult(times=times, histories=histories, half_spectra=half_spectra,
                       stats=stats_list, manifest=manifest, failed_frequencies=failed,
                       full_field=field_hist)


def build_manifest(cfg, eta: float, seconds: float, failed: list) -> dict:
    """driver.py:179-201."""
    dw = 2.0 * math.pi / cfg.period
    return {
        "n_elements": cfg.mesh.n_elements, "n_dofs": cfg.mesh.n_dofs, "period": cfg.period,
        "n_omega": cfg.n_omega, "delta_t": cfg.period / cfg.n_omega, "delta_omega": dw,
        "kappa": cfg.kappa, "eta": eta, "f_nyquist": cfg.n_omega * dw / (4.0 * math.pi),
        "window": cfg.window, "sem_enabled": cfg.sem_enabled, "sem_depth": cfg.sem_depth,
        "gmres_tol": cfg.tol, "gmres_restart": cfg.restart, "workers": cfg.workers,
        "elapsed_seconds": seconds, "failed_frequencies": failed,
    }


def emit_outputs(result: SweepResult, cfg) -> dict:
    """history_<probe>.csv, solve_stats.csv, manifest.txt (driver.py:248-283)."""
    out = Path(cfg.output_dir)
    out.mkdir(parents=True, exist_ok=True)
    written = {}
    for name, series in result.histories.items():
        path = out / f"history_{name}.csv"
        with path.open("w", encoding="ascii") as fh:
            fh.write("t,value\n")
            for t, v in zip(result.times, series):
                fh.write(f"{float(t)!r},{float(v)!r}\n")
        written[f"history_{name}"] = path
    path = out / "solve_stats.csv"
    with path.open("w", encoding="ascii") as fh:
        fh.write(SolveStats.CSV_HEADER + "\n")
        for s in result.stats:
            fh.write(s.csv_row() + "\n")
    written["solve_stats"] = path
    path = out / "manifest.txt"
    with path.open("w", encoding="ascii") as fh:
        for key, value in result.manifest.items():
            fh.write(f"{key} = {value}\n")
        fh.write("# config echo\n")
        for key, value in cfg.raw:
            fh.write(f"config.{key} = {value}\n")
    written["manifest"] = path
    return written
