"""Frequency sweep on one B200 (mirror of reference ``driver.py:92-176``).

``run_sweep(cfg) -> SweepResult`` keeps the reference's sequencing exactly
(ascending k, SEM history pushed after each solve, probes, NaN poisoning of
every history when any solve fails, manifest) while every per-frequency
array stays in HBM:

    per k:  ewb_assemble_system   (assembly + BCs + b + P^{-1}, no T/U)
            ewb_sem_guess         (if history: Y = A X, QR, x0)
            ewb_gmres             (the whole restarted solve, one launch)
            one 64-byte read-back (flags + iteration count + residuals)
    end:    ewb_window_idft       (conjugate fill + window + IDFT for the
                                   probe columns, or all DOFs)

With SEM off and torch.distributed initialised with world > 1, the
frequencies are dealt round-robin to the ranks (the reference's fork pool,
driver.py:113-122, as replicas over NVLink-connected GPUs) and the
per-frequency results are all-gathered once at the end.
"""

from __future__ import annotations

import ctypes
import logging
import math
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from .assembly import DIRICHLET, NEUMANN, Assembler
from .config import SweepConfig
from .linsolve import SolveStats, _SEM_WS, _WS, gmres_device, sem_device
from .transform import (check_residue, eta_from_kappa, forward_mft, frequency_grid,
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
    """All-gather {k: (values (width,) complex, stats tuple)} from every rank.

    Returns (values (n_freq, width) complex ndarray, stats list indexed by k).
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
        vals = total[:, :w2].copy().view(complex)
        meta = total[:, w2:w2 + 6]
        owned = total[:, -1]
    if not np.all(owned == 1):
        raise SweepError("frequency ownership is not a partition of the sweep")
    return vals, meta


def run_sweep(cfg: SweepConfig, full_field: bool = False, assembler: Assembler | None = None,
              distributed: bool = True) -> SweepResult:
    """Run the transient analysis described by ``cfg`` on the GPU."""
    import torch

    t_begin = time.perf_counter()
    _lib.require_cuda()
    eta = eta_from_kappa(cfg.kappa, cfg.period)
    omegas = frequency_grid(cfg.period, cfg.n_omega, eta)
    n_freq = len(omegas)
    log.info("sweep: %d elements, %d frequencies, eta=%.4g 1/s", cfg.mesh.n_elements, n_freq, eta)
    spectra = np.stack([forward_mft(s, cfg.period, cfg.n_omega, eta).values[:n_freq]
                        for s in cfg.signals])
    asm = assembler or Assembler(cfg.mesh, cfg.material)
    n = cfg.mesh.n_dofs
    kinds = np.ascontiguousarray(cfg.bcs.flat_kind(), dtype=np.uint8)
    sig = cfg.bcs.flat_signal()
    # prescribed values for every k, on the device: P[k, d] = spectra[sig[d], k]
    spec_dev = torch.from_numpy(np.ascontiguousarray(spectra.T)).cuda()      # (n_freq, n_sig)
    P = spec_dev[:, torch.from_numpy(sig.astype(np.int64)).cuda()].contiguous()  # (n_freq, n)

    dist = _dist() if distributed else None
    world = dist.get_world_size() if dist else 1
    rank = dist.get_rank() if dist else 0
    parallel = world > 1 and not cfg.sem_enabled
    if world > 1 and cfg.sem_enabled:
        log.info("solution extrapolation is sequential; every rank runs the whole sweep")
    my_k = shard_frequencies(n_freq, rank, world) if parallel else list(range(n_freq))

    sol = torch.zeros((n_freq, n), dtype=torch.complex128, device="cuda")
    x = torch.zeros(n, dtype=torch.complex128, device="cuda")
    K = cfg.sem_depth
    hist = torch.zeros((K, n), dtype=torch.complex128, device="cuda")
    n_hist = 0
    system = None
    stats_local = {}
    res_host = torch.empty(64, dtype=torch.uint8).pin_memory()
    ev = []
    for k in my_k:
        omega = complex(omegas[k])
        try:
            system = asm.assemble_system(omega, cfg.bcs, P[k], out=system if omega != 0 else None,
                                         check=False)
            if system.pinv is None:   # omega == 0 static path (kappa = 0)
                from .linsolve import block_diag_precond

                system.pinv = block_diag_precond(system.A).pinv
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            use_sem = cfg.sem_enabled and n_hist > 0
            if use_sem:
                sem_device(system.A, system.b, hist[:n_hist], 1e-10, x)
            st = SolveStats()
            gmres_device(system.A, system.b, x, use_sem, cfg.tol, cfg.restart, cfg.maxiter,
                         system.pinv, stats=st, sync=False)
            e1.record()
            # one read-back per frequency: fault flags + solver record
            nf = ctypes.c_int32()
            sg = ctypes.c_int32()
            _lib.check(asm._lib.ewb_ctx_flags(asm.ctx, ctypes.byref(nf), ctypes.byref(sg),
                                              _lib.stream_handle()))
            if nf.value:
                raise FloatingPointError(f"non-finite entries assembled at omega = {omega}")
            if sg.value:
                log.warning("%d singular 3x3 diagonal blocks; identity fallback", sg.value)
            from .linsolve import _fill_stats

            _fill_stats(st, _WS.result(), _WS.hist_buf(1))
        except SweepError:
            raise
        except Exception as exc:
            raise SweepError(f"frequency index {k} (omega={omega:.6g}): {exc}") from exc
        st.k = k
        st.omega = omega
        stats_local[k] = st
        ev.append((k, e0, e1))
        sol[k] = x
        if cfg.sem_enabled:
            hist[1:] = hist[:-1].clone()
            hist[0] = x
            n_hist = min(n_hist + 1, K)
        if not st.converged:
            log.warning("GMRES stalled at residual %.3e after %d iterations",
                        st.final_residual, st.iterations)
        log.debug("k=%3d iters=%4d res=%.2e", k, st.iterations, st.final_residual)
    torch.cuda.synchronize()
    for k, e0, e1 in ev:
        stats_local[k].seconds = e0.elapsed_time(e1) * 1e-3

    # probe spectra: u = a (Neumann) else prescribed; t = a (Dirichlet) else prescribed
    probes = list(cfg.probes)
    cols = []
    for p in probes:
        unknown = (kinds[p.dof] == NEUMANN) if p.quantity == "displacement" else \
            (kinds[p.dof] == DIRICHLET)
        cols.append((p.dof, bool(unknown)))
    probe_half = torch.stack([sol[:, d] if unk else P[:, d] for d, unk in cols], dim=1) \
        if cols else torch.zeros((n_freq, 0), dtype=torch.complex128, device="cuda")

    stats_list = [None] * n_freq
    if parallel:
        local = {k: (probe_half[k].cpu().numpy(),
                     (stats_local[k].iterations, stats_local[k].init_residual,
                      stats_local[k].final_residual, stats_local[k].seconds,
                      float(stats_local[k].converged), 0.0)) for k in my_k}
        vals, meta = gather_frequency_results(local, n_freq, len(probes), dist)
        probe_half = torch.from_numpy(vals).cuda()
        for k in range(n_freq):
            it, i0, f0, sec, conv, _ = meta[k]
            stats_list[k] = SolveStats(k=k, omega=complex(omegas[k]), iterations=int(it),
                                       init_residual=float(i0), final_residual=float(f0),
                                       seconds=float(sec), converged=bool(conv))
    else:
        for k in my_k:
            stats_list[k] = stats_local[k]

    failed = [s.k for s in stats_list if not s.converged]
    if failed:
        log.error("non-converged frequencies: %s", failed)
    dt = cfg.period / cfg.n_omega
    times = np.arange(cfg.n_omega) * dt
    histories, half_spectra = {}, {}
    if probes:
        series, residue = windowed_inverse_device(probe_half, cfg.window, eta, cfg.period)
        series_h = series.cpu().numpy()
        residue_h = residue.cpu().numpy()
        half_h = probe_half.cpu().numpy()
        for i, p in enumerate(probes):
            half_spectra[p.name] = half_h[:, i].copy()
            check_residue(float(residue_h[i]))
            s = series_h[:, i].copy()
            histories[p.name] = np.full_like(s, np.nan) if failed else s
    field_hist = None
    if full_field:
        # u for every DOF (displacement field), all on the device
        neu = torch.from_numpy(kinds == NEUMANN).cuda()
        u_half = torch.where(neu[None, :], sol, P)
        field_hist, _ = windowed_inverse_device(u_half, cfg.window, eta, cfg.period)
    manifest = build_manifest(cfg, eta, time.perf_counter() - t_begin, failed)
    return SweepResult(times=times, histories=histories, half_spectra=half_spectra,
                       stats=stats_list, manifest=manifest, failed_frequencies=failed,
                       full_field=field_hist)


def build_manifest(cfg: SweepConfig, eta: float, seconds: float, failed: list) -> dict:
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


def emit_outputs(result: SweepResult, cfg: SweepConfig) -> dict:
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
