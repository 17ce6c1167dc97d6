#!/usr/bin/env python
"""Benchmark of the B200 per-frequency BEM solve (BASELINE.json metric/config).

Default workload = BASELINE configs[1] (cfg2): flipped icosphere L4, 5120
triangles / 15360 complex DOF, unit-step cavity pressure, N_omega = 256 ->
129 sequential solves (SEM K = 4, GMRES tol 1e-8, restart 60).  One step =
one full sweep through the device path (assembly + BCs + preconditioner +
SEM + GMRES for all 129 frequencies + windowed IDFT of the probes) with the
mesh context and the per-run inputs already resident in HBM.  Metric: s per
sweep (lower is better).  `e2e` is the same sweep through the public API
`run_sweep(cfg)` from host arrays (context creation, host->device uploads
and the device->host read-back of histories/stats included).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg1|cfg3|cfg4]

`--impl reference` times the reference algorithm on the host CPU (the numpy
oracle port under oracle/, since the Python reference cannot travel to the
GPU box), on every host core (oracle/parallel.py): the chained sweep from
k = 0, one complete frequency per step; the s/sweep value is measured setup
+ n_freq x the mean measured frequency.
Multi-GPU (torchrun): SEM makes the sweep sequential, so N ranks run N
replica sweeps (scaling "weak"); time = max over ranks of CUDA-event time.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "s per sweep"
BASELINE_METRIC = ("element-pair kernel evals/s (FP64 % peak); complex matvec HBM GB/s; "
                   "s per sweep")


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="cfg2", choices=("cfg2", "cfg1", "cfg3", "cfg4", "cfg5"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the cfg5 matrix-free block")
    return ap.parse_args(argv)


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ----------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "500"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        busy = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "fallback": True}


# ----------------------------------------------------------------------
# CPU side: the reference algorithm (numpy oracle port), bounded sample
# ----------------------------------------------------------------------
def host_info() -> dict:
    """CPU model, core count, numpy BLAS and thread settings of the host the
    CPU baseline ran on (report them beside the number)."""
    import numpy as np

    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = ""
    try:
        b = np.show_config(mode="dicts")["Build Dependencies"]["blas"]
        blas = f"{b.get('name', '')} {b.get('version', '')}".strip()
    except Exception:
        pass
    threads = {k: os.environ[k] for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                           "MKL_NUM_THREADS") if k in os.environ}
    return {"cpu_model": model, "nproc": os.cpu_count(), "numpy": np.__version__,
            "blas": blas, "thread_env": threads}


def oracle_inputs(cfg) -> dict:
    """The sweep inputs of ``cfg`` as the oracle's plain arrays."""
    from oracle import ewbem_oracle as O

    m = cfg.mesh
    return dict(vertices=m.vertices, triangles=m.triangles,
                med=O.Medium(cfg.material.lam, cfg.material.mu, cfg.material.rho),
                kinds=cfg.bcs.flat_kind(), dof_signal=cfg.bcs.flat_signal(),
                signal_samples=[np.asarray(s.sample(cfg.period, cfg.n_omega), float)
                                for s in cfg.signals],
                period=cfg.period, n_omega=cfg.n_omega, kappa=cfg.kappa,
                sem_depth=cfg.sem_depth, sem=cfg.sem_enabled, tol=cfg.tol,
                restart=cfg.restart, maxiter=cfg.maxiter)


def cpu_chained(cfg, n_freq=None):
    """MEASURED: the reference algorithm (oracle port, every host core) runs
    the chained sweep of ``cfg`` for k = 0..n_freq-1 (None = the whole sweep):
    geometry prep + static pass, then per frequency assembly, apply_bcs, SEM,
    block preconditioner and GMRES (driver.py:92-176)."""
    from oracle.parallel import sweep_seconds

    return sweep_seconds(oracle_inputs(cfg), frequencies=n_freq)


# ----------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------
def fp64_peak():
    import ctypes

    from paper_1212_3032_b200 import _lib

    lib = _lib.load()
    tf, ms = ctypes.c_double(), ctypes.c_double()
    best = 0.0
    for _ in range(3):
        _lib.check(lib.ewb_fp64_peak_probe(20000, 4, ctypes.byref(tf), ctypes.byref(ms),
                                           _lib.stream_handle()))
        best = max(best, tf.value)
    return best


TRAFFIC_FILE = ROOT / "profiles" / "traffic.json"


# k_far_multi<true, false>, Neumann path, per (pair, member) of the member loop
# and per point of the per-row set-up (tools/sass_loops.py, round-2 final build)
FAR_FP64_PER_PAIR_MEMBER = 444.0       # DFMA 306 + DMUL 105 + DADD 33
FAR_FLOPS_PER_PAIR_MEMBER = 2 * 306.0 + 105.0 + 33.0
FAR_FP64_SETUP_PER_POINT = 175.0       # geometry, 4 sincos + 2 exp (about 1.6 flop each)


def traffic_record(workload: str) -> dict | None:
    """ncu dram read+write per launch unit, keyed by workload (profiles/traffic.json)."""
    if not TRAFFIC_FILE.exists():
        return None
    return json.loads(TRAFFIC_FILE.read_text()).get(workload)


def cpu_baseline_block(workload: str, cfg, n_freq: int) -> dict:
    """``cpu_baseline`` of our arm: MEASURED runs of the reference algorithm
    (oracle port) on this host, every core.  cfg1: the whole 65-frequency
    sweep.  cfg2: setup + the first two complete chained frequencies (k = 0
    without and k = 1 with SEM); the s/sweep value is derived from them as
    setup + 129 x mean per frequency and labelled so."""
    from paper_1212_3032_b200 import workloads

    host = host_info()
    if workload == "cfg1":
        m = cpu_chained(cfg)
        total = m["setup_s"] + sum(m["per_freq_s"])
        return {"value": round(total, 2), "unit": "s/sweep", "cores": m["workers"],
                "kind": "port", "measured": True,
                "sample": f"the whole cfg1 sweep ({len(m['per_freq_s'])} frequencies), measured",
                "iterations_total": int(sum(m["its"])), "setup_s": round(m["setup_s"], 2),
                "host": host}
    m2 = cpu_chained(cfg, 2)
    per = statistics.mean(m2["per_freq_s"])
    value = m2["setup_s"] + n_freq * per
    m1 = cpu_chained(workloads.cfg1())
    return {"value": round(value, 1), "unit": "s/sweep", "cores": m2["workers"], "kind": "port",
            "measured": False,
            "sample": ("cfg2 setup (geometry prep + static pass) and the first 2 complete chained "
                       "frequencies (assembly, apply_bcs, SEM, preconditioner, GMRES) measured; "
                       f"value = setup + {n_freq} x mean measured frequency"),
            "measured_parts": {"cfg2_setup_s": round(m2["setup_s"], 2),
                               "cfg2_prep_s": round(m2["prep_s"], 2),
                               "cfg2_static_s": round(m2["static_s"], 2),
                               "cfg2_per_freq_s": [round(t, 2) for t in m2["per_freq_s"]],
                               "cfg2_its": m2["its"],
                               "cfg2_freq_parts": [{k: round(v, 3) for k, v in p.items()}
                                                   for p in m2["parts"]],
                               "cfg1_full_sweep_s": round(m1["setup_s"] + sum(m1["per_freq_s"]), 2),
                               "cfg1_frequencies": len(m1["per_freq_s"]),
                               "cfg1_iterations_total": int(sum(m1["its"]))},
            "host": host}


def build_cfg(workload: str):
    from paper_1212_3032_b200 import workloads

    if workload == "cfg1":
        return workloads.cfg1(), ("cfg1: unit cube 768 el / 2304 DOF, z- clamped, z+ unit step "
                                  "traction, N_omega=128 -> 65 solves, SEM K=2, tol 1e-8")
    return workloads.cfg2(), ("cfg2: flipped icosphere L4 5120 el / 15360 DOF, unit step "
                              "cavity pressure, N_omega=256 -> 129 solves, SEM K=4, tol 1e-8, "
                              "restart 60")


def run_ours_sweep(args, rank, world, local_rank):
    import torch

    from paper_1212_3032_b200 import _lib, run_sweep
    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.transform import windowed_inverse_device

    lib = _lib.require_cuda()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    cfg, desc = build_cfg(args.workload)
    peak64 = fp64_peak()

    t0 = time.perf_counter()
    ds = DeviceSweep(cfg)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    counts = ds.asm.pair_counts()
    pe = ds.asm.point_evals()
    n_pairs = counts["far"] + counts["mid"] + counts["near"] + counts["n_elements"]
    flops_per_asm = 397.0 * pe + 120.0 * n_pairs        # SURVEY §8(d) algorithmic count

    host_parts = []

    def one_step():
        t0 = time.perf_counter()
        ds.run(timing=True)
        t1 = time.perf_counter()
        half = ds.probe_half(cfg.probes)
        t2 = time.perf_counter()
        windowed_inverse_device(half, cfg.window, ds.eta, cfg.period)
        t3 = time.perf_counter()
        host_parts.append([round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1),
                           round((t3 - t2) * 1e3, 1)])

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    # host: move the long-lived objects out of the collector's generations so
    # a full GC pass cannot stall the enqueueing thread inside the timed steps
    gc.collect()
    gc.freeze()
    if dist:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    launches0 = lib.ewb_launch_count()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    asm_ms = solve_ms = 0.0
    matvecs = 0
    its = 0
    nfreq = 0
    step_marks, host_split = [], []
    if os.environ.get("BENCH_GC_DISABLE") == "1":
        gc.disable()
    for _ in range(args.steps):
        th0 = time.perf_counter()
        one_step()
        host_split.append([round(ds.phase.get(k, 0.0), 1) for k in
                           ("host_enqueue_ms", "host_wait_ms", "host_post_ms")]
                          + [round((time.perf_counter() - th0) * 1e3, 1)])
        mk = torch.cuda.Event(enable_timing=True)
        mk.record()
        step_marks.append(mk)
        asm_ms += ds.phase["assembly_ms"]
        solve_ms += ds.phase["solve_ms"]
        matvecs += ds.phase["matvecs"]
        nfreq += ds.phase["solves"]
    stop.record()
    torch.cuda.synchronize()
    launches = lib.ewb_launch_count() - launches0
    gc.enable()
    clocks = sampler.stop()
    elapsed_ms = start.elapsed_time(stop)
    step_ms, prev = [], start
    for mk in step_marks:
        step_ms.append(round(prev.elapsed_time(mk), 2))
        prev = mk
    if dist:
        t = torch.tensor([elapsed_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
        dist.barrier()
    ms_per_step = elapsed_ms / args.steps
    value = (elapsed_ms / 1e3) / (args.steps * world)   # s per sweep, whole job
    # per-frequency assembly: FP64 roofline;  solve phase: HBM roofline
    n = ds.n
    asm_per_freq_ms = asm_ms / max(nfreq, 1)
    asm_tflops = flops_per_asm / (asm_per_freq_ms * 1e-3) / 1e12
    bytes_per_pass = 16.0 * n * n + 32.0 * n
    solve_gbs = matvecs * bytes_per_pass / (solve_ms * 1e-3) / 1e9
    peaks = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    pair_evals_per_s = (counts["far"] + counts["mid"] + counts["near"] + counts["n_elements"]) / \
        (asm_per_freq_ms * 1e-3)
    rl_asm = {"bound": "fp64",
              "kernel": "multi-frequency assembly (k_far_multi+k_mid_multi+k_near_multi+"
                        "k_self_multi, %d frequencies per pass, fused BCs)" % ds.batch_size(),
              "achieved": round(asm_tflops, 3), "peak": round(peak64, 3), "unit": "TFLOP/s",
              "frac": round(asm_tflops / peak64, 4),
              "peak_source": "measured DFMA probe in this run (MEASURED_PEAKS.json has no FP64)",
              "traffic": None, "algorithmic_flops_per_launch": flops_per_asm,
              "ms_per_launch": round(asm_per_freq_ms, 4)}
    rl_solve = {"bound": "hbm", "kernel": "k_gmres + k_sem (persistent, dense matvec)",
                "achieved": round(solve_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(solve_gbs / hbm_peak, 4),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)", "traffic": None,
                "algorithmic_bytes_per_pass": bytes_per_pass,
                "passes_per_sweep": matvecs / max(args.steps, 1)}
    if bytes_per_pass < 120e6:
        rl_solve["note"] = ("A = %.0f MB fits the 126 MB L2: a pass is bound by the per-step "
                            "latencies (TMA round trips of a %d-row CTA share, 3 grid barriers, "
                            "the Arnoldi reductions), not by HBM; the fraction is reported "
                            "against the HBM copy peak for continuity only"
                            % (bytes_per_pass / 1e6, -(-n // 148)))
    # DRAM traffic of the dominant kernels from the committed ncu capture of
    # THIS workload (null when none was captured for it)
    tr = traffic_record(args.workload)
    if tr:
        for key, rl in (("solve", rl_solve), ("assembly", rl_asm)):
            if key in tr:
                rl["traffic"] = tr[key]["bytes"]
                rl["traffic_unit"] = tr[key]["unit"]
                rl["traffic_source"] = tr[key]["source"]
    asm_share = asm_ms / max(asm_ms + solve_ms, 1e-9)
    # the same multi-frequency assembly outside the sweep (clocks not pulled
    # down by the power-capped GMRES phase): one batch of mid-sweep members
    nb = ds.batch_size()
    k0 = max(0, min(ds.n_freq - nb, ds.n_freq // 2 - nb // 2))
    ks = list(range(k0, k0 + nb))
    sa_ms = []
    for rep in range(3):
        e_s, e_t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_s.record()
        ds.batch = ds.asm.assemble_system_multi([ds.omegas[k] for k in ks], cfg.bcs,
                                                ds.P[k0:k0 + nb], out=ds.batch, check=False)
        e_t.record()
        torch.cuda.synchronize()
        if rep:
            sa_ms.append(e_s.elapsed_time(e_t) / nb)
    sa_per_freq = statistics.median(sa_ms)
    sa_tf = flops_per_asm / (sa_per_freq * 1e-3) / 1e12
    rl_asm["standalone"] = {"ms_per_freq": round(sa_per_freq, 4), "achieved": round(sa_tf, 3),
                            "frac": round(sa_tf / peak64, 4),
                            "batch": f"k = {k0}..{k0 + nb - 1} in one pass, outside the sweep"}
    # Executed (not algorithmic) FP64 work of the far-pair kernel, from its SASS
    # (tools/sass_loops.py on k_far_multi<RECUR, !SER>, Neumann path): the
    # member loop issues FAR_FP64 FP64 instructions per (pair, member) — DFMA
    # 306, DMUL 105, DADD 33 — plus 175 per point of per-row set-up shared by
    # the batch.  Every FP64 instruction occupies the pipe alike, so
    # instructions / (time x peak DFMA rate) is the pipe fraction ncu reports.
    far_instr = FAR_FP64_PER_PAIR_MEMBER + 3.0 * FAR_FP64_SETUP_PER_POINT / nb
    far_flops = FAR_FLOPS_PER_PAIR_MEMBER + 3.0 * FAR_FP64_SETUP_PER_POINT * 1.6 / nb
    dfma_rate = peak64 * 1e12 / 2.0                      # FP64 instructions / s at peak
    rl_asm["executed"] = {
        "scope": "far pairs only (k_far_multi: %.1f %% of the point evaluations)"
                 % (100.0 * 3.0 * counts["far"] / pe),
        "fp64_instr_per_far_pair_member": round(far_instr, 1),
        "flops_per_far_pair_member": round(far_flops, 1),
        "algorithmic_flops_per_far_pair": 3 * 397 + 120,
        "pipe_frac_standalone": round(counts["far"] * far_instr / (sa_per_freq * 1e-3) / dfma_rate, 4),
        "pipe_frac_in_sweep": round(counts["far"] * far_instr / (asm_per_freq_ms * 1e-3) / dfma_rate, 4),
        "flop_frac_standalone": round(counts["far"] * far_flops / (sa_per_freq * 1e-3) / 1e12 / peak64, 4),
        "note": "far-pair instructions over the WHOLE assembly time (mid / near / self kernels "
                "included in the time, not in the instructions): a lower bound on k_far_multi's "
                "own FP64 pipe fraction (ncu: 57.5 % active); the phase recurrence removed the "
                "transcendentals the algorithmic count credits",
        "source": "static SASS count of the member loop (tools/sass_loops.py), "
                  "profiles/r02/SUMMARY.md"}
    rl_asm["note"] = ("in-sweep figure: assembly runs between power-capped GMRES phases "
                      "(sw_power_cap, lower SM clocks); standalone: the same kernels alone")
    if clocks.get("sm_mhz") and clocks.get("sm_max_mhz"):
        # the DFMA peak scales with the SM clock: the in-sweep rate against the
        # peak AT the median clock sampled under load (not a measured peak)
        scale = clocks["sm_max_mhz"] / clocks["sm_mhz"]
        rl_asm["frac_at_sampled_clock"] = round(asm_tflops / peak64 * scale, 4)
        rl_asm["sampled_sm_mhz"] = clocks["sm_mhz"]
    roof, roof2 = (rl_asm, rl_solve) if asm_share >= 0.5 else (rl_solve, rl_asm)

    # e2e through the public API from host arrays
    e2e_times, h2d, d2h = [], 0, 0
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        keep = []
        t1 = time.perf_counter()
        res = run_sweep(cfg, _sweep_out=keep, distributed=False)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t1)
        h2d, d2h = keep[0].h2d_bytes, keep[0].d2h_bytes
    e2e_s = statistics.median(e2e_times)
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    total_its = res.total_iterations

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_block(args.workload, cfg, ds.n_freq)
    cfg5_block = other_metrics = None
    if rank == 0 and world == 1 and args.workload == "cfg2" and not args.no_cfg5:
        del ds
        gc.collect()
        torch.cuda.empty_cache()
        from benchmarks import micro

        cfg5_block = micro.cfg5_measure(steps=3, warmup=1, peak64=peak64)
        # the other two metrics BASELINE.json names, on their own configs
        other_metrics = {"cfg3_pair_kernels": micro.cfg3_measure(3, 2, peak64),
                         "cfg4_gemv": micro.cfg4_gemv_measure()}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "s/sweep", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (reference-generated mesh + unit step load, BASELINE %s)"
                     % args.workload),
            "config": {"workload": desc, "baseline_metric": BASELINE_METRIC,
                       "l2": "inputs larger than L2 (A = 16 N^2 = %.2f GB)" % (16 * n * n / 1e9),
                       "parallelism": "replicas" if world > 1 else "single GPU"},
            "roofline": roof, "roofline_secondary": roof2,
            "cpu_baseline": cpu,
            "cfg5_matrix_free": cfg5_block,
            "baseline_metrics_other_configs": other_metrics,
            "e2e": {"value": e2e_s / world, "unit": "s/sweep", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clocks,
            "metrics": {"element_pair_evals_per_s": pair_evals_per_s,
                        "point_evals_per_assembly": pe, "assembly_ms_per_freq": asm_per_freq_ms,
                        "assembly_share": round(asm_share, 4),
                        "solve_ms_per_sweep": solve_ms / args.steps,
                        "matvec_hbm_gbs_solve_phase": solve_gbs,
                        "total_gmres_iterations": total_its, "setup_ms": setup_s * 1e3,
                        "step_ms": step_ms,
                        "host_enqueue_wait_post_step_ms": host_split,
                        "host_run_probe_idft_ms": host_parts[-args.steps:],
                        "fp64_peak_tflops_measured": peak64},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_reference(args, rank, world):
    """The reference algorithm on the host CPU (oracle port, every core), rank 0
    only: the chained sweep from k = 0, one complete frequency per step
    (assembly, apply_bcs, SEM, preconditioner, GMRES); W warm-up frequencies,
    then K timed ones.  value = measured setup + n_freq x mean timed frequency."""
    if rank != 0:
        return
    cfg, desc = build_cfg(args.workload)
    nf = cfg.n_omega // 2 + 1
    m = cpu_chained(cfg, min(nf, args.warmup + args.steps))
    timed = m["per_freq_s"][args.warmup:] or m["per_freq_s"]
    per = statistics.mean(timed)
    value = m["setup_s"] + nf * per
    sample = (f"setup + frequencies k = 0..{len(m['per_freq_s']) - 1} of the chained sweep "
              f"measured ({len(timed)} timed after {args.warmup} warm-up); value = setup + "
              f"{nf} x mean timed frequency")
    line = {"metric": METRIC, "value": value, "unit": "s/sweep", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "step": "one complete frequency of the chained sweep (CPU)",
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": desc, "baseline_metric": BASELINE_METRIC},
            "cpu_baseline": {"value": value, "unit": "s/sweep", "cores": m["workers"],
                             "kind": "port", "sample": sample, "measured_setup_s": m["setup_s"],
                             "measured_per_freq_s": m["per_freq_s"], "its": m["its"],
                             "host": host_info()},
            "e2e": {"value": value, "unit": "s/sweep", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main(argv=None):
    args = parse_args(argv)
    rank, world, local_rank = env_rank()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.workload in ("cfg1", "cfg2"):
        run_ours_sweep(args, rank, world, local_rank)
    else:
        from benchmarks import micro

        micro.main(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
