"""Secondary BASELINE workloads for bench.py (--workload cfg3 | cfg4).

cfg3  pair-kernel microbenchmark: 2^14 points x 2^14 random triangles x 16
      complex frequencies omega_r - 2i, gauss7 on every pair, fused reduction
      y(omega) = sum_j [U_ij; T_ij] x_j (ewb_pair_kernels_reduce).
      Metric: element-pair kernel evals/s; FP64 roofline with the SURVEY §8(d)
      algorithmic count 25*7/16 + 372*7 + 120 = 2,735 flop per pair-frequency.
cfg4  batched dense complex matvec: 8 systems of N = 4096 / 8192 / 16384,
      A = (G + iG')/sqrt2 + 3 sqrt(N) I (seeded, generated on the device),
      one TMA-streamed pass over all 8 matrices per launch
      (ewb_gemv_batched).  Metric: complex matvec HBM GB/s (16 N^2 bytes per
      matrix); plus the restart-50, tol-1e-8 GMRES solve of each system.
"""

from __future__ import annotations

import ctypes
import json
import math
import statistics
import time

import numpy as np

PAIR_FLOPS = 25.0 * 7 / 16 + 372.0 * 7 + 120.0


def _peaks():
    import bench

    return bench.measured_peaks()


def cfg3_measure(steps: int, warmup: int, peak64: float) -> dict:
    """cfg3 pair kernels (2^14 x 2^14 x 16, fused U/T reduction), CUDA events."""
    import torch

    from paper_1212_3032_b200 import _lib
    from paper_1212_3032_b200.workloads import UNIT, cfg3_inputs

    lib = _lib.require_cuda()
    x, tris, omegas, xv = cfg3_inputs()
    P, M, F = len(x), len(tris), len(omegas)
    xd = torch.from_numpy(x).cuda()
    td = torch.from_numpy(tris.reshape(M, 9).copy()).cuda()
    vd = torch.from_numpy(xv.copy()).cuda()
    om = np.ascontiguousarray(np.stack([omegas.real, omegas.imag], axis=1))
    yu = torch.empty((F, P, 3), dtype=torch.complex128, device="cuda")
    yt = torch.empty_like(yu)
    ws_bytes = int(lib.ewb_pair_kernels_workspace_bytes(P, M, F))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")

    def step():
        _lib.check(lib.ewb_pair_kernels_reduce(
            _lib.ptr(xd), P, _lib.ptr(td), M, _lib.ptr(vd), om.ctypes.data, F, UNIT.lam,
            UNIT.mu, UNIT.rho, _lib.ptr(yu), _lib.ptr(yt), _lib.ptr(ws), ws_bytes,
            _lib.stream_handle()))

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    evals = float(P) * M * F
    tf = evals / (ms * 1e-3) * PAIR_FLOPS / 1e12
    return {"workload": f"cfg3: {P} points x {M} triangles x {F} omega, gauss7, fused U/T "
                        "reduction", "metric": "element-pair kernel evals/s",
            "value": evals / (ms * 1e-3), "unit": "pair-evals/s", "ms_per_launch": ms,
            "roofline": {"bound": "fp64", "achieved": tf, "peak": peak64, "unit": "TFLOP/s",
                         "frac": tf / peak64, "algorithmic_flops_per_launch": evals * PAIR_FLOPS,
                         "peak_source": "measured DFMA probe"}}


def cfg4_gemv_measure(n: int = 16384, batch: int = 8, reps: int = 5) -> dict:
    """cfg4 batched complex128 GEMV (8 seeded diagonally dominant systems,
    device-generated), CUDA events; HBM roofline."""
    import torch

    from paper_1212_3032_b200 import _lib

    lib = _lib.require_cuda()
    hbm = float(_peaks().get("hbm_gbs", 6650.0))
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    A = torch.empty((batch, n, n), dtype=torch.complex128, device="cuda")
    for s_ in range(batch):
        A[s_] = torch.complex(torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64),
                              torch.randn((n, n), generator=g, device="cuda",
                                          dtype=torch.float64)) / math.sqrt(2.0)
        A[s_].diagonal().add_(3.0 * math.sqrt(n))
    b = torch.complex(torch.randn((batch, n), generator=g, device="cuda", dtype=torch.float64),
                      torch.randn((batch, n), generator=g, device="cuda", dtype=torch.float64))
    y = torch.empty_like(b)

    def step():
        _lib.check(lib.ewb_gemv_batched(_lib.ptr(A), _lib.ptr(b), _lib.ptr(y), n, batch,
                                        _lib.stream_handle()))

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    gbs = batch * (16.0 * n * n + 32.0 * n) / (ms * 1e-3) / 1e9
    ref = A[batch - 1] @ b[batch - 1]
    err = float((y[batch - 1] - ref).abs().max() / ref.abs().max())
    del A, b, y
    torch.cuda.empty_cache()
    return {"workload": f"cfg4: batched dense complex128 matvec, {batch} systems, N={n}",
            "metric": "complex matvec HBM GB/s", "value": gbs, "unit": "GB/s",
            "ms_per_launch": ms, "relerr_vs_torch": err,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                         "frac": gbs / hbm,
                         "algorithmic_bytes_per_launch": batch * (16.0 * n * n + 32.0 * n),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"}}


def run_cfg3(args, rank, world, local_rank):
    import torch

    import bench
    from paper_1212_3032_b200 import _lib
    from paper_1212_3032_b200.workloads import UNIT, cfg3_inputs

    lib = _lib.require_cuda()
    torch.cuda.set_device(local_rank)
    x, tris, omegas, xv = cfg3_inputs()
    P, M, F = len(x), len(tris), len(omegas)
    xd = torch.from_numpy(x).cuda()
    td = torch.from_numpy(tris.reshape(M, 9).copy()).cuda()
    vd = torch.from_numpy(xv.copy()).cuda()
    om = np.ascontiguousarray(np.stack([omegas.real, omegas.imag], axis=1))
    yu = torch.empty((F, P, 3), dtype=torch.complex128, device="cuda")
    yt = torch.empty_like(yu)
    ws_bytes = int(lib.ewb_pair_kernels_workspace_bytes(P, M, F))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    mat = UNIT

    def step():
        _lib.check(lib.ewb_pair_kernels_reduce(
            _lib.ptr(xd), P, _lib.ptr(td), M, _lib.ptr(vd), om.ctypes.data, F, mat.lam, mat.mu,
            mat.rho, _lib.ptr(yu), _lib.ptr(yt), _lib.ptr(ws), ws_bytes, _lib.stream_handle()))

    peak64 = bench.fp64_peak()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = bench.ClockSampler(local_rank)
    l0 = lib.ewb_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    evals = float(P) * M * F
    rate = evals / (ms * 1e-3)
    tf = rate * PAIR_FLOPS / 1e12
    line = {
        "metric": "element-pair kernel evals/s", "value": rate, "unit": "pair-evals/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded cfg3 inputs)",
        "config": {"workload": f"cfg3: {P} points x {M} triangles x {F} omega, gauss7, fused "
                               "U/T reduction", "l2": "compute-bound; inputs 1.3 MB"},
        "roofline": {"bound": "fp64", "achieved": tf, "peak": peak64, "unit": "TFLOP/s",
                     "frac": tf / peak64, "traffic": None,
                     "algorithmic_flops_per_launch": evals * PAIR_FLOPS,
                     "peak_source": "measured DFMA probe"},
        "gpu_launches": lib.ewb_launch_count() - l0, "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def _concurrent_gmres(As, bs, pinvs, n):
    """The batch's independent solves side by side (gmres_device_concurrent)."""
    import torch

    from paper_1212_3032_b200.linsolve import gmres_device_concurrent

    xs = [torch.zeros(n, dtype=torch.complex128, device="cuda") for _ in bs]
    gmres_device_concurrent(As, bs, xs, 1e-8, 50, 1000, pinvs)   # warm-up (workspaces)
    xs = [torch.zeros(n, dtype=torch.complex128, device="cuda") for _ in bs]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = gmres_device_concurrent(As, bs, xs, 1e-8, 50, 1000, pinvs, sync=False)
    e1.record()
    torch.cuda.synchronize()
    st = gmres_device_concurrent(As, bs, [torch.zeros_like(x) for x in xs], 1e-8, 50, 1000, pinvs)
    ms = e0.elapsed_time(e1)
    passes = sum(s.matvecs for s in st)
    return dict(gmres_concurrent_ms_total=ms,
                gmres_concurrent_iterations=[s.iterations for s in st],
                gmres_concurrent_solve_gbs=passes * 16.0 * n * n / (ms * 1e-3) / 1e9)


def run_cfg4(args, rank, world, local_rank):
    import torch

    import bench
    from paper_1212_3032_b200 import _lib
    from paper_1212_3032_b200.linsolve import _Workspace, gmres_device

    lib = _lib.require_cuda()
    torch.cuda.set_device(local_rank)
    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    batch = 8
    results = {}
    for n in (4096, 8192, 16384):
        g = torch.Generator(device="cuda")
        g.manual_seed(n)
        A = torch.empty((batch, n, n), dtype=torch.complex128, device="cuda")
        for s in range(batch):
            re = torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64)
            im = torch.randn((n, n), generator=g, device="cuda", dtype=torch.float64)
            A[s] = torch.complex(re, im) / math.sqrt(2.0)
            A[s].diagonal().add_(3.0 * math.sqrt(n))
            del re, im
        b = torch.complex(torch.randn((batch, n), generator=g, device="cuda", dtype=torch.float64),
                          torch.randn((batch, n), generator=g, device="cuda",
                                      dtype=torch.float64)) / math.sqrt(2.0)
        y = torch.empty_like(b)

        def step():
            _lib.check(lib.ewb_gemv_batched(_lib.ptr(A), _lib.ptr(b), _lib.ptr(y), n, batch,
                                            _lib.stream_handle()))

        for _ in range(max(3, args.warmup)):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(5, args.steps)
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = batch * (16.0 * n * n + 32.0 * n) / (ms * 1e-3) / 1e9
        # correctness spot check against a torch matvec of one system
        ref = A[batch - 1] @ b[batch - 1]
        err = float((y[batch - 1] - ref).abs().max() / ref.abs().max())
        # GMRES per system: restart 50, tol 1e-8, no preconditioner
        ws = _Workspace()
        its, t_solve, passes = [], 0.0, 0
        for s in range(batch):
            xs = torch.zeros(n, dtype=torch.complex128, device="cuda")
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            st = gmres_device(A[s], b[s].contiguous(), xs, False, 1e-8, 50, 1000, None, ws=ws)
            f1.record()
            torch.cuda.synchronize()
            t_solve += f0.elapsed_time(f1)
            its.append(st.iterations)
            passes += st.matvecs
        solve_gbs = passes * 16.0 * n * n / (t_solve * 1e-3) / 1e9
        conc = _concurrent_gmres([A[s] for s in range(batch)],
                                 [b[s].contiguous() for s in range(batch)], None, n)
        results[n] = dict(gemv_ms=ms, gemv_gbs=gbs, gemv_frac=gbs / hbm, gemv_relerr=err,
                          gmres_iterations=its, gmres_ms_total=t_solve,
                          gmres_passes=passes, gmres_solve_gbs=solve_gbs, **conc)
        del A, b, y
        torch.cuda.empty_cache()
    # cfg4-ii: assembled BEM operators, 8 consecutive frequencies from one
    # multi-frequency assembly pass, the same batched GEMV + per-system GMRES
    # (restart 50, tol 1e-8, the sweep's block preconditioner)
    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.transform import eta_from_kappa, frequency_grid
    from paper_1212_3032_b200.workloads import cfg4_assembled

    assembled = {}
    for name, cfg in cfg4_assembled():
        asm = Assembler(cfg.mesh, cfg.material)
        om = frequency_grid(cfg.period, cfg.n_omega, eta_from_kappa(cfg.kappa, cfg.period))
        n = asm.n
        ks = list(range(40, 40 + batch))
        gP = torch.Generator(device="cuda")
        gP.manual_seed(n)
        P = torch.complex(torch.randn((batch, n), generator=gP, device="cuda", dtype=torch.float64),
                          torch.randn((batch, n), generator=gP, device="cuda", dtype=torch.float64))
        sb = asm.assemble_system_multi([om[k] for k in ks], cfg.bcs, P)
        xb = sb.b.clone()
        y = torch.empty_like(xb)

        def step():
            _lib.check(lib.ewb_gemv_batched(_lib.ptr(sb.A), _lib.ptr(xb), _lib.ptr(y), n, batch,
                                            _lib.stream_handle()))

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        gbs = batch * (16.0 * n * n + 32.0 * n) / (ms * 1e-3) / 1e9
        ref = sb.A[batch - 1] @ xb[batch - 1]
        err = float((y[batch - 1] - ref).abs().max() / ref.abs().max())
        ws = _Workspace()
        its, t_solve, passes = [], 0.0, 0
        for s_ in range(batch):
            xs = torch.zeros(n, dtype=torch.complex128, device="cuda")
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            st = gmres_device(sb.A[s_], sb.b[s_], xs, False, 1e-8, 50, 1000, sb.pinv[s_], ws=ws)
            f1.record()
            torch.cuda.synchronize()
            t_solve += f0.elapsed_time(f1)
            its.append(st.iterations)
            passes += st.matvecs
        conc = _concurrent_gmres([sb.A[s_] for s_ in range(batch)],
                                 [sb.b[s_] for s_ in range(batch)],
                                 [sb.pinv[s_] for s_ in range(batch)], n)
        assembled[name] = dict(n=n, frequencies=ks, gemv_ms=ms, gemv_gbs=gbs,
                               gemv_frac=gbs / hbm, gemv_relerr=err, gmres_iterations=its,
                               gmres_ms_total=t_solve, gmres_passes=passes,
                               gmres_solve_gbs=passes * 16.0 * n * n / (t_solve * 1e-3) / 1e9,
                               **conc)
        del sb, xb, y, P, asm
        torch.cuda.empty_cache()
    top = results[16384]
    line = {
        "metric": "complex matvec HBM GB/s", "value": top["gemv_gbs"], "unit": "GB/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": top["gemv_ms"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded diagonally dominant complex Gaussian, device-generated)",
        "config": {"workload": "cfg4: batched dense complex128 matvec, 8 systems, N=16384 "
                               "(4096/8192 in metrics)", "l2": "inputs larger than L2 (34 GB)"},
        "roofline": {"bound": "hbm", "achieved": top["gemv_gbs"], "peak": hbm, "unit": "GB/s",
                     "frac": top["gemv_frac"], "traffic": None,
                     "algorithmic_bytes_per_launch": 8 * (16.0 * 16384 ** 2 + 32 * 16384),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
        "metrics": {**{str(k): v for k, v in results.items()}, "assembled": assembled},
    }
    print(json.dumps(line), flush=True)


def cfg5_measure(steps: int, warmup: int, peak64: float | None = None) -> dict:
    """cfg5: ico6 cavity, 81,920 el / 245,760 DOF, matrix-free (966 GB dense).

    One matrix-free operator application (6.7e9 pairs, 2.04e10 quadrature
    points, K = 1) timed with CUDA events, plus the first two frequencies of
    the SEM sweep (the reference's own check range).  Returns the figures."""
    import torch

    import bench
    from paper_1212_3032_b200 import _lib
    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.matfree import MatrixFreeOperator
    from paper_1212_3032_b200.workloads import cfg5

    lib = _lib.require_cuda()
    peak64 = peak64 or bench.fp64_peak()
    cfg = cfg5()
    t0 = time.perf_counter()
    ds = DeviceSweep(cfg, frequencies=[0, 1])
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    pc = ds.asm.pair_counts()
    pairs = pc["far"] + pc["mid"] + pc["near"] + pc["n_elements"]
    pe = ds.asm.point_evals()
    flops = 397.0 * pe + 72.0 * pairs            # SURVEY §8(d) matrix-free count
    op = MatrixFreeOperator(ds.asm, complex(ds.omegas[1]))
    v = torch.randn((1, ds.n), dtype=torch.complex128, device="cuda")
    for _ in range(max(1, warmup)):
        op.apply_multi(v)
    torch.cuda.synchronize()
    sampler = bench.ClockSampler(torch.cuda.current_device())
    l0 = lib.ewb_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        op.apply_multi(v)
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = lib.ewb_launch_count() - l0
    ms = e0.elapsed_time(e1) / steps
    ds.matrix_free = True
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stats = ds.run()
    torch.cuda.synchronize()
    first2 = time.perf_counter() - t1
    tf = flops / (ms * 1e-3) / 1e12
    return {
        "workload": "cfg5: flipped icosphere L6, 81920 el / 245760 DOF, matrix-free",
        "application_ms": ms, "pair_evals_per_s": pairs / (ms * 1e-3),
        "point_evals_per_application": pe, "pairs": pc, "steps": steps,
        "roofline": {"bound": "fp64", "kernel": "k_mf_farmid<1> (+ k_mf_near, k_mf_self): one A v",
                     "achieved": tf, "peak": peak64, "unit": "TFLOP/s", "frac": tf / peak64,
                     "traffic": None, "algorithmic_flops_per_launch": flops,
                     "peak_source": "measured DFMA probe",
                     "ncu": "profiles/r02/SUMMARY.md (matrix-free capture)"},
        "gpu_launches": launches, "clocks": clocks, "setup_s": setup_s,
        "first_two_frequencies_s": first2,
        "first_two": {int(k): dict(iterations=s.iterations, applications=s.matvecs,
                                   init_residual=s.init_residual,
                                   final_residual=s.final_residual)
                      for k, s in stats.items()},
    }


def run_cfg5(args, rank, world, local_rank):
    import torch

    torch.cuda.set_device(local_rank)
    r = cfg5_measure(args.steps, args.warmup)
    line = {
        "metric": "element-pair kernel evals/s", "value": r["pair_evals_per_s"],
        "unit": "pair-evals/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r["application_ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference-generated ico6 cavity, unit step pressure)",
        "config": {"workload": r["workload"] + " operator application (one step = one A v "
                                               "over all 6.7e9 pairs)", "l2": "compute-bound"},
        "roofline": r["roofline"], "gpu_launches": r["gpu_launches"], "clocks": r["clocks"],
        "metrics": {k: r[k] for k in ("setup_s", "point_evals_per_application", "pairs",
                                      "first_two_frequencies_s", "first_two")},
    }
    print(json.dumps(line), flush=True)


def main(args, rank, world, local_rank):
    if rank != 0:
        return
    if args.workload == "cfg3":
        run_cfg3(args, rank, world, local_rank)
    elif args.workload == "cfg4":
        run_cfg4(args, rank, world, local_rank)
    elif args.workload == "cfg5":
        run_cfg5(args, rank, world, local_rank)
