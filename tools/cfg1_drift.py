"""cfg1 chained sweep: GPU iteration counts vs the golden reference run and
vs the oracle's sweep run on THIS host (the same-box comparison SURVEY App.
B-3 asks for).  Prints one JSON line; test infrastructure (imports oracle/).

    python tools/cfg1_drift.py [--no-oracle]
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def oracle_cfg1_sweep(cfg):
    from oracle import ewbem_oracle as O

    med = O.Medium(cfg.material.lam, cfg.material.mu, cfg.material.rho)
    m = cfg.mesh
    samples = [np.asarray(s.sample(cfg.period, cfg.n_omega), float) for s in cfg.signals]
    probes = [(p.name, 3 * p.element + p.component, p.quantity) for p in cfg.probes]
    t0 = time.perf_counter()
    _, hists, stats, _ = O.sweep(m.vertices, m.triangles, med, cfg.bcs.flat_kind(),
                                 cfg.bcs.flat_signal(), samples, probes, cfg.period,
                                 cfg.n_omega, cfg.kappa, cfg.window, cfg.sem_depth,
                                 cfg.sem_enabled, cfg.tol, cfg.restart, cfg.maxiter)
    return time.perf_counter() - t0, hists, stats


def main():
    from paper_1212_3032_b200 import run_sweep
    from paper_1212_3032_b200.workloads import cfg1

    g = dict(np.load(ROOT / "tests" / "golden" / "cfg1_sweep.npz"))
    cfg = cfg1()
    res = run_sweep(cfg)
    its = np.array([s.iterations for s in res.stats])
    gi = g["cfg1_its"]
    out = {"gpu_its": its.tolist(), "golden_its": gi.tolist(),
           "d_golden": (its - gi).tolist(),
           "gpu_init": [s.init_residual for s in res.stats],
           "gpu_final": [s.final_residual for s in res.stats]}
    if "--no-oracle" not in sys.argv:
        secs, hists, stats = oracle_cfg1_sweep(cfg)
        oi = np.array([s.iterations for s in stats])
        out.update(oracle_s=secs, oracle_its=oi.tolist(), d_oracle=(its - oi).tolist(),
                   oracle_vs_golden=(oi - gi).tolist(), nproc=os.cpu_count(),
                   oracle_init=[s.init_residual for s in stats],
                   hist_rel={n: float(np.linalg.norm(res.histories[n] - hists[n]) /
                                      np.linalg.norm(hists[n])) for n in hists})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
