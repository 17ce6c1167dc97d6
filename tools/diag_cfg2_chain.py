"""cfg2 (129 SEM-chained solves): our sweep vs the live reference's run
(tests/golden/cfg2_sweep.npz) and vs the reference's solver (the oracle,
bitwise equal to linsolve.py) chained over the SAME assembled systems on
this host.  Test infrastructure; ~10 min of host BLAS on 16 cores.

    python tools/diag_cfg2_chain.py [--no-chain]
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import run_sweep
    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.workloads import cfg2

    g = dict(np.load(ROOT / "tests" / "golden" / "cfg2_sweep.npz"))
    cfg = cfg2()
    res = run_sweep(cfg)
    its = np.array([s.iterations for s in res.stats])
    out = {"gpu_its": its.tolist(), "golden_its": g["cfg2_its"].tolist(),
           "d_golden": (its - g["cfg2_its"]).tolist(),
           "gpu_init": [s.init_residual for s in res.stats],
           "golden_init": g["cfg2_init"].tolist(),
           "hist_rel": {str(nm): float(np.linalg.norm(res.histories[str(nm)] - g[f"cfg2_h_{nm}"])
                                       / np.linalg.norm(g[f"cfg2_h_{nm}"]))
                        for nm in g["cfg2_probes"]},
           "gpu_total": int(its.sum()), "golden_total": int(g["cfg2_its"].sum()),
           "spec_rel_gpu": {str(nm): (np.abs(np.asarray(res.half_spectra[str(nm)]) - g[f"cfg2_s_{nm}"])
                                      / np.abs(g[f"cfg2_s_{nm}"]).max()).tolist()
                            for nm in g["cfg2_probes"]}}
    if "--no-chain" not in sys.argv:
        ds = DeviceSweep(cfg)
        nb = ds.batch_size()
        hist = O.History(cfg.sem_depth)
        och, batch, t0 = [], None, time.perf_counter()
        probe_vals = {p.name: [] for p in cfg.probes}
        for k0 in range(0, ds.n_freq, nb):
            ks = list(range(k0, min(ds.n_freq, k0 + nb)))
            batch = ds.asm.assemble_system_multi([ds.omegas[k] for k in ks], cfg.bcs,
                                                 ds.P[ks[0]:ks[-1] + 1], out=batch, check=False)
            for f in range(len(ks)):
                m = batch.member(f)
                a, b = m.A.cpu().numpy(), m.b.cpu().numpy()
                x0 = O.sem_guess(hist, a, b) if len(hist) else None
                pc, _ = O.block_precond(a)
                x, st = O.gmres(a, b, x0=x0, tol=cfg.tol, restart=cfg.restart,
                                maxiter=cfg.maxiter, precond=pc)
                och.append(st.iterations)
                hist.push(x)
                for p in cfg.probes:          # all-Neumann: displacement = unknown
                    probe_vals[p.name].append(x[p.dof])
                print(f"k={ks[f]} gpu={its[ks[f]]} ref_solver={st.iterations} "
                      f"golden={g['cfg2_its'][ks[f]]} {time.perf_counter() - t0:.0f}s",
                      file=sys.stderr, flush=True)
        och = np.array(och)
        eta = O.eta_from_kappa(cfg.kappa, cfg.period)
        h_ref_solver = {}
        for nm, vals in probe_vals.items():
            series, _ = O.inverse_transform(O.conjugate_fill(np.array(vals)), cfg.window, eta,
                                            cfg.period)
            h_ref_solver[nm] = series
        out["hist_rel_ref_solver_vs_golden"] = {
            nm: float(np.linalg.norm(h_ref_solver[nm] - g[f"cfg2_h_{nm}"])
                      / np.linalg.norm(g[f"cfg2_h_{nm}"])) for nm in h_ref_solver}
        out["hist_rel_gpu_vs_ref_solver"] = {
            nm: float(np.linalg.norm(res.histories[nm] - h_ref_solver[nm])
                      / np.linalg.norm(h_ref_solver[nm])) for nm in h_ref_solver}
        out["spec_rel_ref_solver"] = {
            nm: (np.abs(np.array(vals) - g[f"cfg2_s_{nm}"]) / np.abs(g[f"cfg2_s_{nm}"]).max()).tolist()
            for nm, vals in probe_vals.items()}
        out.update(ref_solver_its=och.tolist(), d_ref_solver=(its - och).tolist(),
                   ref_solver_vs_golden=(och - g["cfg2_its"]).tolist(),
                   chain_seconds=time.perf_counter() - t0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
