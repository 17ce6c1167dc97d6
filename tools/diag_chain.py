"""cfg1 chained solves k = 0..K-1 in four combinations (test infrastructure):
solver in {GPU, oracle} x matrices in {GPU-assembled, oracle-assembled},
each chain feeding its own SEM history.  Prints per-k iterations and the
relative difference of each chain's solution from the reference's own
(tests/golden/cfg1_solutions.npz).

    python tools/diag_chain.py [K] [Gg,Go,Og,Oo]
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.linsolve import gmres_device, sem_device
    from paper_1212_3032_b200.transform import eta_from_kappa, forward_mft, frequency_grid
    from paper_1212_3032_b200.workloads import cfg1

    K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    combos = sys.argv[2].split(",") if len(sys.argv) > 2 else ["Gg", "Go", "Og", "Oo"]
    need_o = any(c[1] == "o" for c in combos)
    xref = np.load(ROOT / "tests" / "golden" / "cfg1_solutions.npz")["x"]
    cfg = cfg1()
    asm = Assembler(cfg.mesh, cfg.material)
    eta = eta_from_kappa(cfg.kappa, cfg.period)
    om = frequency_grid(cfg.period, cfg.n_omega, eta)
    spectra = np.stack([forward_mft(s, cfg.period, cfg.n_omega, eta).values for s in cfg.signals])
    sig, kinds = cfg.bcs.flat_signal(), cfg.bcs.flat_kind()
    med = O.Medium(cfg.material.lam, cfg.material.mu, cfg.material.rho)
    systems = []
    dense = O.DenseOracle(cfg.mesh.vertices, cfg.mesh.triangles, med) if need_o else None
    for k in range(K):
        p = spectra[sig, k]
        s = asm.assemble_system(om[k], cfg.bcs, p)
        entry = {"g": (s.A.cpu().numpy(), s.b.cpu().numpy())}
        if need_o:
            t_o, u_o = dense.tu(om[k])
            entry["o"] = O.apply_bcs(t_o, u_o, kinds, p)
        systems.append(entry)

    def gpu_step(a, b, hist):
        ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        pinv = torch.from_numpy(O.block_precond(a)[1]).cuda()
        x = torch.zeros_like(bd)
        if hist:
            sem_device(ad, bd, torch.from_numpy(np.stack(hist)).cuda(), 1e-10, x)
        st = gmres_device(ad, bd, x, bool(hist), cfg.tol, cfg.restart, cfg.maxiter, pinv)
        return x.cpu().numpy(), st

    def oracle_step(a, b, hist):
        H = O.History(2)
        for v in hist[::-1]:
            H.push(v)
        x0 = O.sem_guess(H, a, b) if hist else None
        pc, _ = O.block_precond(a)
        return O.gmres(a, b, x0=x0, tol=cfg.tol, restart=cfg.restart, maxiter=cfg.maxiter,
                       precond=pc)

    out = {}
    for combo in combos:
        solver, mats = combo[0], combo[1]
        step = gpu_step if solver == "G" else oracle_step
        if True:
            hist, its, dx, fin = [], [], [], []
            for k in range(K):
                a, b = systems[k][mats]
                x, st = step(a, b, hist[:2])
                its.append(st.iterations)
                fin.append(st.final_residual)
                dx.append(float(np.linalg.norm(x - xref[k]) / np.linalg.norm(xref[k])))
                hist = [x] + hist
            out[combo] = {"its": its, "dx_vs_ref": dx, "final": fin}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
