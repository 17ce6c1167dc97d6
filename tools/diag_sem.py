"""Where does a cfg1 solution differ from the reference's at the tolerance
level?  Fed the reference's own history (tests/golden/cfg1_solutions.npz),
compare the SEM guesses and the GMRES iterates of GPU and oracle at k
(test infrastructure).

    python tools/diag_sem.py K [K ...]
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    import torch

    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.linsolve import gmres_device, sem_device
    from paper_1212_3032_b200.transform import eta_from_kappa, forward_mft, frequency_grid
    from paper_1212_3032_b200.workloads import cfg1

    ks = [int(a) for a in sys.argv[1:]] or [3]
    g = dict(np.load(ROOT / "tests" / "golden" / "cfg1_solutions.npz"))
    xref = g["x"]
    cfg = cfg1()
    asm = Assembler(cfg.mesh, cfg.material)
    eta = eta_from_kappa(cfg.kappa, cfg.period)
    om = frequency_grid(cfg.period, cfg.n_omega, eta)
    spectra = np.stack([forward_mft(s, cfg.period, cfg.n_omega, eta).values for s in cfg.signals])
    sig, kinds = cfg.bcs.flat_signal(), cfg.bcs.flat_kind()
    med = O.Medium(cfg.material.lam, cfg.material.mu, cfg.material.rho)
    dense = O.DenseOracle(cfg.mesh.vertices, cfg.mesh.triangles, med)
    out = {}
    for k in ks:
        p = spectra[sig, k]
        t_o, u_o = dense.tu(om[k])
        a, b = O.apply_bcs(t_o, u_o, kinds, p)
        H = O.History(2)
        for v in xref[max(0, k - 2):k]:
            H.push(v)
        X = H.matrix()
        Y = a @ X
        sv = np.linalg.svd(Y, compute_uv=False)
        x0_o = O.sem_guess(H, a, b)
        ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        xx = torch.zeros_like(bd)
        sem_device(ad, bd, torch.from_numpy(np.ascontiguousarray(X.T)).cuda(), 1e-10, xx)
        x0_g = xx.cpu().numpy()
        s_o = np.linalg.lstsq(X, x0_o, rcond=None)[0]
        s_g = np.linalg.lstsq(X, x0_g, rcond=None)[0]
        # exact-ish LS in extended precision via normal equations on the small system
        pc, inv = O.block_precond(a)
        row = {"cond_Y": float(sv[0] / sv[-1]), "sv": sv.tolist(), "s_o": [str(v) for v in s_o],
               "s_rel_diff": float(np.abs(s_g - s_o).max() / np.abs(s_o).max()),
               "x0_rel_diff": rel(x0_g, x0_o),
               "r0_o": float(np.linalg.norm(b - a @ x0_o) / np.linalg.norm(b)),
               "r0_g": float(np.linalg.norm(b - a @ x0_g) / np.linalg.norm(b))}
        pinv = torch.from_numpy(inv).cuda()
        for name, x0 in (("o", x0_o), ("g", x0_g)):
            xo, st_o = O.gmres(a, b, x0=x0, tol=cfg.tol, restart=cfg.restart,
                               maxiter=cfg.maxiter, precond=pc)
            xg = torch.from_numpy(x0.copy()).cuda()
            st_g = gmres_device(ad, bd, xg, True, cfg.tol, cfg.restart, cfg.maxiter, pinv)
            xg = xg.cpu().numpy()
            row[f"from_x0{name}"] = {
                "its_oracle": st_o.iterations, "its_gpu": st_g.iterations,
                "x_gpu_vs_oracle": rel(xg, xo), "x_oracle_vs_ref": rel(xo, xref[k]),
                "x_gpu_vs_ref": rel(xg, xref[k]), "final_o": st_o.final_residual,
                "final_g": st_g.final_residual}
        out[k] = row
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
