"""Diagnose a cfg1 frequency whose chained iteration count drifts: GPU vs
oracle GMRES residual histories on identical inputs (test infrastructure).

    python tools/diag_cfg1_k.py K [K ...]

For each k: history x_{k-1}, x_{k-2} = the GPU sweep's own solutions; the
system assembled by the GPU (A_g, b_g) and by the oracle (A_o, b_o).  Runs
  GG  GPU SEM + GPU GMRES on A_g          (the sweep's path)
  OO  oracle SEM + oracle GMRES on A_o    (the reference's path)
  OG  oracle SEM + oracle GMRES on A_g    (solver effect)
  GO  GPU SEM + GPU GMRES on A_o          (assembly effect)
and prints iterations and the residual histories' last 8 values.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.linsolve import gmres_device, sem_device
    from paper_1212_3032_b200.transform import eta_from_kappa, forward_mft, frequency_grid
    from paper_1212_3032_b200.workloads import cfg1

    ks = [int(a) for a in sys.argv[1:]] or [4]
    cfg = cfg1()
    asm = Assembler(cfg.mesh, cfg.material)
    eta = eta_from_kappa(cfg.kappa, cfg.period)
    om = frequency_grid(cfg.period, cfg.n_omega, eta)
    spectra = np.stack([forward_mft(s, cfg.period, cfg.n_omega, eta).values for s in cfg.signals])
    sig = cfg.bcs.flat_signal()
    kinds = cfg.bcs.flat_kind()
    med = O.Medium(cfg.material.lam, cfg.material.mu, cfg.material.rho)
    dense = O.DenseOracle(cfg.mesh.vertices, cfg.mesh.triangles, med)
    # GPU chained solutions: rerun the chain on the device, keeping x_k
    xs, its = [], []
    x = torch.zeros(cfg.mesh.n_dofs, dtype=torch.complex128, device="cuda")
    sysm = None
    for k in range(max(ks) + 1):
        sysm = asm.assemble_system(om[k], cfg.bcs, spectra[sig, k], out=sysm)
        if k:
            hist = torch.stack(xs[max(0, k - 2):k][::-1])
            sem_device(sysm.A, sysm.b, hist, 1e-10, x)
        st = gmres_device(sysm.A, sysm.b, x, k > 0, cfg.tol, cfg.restart, cfg.maxiter, sysm.pinv)
        xs.append(x.clone())
        its.append(st.iterations)
    out = {"chain_its": its}
    for k in ks:
        p = spectra[sig, k]
        sysm = asm.assemble_system(om[k], cfg.bcs, p)
        a_g = sysm.A.cpu().numpy()
        b_g = sysm.b.cpu().numpy()
        t_o, u_o = dense.tu(om[k])
        a_o, b_o = O.apply_bcs(t_o, u_o, kinds, p)
        hx = [xs[j].cpu().numpy() for j in range(max(0, k - 2), k)]
        H = O.History(2)
        for v in hx:
            H.push(v)
        row = {"dA": float(np.abs(a_g - a_o).max() / np.abs(a_o).max()),
               "db": float(np.abs(b_g - b_o).max() / np.abs(b_o).max())}

        def oracle_solve(a, b):
            x0 = O.sem_guess(H, a, b)
            pc, _ = O.block_precond(a)
            x, st = O.gmres(a, b, x0=x0, tol=cfg.tol, restart=cfg.restart, maxiter=cfg.maxiter,
                            precond=pc)
            return st

        def gpu_solve(a, b):
            ad = torch.from_numpy(np.ascontiguousarray(a)).cuda()
            bd = torch.from_numpy(b).cuda()
            pinv = torch.from_numpy(O.block_precond(a)[1]).cuda()
            xx = torch.zeros_like(bd)
            hist = torch.from_numpy(np.stack(hx[::-1])).cuda()
            sem_device(ad, bd, hist, 1e-10, xx)
            return gmres_device(ad, bd, xx, True, cfg.tol, cfg.restart, cfg.maxiter, pinv)

        for name, fn, a, b in (("GG", gpu_solve, a_g, b_g), ("OO", oracle_solve, a_o, b_o),
                               ("OG", oracle_solve, a_g, b_g), ("GO", gpu_solve, a_o, b_o)):
            st = fn(a, b)
            h = list(map(float, st.residual_history))
            row[name] = {"its": st.iterations, "init": st.init_residual,
                         "final": st.final_residual, "tail": h[-10:]}
        out[str(k)] = row
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
