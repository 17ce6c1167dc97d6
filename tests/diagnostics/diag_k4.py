"""Cross-check at cfg1 k=4: oracle GMRES vs GPU GMRES on oracle-/GPU-assembled A.

Test infrastructure (the oracle is the checker); not collected by pytest.
Run from the repo root: python tests/diagnostics/diag_k4.py"""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import ewbem_oracle as O
from paper_1212_3032_b200 import Assembler
from paper_1212_3032_b200.linsolve import gmres_device, sem_device
from paper_1212_3032_b200.workloads import cfg1
cfg = cfg1()
m = cfg.mesh; med = O.Medium(cfg.material.lam, cfg.material.mu, cfg.material.rho)
eta = O.eta_from_kappa(cfg.kappa, cfg.period); om = O.frequency_grid(cfg.period, cfg.n_omega, eta)
spectra = np.stack([O.forward_spectrum(s.sample(cfg.period, cfg.n_omega), cfg.period, eta)[:len(om)] for s in cfg.signals])
kinds = cfg.bcs.flat_kind(); sig = cfg.bcs.flat_signal()
asm_o = O.DenseOracle(m.vertices, m.triangles, med); asm_o.rowsums()
asm_g = Assembler(m, cfg.material)
hist = O.History(2)
for k in range(6):
    t, u = asm_o.tu(om[k]); p = spectra[sig, k]
    a, b = O.apply_bcs(t, u, kinds, p)
    sysg = asm_g.assemble_system(om[k], cfg.bcs, p)
    ag = sysg.A.cpu().numpy(); bg = sysg.b.cpu().numpy()
    print(f"k={k} |dA|={np.abs(ag-a).max()/np.abs(a).max():.2e} |db|={np.abs(bg-b).max()/np.abs(b).max():.2e}")
    x0 = O.sem_guess(hist, a, b) if len(hist) else None
    pc, inv = O.block_precond(a)
    x, st = O.gmres(a, b, x0=x0, tol=1e-8, restart=60, maxiter=1000, precond=pc)
    x0g = O.sem_guess(hist, ag, bg) if len(hist) else None
    pcg, _ = O.block_precond(ag)
    _, st2 = O.gmres(ag, bg, x0=x0g, tol=1e-8, restart=60, maxiter=1000, precond=pcg)
    # GPU gmres on the oracle system with the oracle x0 and oracle pinv
    A = torch.from_numpy(a).cuda(); B = torch.from_numpy(b).cuda()
    X = torch.from_numpy(x0 if x0 is not None else np.zeros_like(b)).cuda()
    PI = torch.from_numpy(np.ascontiguousarray(inv)).cuda()
    st3 = gmres_device(A, B, X, x0 is not None, 1e-8, 60, 1000, PI)
    # GPU SEM on oracle system
    if len(hist):
        XC = torch.from_numpy(np.ascontiguousarray(hist.matrix().T)).cuda()
        x0d = torch.empty_like(B); sem_device(A, B, XC, 1e-10, x0d)
        dx0 = np.abs(x0d.cpu().numpy()-x0).max()/np.abs(x0).max()
    else:
        dx0 = 0
    print(f"   oracle(A_o)={st.iterations} oracle(A_gpu)={st2.iterations} gpu_gmres(A_o)={st3.iterations} |dx0 sem|={dx0:.2e}", flush=True)
    hist.push(x)
