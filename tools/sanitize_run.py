"""Small workloads for compute-sanitizer: every product kernel
launches at least once, at sizes the sanitizer finishes in minutes.

    compute-sanitizer --tool {memcheck,racecheck,synccheck} \
        python tools/sanitize_run.py {dense,matfree,gemv}

dense    reduced cfg1 sweep (8x8x8 box, 3 SEM-chained solves: multi-frequency
         assembly, fused BCs/preconditioner, SEM, cooperative GMRES, IDFT)
matfree  ico2 matrix-free SEM sweep (operator GMRES seam) + one ico3 apply
gemv     batched TMA GEMV and the multi-column SEM product (cfg4 kernels)
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def dense():
    from paper_1212_3032_b200 import run_sweep
    from paper_1212_3032_b200.workloads import cfg1

    res = run_sweep(cfg1(n_omega=4))
    print("dense its", [s.iterations for s in res.stats], "failed", res.failed_frequencies)


def matfree():
    import torch

    from paper_1212_3032_b200 import Assembler, MatrixFreeOperator, run_sweep
    from paper_1212_3032_b200.workloads import sphere_pressure

    res = run_sweep(sphere_pressure(2, 6), matrix_free=True)
    print("matfree its", [s.iterations for s in res.stats], "failed", res.failed_frequencies)
    cfg = sphere_pressure(3, 8)
    op = MatrixFreeOperator(Assembler(cfg.mesh, cfg.material), 3.0 - 0.2j)
    v = torch.randn((2, cfg.mesh.n_dofs), dtype=torch.complex128, device="cuda")
    y = op.apply_multi(v, want_pinv=True)
    torch.cuda.synchronize()
    print("ico3 apply", float(y.abs().max()))


def gemv():
    import torch

    from paper_1212_3032_b200 import _lib, gmres
    from paper_1212_3032_b200.workloads import cfg4_random_system

    lib = _lib.load()
    a, b = cfg4_random_system(4096, 1)
    A = torch.from_numpy(np.stack([a, a])).cuda()
    X = torch.from_numpy(np.stack([b, b])).cuda()
    Y = torch.empty_like(X)
    _lib.check(lib.ewb_gemv_batched(_lib.ptr(A), _lib.ptr(X), _lib.ptr(Y), 4096, 2,
                                    _lib.stream_handle()))
    torch.cuda.synchronize()
    print("gemv", float((Y[0] - Y[1]).abs().max()))
    x, st = gmres(A[0], b, tol=1e-8, restart=50, maxiter=1000)
    print("gmres its", st.iterations)


if __name__ == "__main__":
    {"dense": dense, "matfree": matfree, "gemv": gemv}[sys.argv[1]]()
