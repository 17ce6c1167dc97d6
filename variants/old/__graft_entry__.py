"""Driver entry points: build() compiles the sm_100a library; smoke() runs one
small solve on cuda:0 and checks it against the CPU oracle (test
infrastructure under oracle/, used here only as the checker)."""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent


def build() -> None:
    sys.path.insert(0, str(ROOT))
    from paper_1212_3032_b200.build import build as _build

    _build(force=True)
    import paper_1212_3032_b200  # noqa: F401
    from paper_1212_3032_b200 import _lib

    _lib.load()


def smoke() -> None:
    """Tiny dense assembly + fused system + GMRES on cuda:0 vs the oracle."""
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch

    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import (Assembler, BoundaryConditionSet, DIRICHLET, Material,
                                      NEUMANN, block_diag_precond, generate_box_mesh, gmres)

    assert torch.cuda.is_available(), "smoke() needs a GPU"
    mesh = generate_box_mesh((1, 1, 1), (2, 2, 2))
    mat = Material.from_young_poisson(1.0, 0.25, 1.0)
    omega = 2.0 - 0.47j
    asm = Assembler(mesh, mat)
    t, u = asm.assemble_tu(omega, host=True)
    ref = O.DenseOracle(mesh.vertices, mesh.triangles, O.Medium(mat.lam, mat.mu, mat.rho))
    tr, ur = ref.tu(omega)
    et = np.abs(t - tr).max() / np.abs(tr).max()
    eu = np.abs(u - ur).max() / np.abs(ur).max()
    assert et < 1e-10 and eu < 1e-10, (et, eu)
    bcs = BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.set_region(mesh, 4, (0, 1, 2), DIRICHLET, 0)
    bcs.set_region(mesh, 5, (2,), NEUMANN, 1)
    p = np.zeros(mesh.n_dofs, complex)
    p[3 * np.flatnonzero(mesh.region_tag == 5) + 2] = -1.0
    sysm = asm.assemble_system(omega, bcs, p)
    x, st = gmres(sysm.A, sysm.b, tol=1e-10, precond=block_diag_precond(sysm.A))
    a_ref, b_ref = O.apply_bcs(tr, ur, bcs.flat_kind(), p)
    x_ref = np.linalg.solve(a_ref, b_ref)
    ex = np.abs(x.cpu().numpy() - x_ref).max() / np.abs(x_ref).max()
    assert st.converged and ex < 1e-8, (st, ex)
    print(f"smoke ok: |dT|={et:.2e} |dU|={eu:.2e} |dx|={ex:.2e} its={st.iterations}")


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "smoke"
    {"build": build, "smoke": smoke}[cmd]()
