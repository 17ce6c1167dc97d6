"""GPU parity: matrix-free operator (north-star item 2) and the cfg3 pair kernels."""

import numpy as np
import pytest

from conftest import golden, rel_max

pytestmark = pytest.mark.gpu


def _unit():
    from paper_1212_3032_b200 import Material

    return Material.from_young_poisson(1.0, 0.25, 1.0)


def _rod_bcs(mesh):
    from paper_1212_3032_b200 import DIRICHLET, NEUMANN, BoundaryConditionSet

    bcs = BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.set_region(mesh, 0, (0, 1, 2), DIRICHLET, 0)
    bcs.set_region(mesh, 1, (0,), NEUMANN, 1)
    return bcs


@pytest.mark.parametrize("mesh_kind", ["box", "ico"])
def test_matfree_matvec_equals_dense_system(cuda, mesh_kind):
    """A v and b from the matrix-free kernels == the fused dense system (1e-10)."""
    import torch

    from paper_1212_3032_b200 import Assembler, MatrixFreeOperator
    from paper_1212_3032_b200.workloads import box_mesh, cavity_mesh

    mesh = (box_mesh((1, 1, 1), (4, 4, 4)) if mesh_kind == "box"
            else cavity_mesh(2))
    asm = Assembler(mesh, _unit())
    bcs = _rod_bcs(mesh) if mesh_kind == "box" else None
    from paper_1212_3032_b200 import BoundaryConditionSet

    bcs_dense = bcs or BoundaryConditionSet.traction_free(mesh.n_elements)
    rng = np.random.default_rng(4)
    n = mesh.n_dofs
    p = rng.normal(size=n) + 1j * rng.normal(size=n)
    for om in (0.3 - 0.2j, 5.0 - 0.47j):
        dense = asm.assemble_system(om, bcs_dense, p)
        A = dense.A
        op = MatrixFreeOperator(asm, om, bcs)
        V = torch.from_numpy(rng.normal(size=(3, n)) + 1j * rng.normal(size=(3, n))).cuda()
        Y = op.apply_multi(V, want_pinv=True)
        ref = (A @ V.T).T
        assert rel_max(Y.cpu().numpy(), ref.cpu().numpy()) <= 1e-10
        assert rel_max(op.pinv.cpu().numpy(), dense.pinv.cpu().numpy()) <= 1e-10
        b, Y2 = op.rhs_and_apply(torch.from_numpy(p).cuda(), V[:2])
        assert rel_max(b.cpu().numpy(), dense.b.cpu().numpy()) <= 1e-10
        assert rel_max(Y2.cpu().numpy(), ref[:2].cpu().numpy()) <= 1e-10


def test_matfree_gmres_and_sem_match_dense(cuda):
    """Device Arnoldi with a matrix-free callable == dense GMRES (its +-1, x 1e-8)."""
    import torch

    from paper_1212_3032_b200 import (Assembler, BoundaryConditionSet, MatrixFreeOperator,
                                      SolutionHistory, gmres, sem_initial_guess)
    from paper_1212_3032_b200.workloads import cavity_mesh

    mesh = cavity_mesh(2)
    asm = Assembler(mesh, _unit())
    bcs = BoundaryConditionSet.traction_free(mesh.n_elements)
    load = (-1.0 * mesh.normals).ravel().astype(complex)
    om = 2.0 - 0.37j
    dense = asm.assemble_system(om, bcs, load)
    op = MatrixFreeOperator(asm, om, bcs)
    b, _ = op.rhs_and_apply(torch.from_numpy(load).cuda())
    pc = op.block_preconditioner()
    x_mf, st_mf = gmres(op, b, tol=1e-8, restart=60, precond=pc)
    from paper_1212_3032_b200 import block_diag_precond

    x_d, st_d = gmres(dense.A, dense.b, tol=1e-8, restart=60, precond=block_diag_precond(dense.A))
    assert abs(st_mf.iterations - st_d.iterations) <= 1
    assert rel_max(x_mf.cpu().numpy(), x_d.cpu().numpy()) <= 1e-7
    hist = SolutionHistory(4)
    rng = np.random.default_rng(1)
    for _ in range(3):
        hist.push(x_d + 1e-3 * torch.from_numpy(rng.normal(size=mesh.n_dofs) + 0j).cuda())
    x0_mf = sem_initial_guess(hist, op, b)
    x0_d = sem_initial_guess(hist, dense.A, dense.b)
    assert rel_max(x0_mf.cpu().numpy(), x0_d.cpu().numpy()) <= 1e-8


def test_matfree_sampled_rows_vs_oracle(cuda):
    """cfg5-style check: rows of the matrix-free product vs the streaming
    row-sampled CPU oracle on an ico3 cavity (1280 el)."""
    import torch

    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import Assembler, MatrixFreeOperator
    from paper_1212_3032_b200.workloads import cavity_mesh

    mesh = cavity_mesh(3)
    mat = _unit()
    asm = Assembler(mesh, mat)
    om = 1.7 - 0.3j
    op = MatrixFreeOperator(asm, om)
    rng = np.random.default_rng(9)
    v = rng.normal(size=(mesh.n_dofs, 1)) + 1j * rng.normal(size=(mesh.n_dofs, 1))
    y = op(torch.from_numpy(v[:, 0].copy()).cuda()).cpu().numpy()
    rows = np.sort(rng.choice(mesh.n_elements, 24, replace=False))
    tv, _, _ = O.sampled_row_operator(mesh.vertices, mesh.triangles,
                                      O.Medium(mat.lam, mat.mu, mat.rho), rows, om, v, v,
                                      col_block=512)
    dof = (3 * rows[:, None] + np.arange(3)).ravel()
    assert rel_max(y[dof], tv[:, 0]) <= 1e-10


def test_pair_kernels_blocks_and_reduction_vs_oracle(cuda):
    """cfg3 microbenchmark kernels on a 48 x 40 x 3 subsample vs the oracle."""
    import ctypes

    import torch

    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import _lib
    from paper_1212_3032_b200.workloads import UNIT, cfg3_inputs

    lib = _lib.load()
    x, tris, om, xv = cfg3_inputs(48, 40, 3, seed=11)
    P, M, F = len(x), len(tris), len(om)
    xd = torch.from_numpy(x).cuda()
    td = torch.from_numpy(tris.reshape(M, 9).copy()).cuda()
    omh = np.ascontiguousarray(np.stack([om.real, om.imag], axis=1))
    u = torch.empty((F, P, M, 3, 3), dtype=torch.complex128, device="cuda")
    t = torch.empty_like(u)
    _lib.check(lib.ewb_pair_kernels_blocks(_lib.ptr(xd), P, _lib.ptr(td), M, omh.ctypes.data, F,
                                           UNIT.lam, UNIT.mu, UNIT.rho, _lib.ptr(u), _lib.ptr(t),
                                           _lib.stream_handle()))
    med = O.Medium(UNIT.lam, UNIT.mu, UNIT.rho)
    bary, wts = O.rule_g7()
    uref = np.empty((F, P, M, 3, 3), complex)
    tref = np.empty_like(uref)
    for m in range(M):
        v = tris[m]
        geo = O.element_geometry(v, np.array([[0, 1, 2]]))
        r, d, dn = O.pair_geom(x, bary @ v, geo["normals"][0])
        for f in range(F):
            ub, tb = O.blocks_dynamic(r, d, dn, wts * geo["areas"][0], geo["normals"][0], med, om[f])
            uref[f, :, m], tref[f, :, m] = ub, tb
    assert rel_max(u.cpu().numpy(), uref) <= 1e-10
    assert rel_max(t.cpu().numpy(), tref) <= 1e-10
    vd = torch.from_numpy(xv.copy()).cuda()
    yu = torch.empty((F, P, 3), dtype=torch.complex128, device="cuda")
    yt = torch.empty_like(yu)
    wsb = int(lib.ewb_pair_kernels_workspace_bytes(P, M, F))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.ewb_pair_kernels_reduce(_lib.ptr(xd), P, _lib.ptr(td), M, _lib.ptr(vd),
                                           omh.ctypes.data, F, UNIT.lam, UNIT.mu, UNIT.rho,
                                           _lib.ptr(yu), _lib.ptr(yt), _lib.ptr(ws), wsb,
                                           _lib.stream_handle()))
    assert rel_max(yu.cpu().numpy(), np.einsum("fpmab,mb->fpa", uref, xv)) <= 1e-10
    assert rel_max(yt.cpu().numpy(), np.einsum("fpmab,mb->fpa", tref, xv)) <= 1e-10
