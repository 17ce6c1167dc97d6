"""GPU parity: dense assembly, static pass, fused system vs golden + oracle.

Tolerance (north star): matrix entries within 1e-10 of max|entry|
(max-abs normalisation as test_assembly.py:70 uses).
"""

import numpy as np
import pytest

from conftest import golden, rel_max

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _unit():
    from paper_1212_3032_b200 import Material

    return Material.from_young_poisson(1.0, 0.25, 1.0)


def _steel():
    from paper_1212_3032_b200 import Material

    return Material.from_young_poisson(2.11e11, 0.0, 7850.0)


@pytest.fixture(scope="module")
def cube(cuda):
    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.workloads import box_mesh

    return Assembler(box_mesh((1, 1, 1), (2, 2, 2)), _unit())


def test_cube_tu_all_frequencies_match_golden(cube):
    g = golden("small")
    assert np.array_equal(cube.mesh.vertices, g["cube_vertices"])
    for i, om in enumerate(g["cube_omegas"]):
        t, u = cube.assemble_tu(complex(om), host=True)
        assert rel_max(t, g[f"cube_T{i}"]) <= TOL, (om, rel_max(t, g[f"cube_T{i}"]))
        assert rel_max(u, g[f"cube_U{i}"]) <= TOL, (om, rel_max(u, g[f"cube_U{i}"]))


def test_cube_rowsums_match_golden(cube):
    g = golden("small")
    assert rel_max(cube.static_offdiag_rowsums(), g["cube_rowsums"]) <= 1e-12


def test_rod32_steel_matches_golden(cuda):
    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.workloads import box_mesh

    g = golden("small")
    t, u = Assembler(box_mesh((1, 1, 2), (2, 2, 1)), _steel()).assemble_tu(
        2000.0 - 300.0j, host=True)
    assert rel_max(t, g["rod32_T"]) <= TOL
    assert rel_max(u, g["rod32_U"]) <= TOL


def test_flipped_icosphere_matches_golden(cuda):
    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.workloads import cavity_mesh

    g = golden("small")
    t, u = Assembler(cavity_mesh(1), _unit()).assemble_tu(
        1.5 - 0.3j, host=True)
    assert rel_max(t, g["ico1_T"]) <= TOL
    assert rel_max(u, g["ico1_U"]) <= TOL


@pytest.fixture(scope="module")
def cfg1_asm(cuda):
    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.workloads import box_mesh

    return Assembler(box_mesh((1, 1, 1), (8, 8, 8)), _unit())


def test_cfg1_pair_census_matches_reference_tiers(cfg1_asm):
    """GPU exact-rounding tiers == numpy tiers on the box mesh with 388 ties."""
    g = golden("tiers")
    n = int(g["cfg1_n"])
    bits = np.unpackbits(g["cfg1_tier"])[: 2 * n * n].reshape(2, n, n)
    tier = bits[0] + 2 * bits[1]
    off = ~np.eye(n, dtype=bool)
    pc = cfg1_asm.pair_counts()
    assert pc["far"] == int(((tier == 0) & off).sum())
    assert pc["mid"] == int(((tier == 1) & off).sum())
    assert pc["near"] == int(((tier == 2) & off).sum())
    near = g["cfg1_near"]
    for lvl in (1, 2, 3, 4):
        assert pc["near_levels"][lvl] == int((near[2] == lvl).sum())
    assert cfg1_asm.point_evals() == 4825892


def test_cfg1_rows_diagonals_and_matvecs_match_golden(cfg1_asm):
    from paper_1212_3032_b200.transform import eta_from_kappa, frequency_grid

    g = golden("cfg1_rows")
    c_s = _unit().c_s
    period = 8.0 / c_s
    om = frequency_grid(period, 128, eta_from_kappa(6.0 / np.log(10.0), period))
    elems = g["elements"]
    rows = (3 * elems[:, None] + np.arange(3)).ravel()
    assert rel_max(cfg1_asm.static_offdiag_rowsums(), g["rowsums"]) <= 1e-12
    v = g["v"]
    for k in (1, 64):
        t, u = cfg1_asm.assemble_tu(om[k], host=True)
        tmax, umax = float(g[f"Tmax_k{k}"]), float(g[f"Umax_k{k}"])
        assert np.abs(t[rows] - g[f"T_rows_k{k}"]).max() <= TOL * tmax
        assert np.abs(u[rows] - g[f"U_rows_k{k}"]).max() <= TOL * umax
        tb, ub = t.reshape(768, 3, 768, 3), u.reshape(768, 3, 768, 3)
        ids = np.arange(768)
        assert np.abs(tb[ids, :, ids, :] - g[f"T_diag_k{k}"]).max() <= TOL * tmax
        assert np.abs(ub[ids, :, ids, :] - g[f"U_diag_k{k}"]).max() <= TOL * umax
        assert rel_max(t @ v, g[f"Tv_k{k}"]) <= TOL
        assert rel_max(u @ v, g[f"Uv_k{k}"]) <= TOL


def test_assembly_is_bit_deterministic(cube):
    t1, u1 = cube.assemble_tu(0.7 - 0.2j, host=True)
    t2, u2 = cube.assemble_tu(0.7 - 0.2j, host=True)
    assert np.array_equal(t1, t2) and np.array_equal(u1, u2)


def test_conjugate_reflection(cube):
    om = 4.05 - 0.594j
    t, u = cube.assemble_tu(om, host=True)
    tr, ur = cube.assemble_tu(-np.conj(om), host=True)
    assert np.abs(tr - np.conj(t)).max() <= 1e-12 * np.abs(t).max()
    assert np.abs(ur - np.conj(u)).max() <= 1e-12 * np.abs(u).max()


def test_rigid_body_rowsum_near_static(cube):
    t, _ = cube.assemble_tu(-1e-6j, host=True)
    ones = np.tile(np.eye(3), (cube.mesh.n_elements, 1))
    assert np.abs(t @ ones).max() <= 1e-7 * np.abs(t).max()
    ts, _ = cube.assemble_static_tu(host=True)
    assert np.abs(ts @ ones).max() <= 1e-12 * np.abs(ts).max()


def test_positive_imaginary_frequency_rejected(cube):
    with pytest.raises(ValueError, match="positive imaginary"):
        cube.assemble_tu(1.0 + 0.5j)


def _rod_bcs(mesh):
    from paper_1212_3032_b200 import DIRICHLET, NEUMANN, BoundaryConditionSet

    bcs = BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.set_region(mesh, 0, (0, 1, 2), DIRICHLET, 0)
    bcs.set_region(mesh, 1, (0,), NEUMANN, 1)
    return bcs


def test_fused_system_equals_oracle_apply_bcs(cube):
    from oracle import ewbem_oracle as O

    g = golden("small")
    rng = np.random.default_rng(3)
    bcs = _rod_bcs(cube.mesh)
    p = rng.normal(size=cube.n) + 1j * rng.normal(size=cube.n)
    om = complex(g["cube_omegas"][3])
    a_ref, b_ref = O.apply_bcs(g["cube_T3"], g["cube_U3"], bcs.flat_kind(), p)
    sysm = cube.assemble_system(om, bcs, p)
    a = sysm.A.cpu().numpy()
    assert rel_max(a, a_ref) <= TOL
    assert rel_max(sysm.b.cpu().numpy(), b_ref) <= TOL
    _, inv = O.block_precond(a_ref)
    assert rel_max(sysm.pinv.cpu().numpy(), inv) <= 1e-9


def test_apply_bcs_device_matches_oracle(cube):
    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import apply_bcs, scatter_solution

    g = golden("small")
    rng = np.random.default_rng(8)
    bcs = _rod_bcs(cube.mesh)
    p = rng.normal(size=cube.n) + 1j * rng.normal(size=cube.n)
    a_ref, b_ref = O.apply_bcs(g["cube_T2"], g["cube_U2"], bcs.flat_kind(), p)
    sysm = apply_bcs(g["cube_T2"], g["cube_U2"], bcs, p)
    assert np.array_equal(sysm.A.cpu().numpy(), a_ref)
    assert rel_max(sysm.b.cpu().numpy(), b_ref) <= 1e-13
    with pytest.raises(ValueError, match="unresolved"):
        apply_bcs(g["cube_T2"], g["cube_U2"], bcs, np.full(cube.n, np.nan, complex))
    with pytest.raises(ValueError, match="length"):
        apply_bcs(g["cube_T2"], g["cube_U2"], bcs, np.zeros(3, complex))
    a = np.linalg.solve(a_ref, b_ref)
    u, t = scatter_solution(sysm, a, p)
    kinds = bcs.flat_kind()
    assert np.array_equal(u.cpu().numpy()[kinds == 1], p[kinds == 1])
    assert np.array_equal(t.cpu().numpy()[kinds == 0], p[kinds == 0])


# ---------------------------------------------------------------------------
# multi-frequency system assembly (ewb_assemble_system_multi)
# ---------------------------------------------------------------------------
def _cfg1_bcs(mesh):
    from paper_1212_3032_b200 import DIRICHLET, NEUMANN, BoundaryConditionSet

    bcs = BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.set_region(mesh, 4, (0, 1, 2), DIRICHLET, 0)
    bcs.set_region(mesh, 5, (2,), NEUMANN, 1)
    return bcs


def _cfg1_omegas():
    from paper_1212_3032_b200.transform import eta_from_kappa, frequency_grid

    period = 8.0 / _unit().c_s
    return frequency_grid(period, 128, eta_from_kappa(6.0 / np.log(10.0), period))


@pytest.mark.parametrize("ks", [list(range(0, 8)), list(range(57, 65)), [1, 2, 3, 4],
                                [3, 9, 10, 40, 41], [20]])
def test_multi_frequency_system_equals_single(cfg1_asm, ks):
    """Each batch member == the single-frequency fused system (phase recurrence for
    the equispaced batches, direct evaluation for the others)."""
    import torch

    om = _cfg1_omegas()
    mesh = cfg1_asm.mesh
    bcs = _cfg1_bcs(mesh)
    rng = np.random.default_rng(11)
    n = cfg1_asm.n
    P = rng.normal(size=(len(ks), n)) + 1j * rng.normal(size=(len(ks), n))
    batch = cfg1_asm.assemble_system_multi([om[k] for k in ks], bcs, P)
    for f, k in enumerate(ks):
        ref = cfg1_asm.assemble_system(om[k], bcs, P[f])
        m = batch.member(f)
        amax = torch.abs(ref.A).max().item()
        assert torch.abs(m.A - ref.A).max().item() <= 1e-13 * amax, (k, f)
        assert torch.abs(m.b - ref.b).max().item() <= 1e-12 * torch.abs(ref.b).max().item()
        assert torch.abs(m.pinv - ref.pinv).max().item() <= 1e-10 * torch.abs(ref.pinv).max().item()


def test_multi_frequency_rows_match_reference_golden(cfg1_asm):
    """Batch members at k = 1 and k = 64 against the live reference's T/U rows."""
    g = golden("cfg1_rows")
    om = _cfg1_omegas()
    bcs = _cfg1_bcs(cfg1_asm.mesh)
    kinds = bcs.flat_kind()
    n = cfg1_asm.n
    elems = g["elements"]
    rows = (3 * elems[:, None] + np.arange(3)).ravel()
    p = np.zeros(n, complex)
    p[kinds == 0] = 0.3 - 0.1j
    for ks in ([1, 2, 3, 4, 5, 6, 7, 8], [57, 58, 59, 60, 61, 62, 63, 64]):
        batch = cfg1_asm.assemble_system_multi([om[k] for k in ks], bcs, np.tile(p, (8, 1)))
        for k in (1, 64):
            if k not in ks:
                continue
            f = ks.index(k)
            a_rows = batch.A[f].cpu().numpy()[rows]
            t_rows, u_rows = g[f"T_rows_k{k}"], g[f"U_rows_k{k}"]
            a_ref = np.where(kinds[None, :] == 1, -u_rows, t_rows)
            amax = max(float(g[f"Tmax_k{k}"]), float(g[f"Umax_k{k}"]))
            assert np.abs(a_rows - a_ref).max() <= TOL * amax, k
            neu, dirc = kinds == 0, kinds == 1
            b_ref = u_rows[:, neu] @ p[neu] - t_rows[:, dirc] @ p[dirc]   # assembly.py:295-296
            b_rows = batch.b[f].cpu().numpy()[rows]
            assert rel_max(b_rows, b_ref) <= TOL


def test_multi_frequency_is_bit_deterministic_and_validates(cfg1_asm):
    om = _cfg1_omegas()
    bcs = _cfg1_bcs(cfg1_asm.mesh)
    P = np.ones((4, cfg1_asm.n), complex)
    a = cfg1_asm.assemble_system_multi(om[10:14], bcs, P)
    A1, b1 = a.A.cpu().numpy(), a.b.cpu().numpy()
    a = cfg1_asm.assemble_system_multi(om[10:14], bcs, P, out=a)
    assert np.array_equal(A1, a.A.cpu().numpy()) and np.array_equal(b1, a.b.cpu().numpy())
    with pytest.raises(ValueError, match="static path"):
        cfg1_asm.assemble_system_multi([0.0, 1.0 - 0.1j], bcs, P[:2])
    with pytest.raises(ValueError, match="positive imaginary"):
        cfg1_asm.assemble_system_multi([1.0 + 0.5j], bcs, P[:1])
    with pytest.raises(ValueError, match="batch of 33"):
        cfg1_asm.assemble_system_multi(om[:33], bcs, np.ones((33, cfg1_asm.n), complex))
    with pytest.raises(ValueError, match=r"\(nf, N\)"):
        cfg1_asm.assemble_system_multi(om[1:3], bcs, P)


def test_non_finite_entries_raise_per_member(cuda):
    """A duplicated element puts a quadrature node on a collocation point
    (r = 0; the reference's pair_geometry raises there, kernels.py:196-203):
    every member of a batch flags non-finite entries -> FloatingPointError,
    and the sweep reports the first frequency (driver.py:141-145)."""
    import dataclasses

    from paper_1212_3032_b200 import Assembler, SurfaceMesh, SweepError, run_sweep
    from paper_1212_3032_b200.workloads import box_mesh, cfg1

    m = box_mesh((1, 1, 1), (2, 2, 2))
    tris = np.vstack([m.triangles, m.triangles[:1]])
    tags = np.concatenate([m.region_tag, m.region_tag[:1]])
    mesh = SurfaceMesh(m.vertices, tris, tags)
    asm = Assembler(mesh, _unit())
    bcs = _cfg1_bcs(mesh)
    P = np.ones((3, mesh.n_dofs), complex)
    with pytest.raises(FloatingPointError, match="non-finite"):
        asm.assemble_system_multi([1.0 - 0.2j, 1.5 - 0.2j, 2.0 - 0.2j], bcs, P)
    cfg = dataclasses.replace(cfg1(), mesh=mesh, bcs=bcs, probes=[], allow_floating=True)
    with pytest.raises(SweepError, match="frequency index 0"):
        run_sweep(cfg)


def test_device_sincos_exp_vs_libm(cuda):
    """fast_sincos / fast_exp (the kernel phases e^{-i z}, kernels.py:103-104)
    against numpy's libm: <= 2 ulp on the BEM argument ranges, the libdevice
    path beyond |x| = 1e5, NaN / inf / underflow behaviour."""
    import ctypes

    from paper_1212_3032_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(1212)
    x = np.concatenate([rng.uniform(-4, 4, 400_000), rng.uniform(-200, 200, 400_000),
                        rng.uniform(-1e5, 1e5, 200_000), rng.uniform(-746, 0, 400_000),
                        10.0 ** rng.uniform(-300, -2, 100_000),
                        np.arange(-2000, 2000) * (np.pi / 2),
                        [0.0, -0.0, 1e6, -3e7, 1e300, np.inf, -np.inf, np.nan, 709.7, 710.0,
                         -745.0, -746.0, -800.0]])
    n = len(x)
    s, c, e = np.empty(n), np.empty(n), np.empty(n)
    _lib.check(lib.ewb_math_selftest(x.ctypes.data, n, s.ctypes.data, c.ctypes.data,
                                     e.ctypes.data, _lib.stream_handle()))
    with np.errstate(all="ignore"):
        rs, rc, re_ = np.sin(x), np.cos(x), np.exp(x)
    fin = np.isfinite(x)
    for got, ref in ((s, rs), (c, rc)):
        assert np.array_equal(np.isnan(got), np.isnan(ref))
        m = fin & (np.abs(x) <= 1e5)
        ulp = np.abs(got[m] - ref[m]) / np.spacing(np.maximum(np.abs(ref[m]), 1e-300))
        big = np.abs(ref[m]) >= 1e-3     # near a zero of sin/cos: absolute error instead
        assert ulp[big].max() <= 2.0, ulp[big].max()
        assert np.abs(got[m] - ref[m])[~big].max() <= 1e-19 * max(1.0, np.abs(x[m]).max())
    m = fin & (x < 709.5) & (x > -708)
    ulp = np.abs(e[m] - re_[m]) / np.spacing(re_[m])
    assert ulp.max() <= 2.0, ulp.max()
    assert np.isnan(e[np.isnan(x)]).all() and e[x == np.inf][0] == np.inf
    assert e[x == -np.inf][0] == 0.0 and e[x == -800.0][0] == 0.0 and e[x == 710.0][0] == np.inf
    assert e[x == -745.0][0] <= 1e-323
    # exp_small: the damping-factor step between a far pair's quadrature points
    t = np.concatenate([rng.uniform(-0.0625, 0.0625, 300_000), rng.uniform(-1e-3, 1e-3, 100_000),
                        10.0 ** rng.uniform(-300, -3, 50_000), [0.0, -0.0, 0.0625, -0.0625]])
    es = np.empty(len(t))
    _lib.check(lib.ewb_math_selftest_delta(t.ctypes.data, len(t), es.ctypes.data,
                                           _lib.stream_handle()))
    ulp = np.abs(es - np.exp(t)) / np.spacing(np.exp(t))
    assert ulp.max() <= 1.0, ulp.max()
    assert lib.ewb_math_selftest_delta(np.array([0.07]).ctypes.data, 1, es.ctypes.data,
                                       _lib.stream_handle()) != 0
