"""Pin the CPU oracle to the reference: golden fixtures (always) and the live
reference package (build container only).  No GPU needed."""

import numpy as np
import pytest

from conftest import golden, rel_max
from oracle import ewbem_oracle as O

UNIT = O.Medium.young_poisson(1.0, 0.25, 1.0)
STEEL0 = O.Medium.young_poisson(2.11e11, 0.0, 7850.0)


def _box(lengths, div):
    from paper_1212_3032_b200.workloads import box_mesh

    return box_mesh(lengths, div)


def _ico(level):
    from paper_1212_3032_b200.workloads import cavity_mesh

    return cavity_mesh(level)


def test_rules_match_golden_bitwise():
    g = golden("small")
    b, w = O.rule_g3()
    assert np.array_equal(b, g["gauss3_pts"]) and np.array_equal(w, g["gauss3_w"])
    b, w = O.rule_g7()
    assert np.array_equal(b, g["gauss7_pts"]) and np.array_equal(w, g["gauss7_w"])
    for lvl in range(1, 5):
        b, w = O.rule_refine(O.rule_g7(), lvl)
        assert np.array_equal(b, g[f"sub{lvl}_pts"]) and np.array_equal(w, g[f"sub{lvl}_w"])
    y, w = O.self_points(g["self_verts"])
    assert np.array_equal(y, g["self_y"]) and np.array_equal(w, g["self_w"])


def test_radial_scalars_match_golden():
    g = golden("small")
    ks, kp = g["radial_k"]
    f = np.stack(O.radial_scalars(g["radial_r"], ks, kp))
    assert rel_max(f, g["radial_f"]) <= 1e-15
    assert rel_max(np.stack(O.static_scalars(g["radial_r"], UNIT)), g["static_f"]) <= 1e-15


def test_cube_assembly_matches_golden_bitwise():
    g = golden("small")
    asm = O.DenseOracle(g["cube_vertices"], g["cube_triangles"], UNIT)
    assert np.array_equal(asm.rowsums(), g["cube_rowsums"])
    for i, om in enumerate(g["cube_omegas"]):
        t, u = asm.tu(complex(om))
        assert rel_max(t, g[f"cube_T{i}"]) <= 1e-14
        assert rel_max(u, g[f"cube_U{i}"]) <= 1e-14


def test_rod32_and_ico1_match_golden():
    g = golden("small")
    m = _box((1, 1, 2), (2, 2, 1))
    t, u = O.DenseOracle(m.vertices, m.triangles, STEEL0).tu(2000.0 - 300.0j)
    assert rel_max(t, g["rod32_T"]) <= 1e-14 and rel_max(u, g["rod32_U"]) <= 1e-14
    m = _ico(1)
    t, u = O.DenseOracle(m.vertices, m.triangles, UNIT).tu(1.5 - 0.3j)
    assert rel_max(t, g["ico1_T"]) <= 1e-14 and rel_max(u, g["ico1_U"]) <= 1e-14


@pytest.mark.parametrize("name,builder", [
    ("cfg1", lambda: _box((1, 1, 1), (8, 8, 8))),
    ("rod", lambda: _box((3, 1, 1), (12, 4, 4))),
])
def test_tier_tables_match_golden_bitwise(name, builder):
    """The last-bit trap: 388 exact-4.0 ratios on the cube."""
    g = golden("tiers")
    m = builder()
    geo = O.element_geometry(m.vertices, m.triangles)
    tier = O.tier_table(geo["centroids"], geo["diameters"])
    n = int(g[f"{name}_n"])
    bits = np.unpackbits(g[f"{name}_tier"])[: 2 * n * n].reshape(2, n, n)
    assert np.array_equal(tier, bits[0] + 2 * bits[1])


def test_near_levels_match_golden():
    g = golden("tiers")
    m = _box((1, 1, 1), (8, 8, 8))
    geo = O.element_geometry(m.vertices, m.triangles)
    near = g["cfg1_near"]
    for j in np.unique(near[1])[:64]:
        sel = near[1] == j
        rows = near[0][sel]
        lv = O.near_level(O.surface_distance(geo["centroids"][rows], geo["corners"][j])
                          / geo["diameters"][j])
        assert np.array_equal(lv, near[2][sel])


def test_gmres_matches_golden_exactly():
    g = golden("linsolve")
    x, st = O.gmres(g["rod_A"], g["rod_b"], tol=1e-6, precond=O.block_precond(g["rod_A"])[0])
    assert st.iterations == int(g["rod_its"])
    assert rel_max(x, g["rod_x"]) <= 1e-12
    x, st = O.gmres(g["nc_A"], g["nc_b"], tol=1e-14, restart=5, maxiter=10)
    assert st.iterations == 10 and not st.converged
    assert rel_max(x, g["nc_x"]) <= 1e-12


def test_sem_matches_golden():
    g = golden("linsolve")
    hist = O.History(4)
    for c in g["sem_X"].T[::-1]:
        hist.push(c)
    assert rel_max(O.sem_guess(hist, g["sem_A"], g["sem_b"]), g["sem_x0"]) <= 1e-12


def test_transform_matches_golden():
    from paper_1212_3032_b200.transform import TimeSignal

    g = golden("transform")
    period, eta, n = float(g["period"]), float(g["eta"]), int(g["n"])
    assert np.array_equal(O.frequency_grid(period, n, eta), g["grid"])
    h = O.forward_spectrum(TimeSignal.heaviside(-1e6).sample(period, n), period, eta)
    assert rel_max(h, g["fwd_heaviside"]) <= 1e-15
    full = O.conjugate_fill(g["half"])
    assert np.array_equal(full, g["full"])
    for w in ("rectangular", "hanning", "blackman"):
        out, res = O.inverse_transform(full, w, eta, period)
        assert rel_max(out, g[f"inv_{w}"]) <= 1e-14 and res < 1e-12
        assert np.array_equal(O.window(w, n), g[f"win_{w}"])


def test_tiny_sweep_matches_golden():
    g = golden("sweeps")
    m = _box((3.0, 1.0, 1.0), (1, 1, 1))
    kinds = np.zeros((m.n_elements, 3), np.uint8)
    sig = np.zeros((m.n_elements, 3), np.int64)
    kinds[m.region_tag == 0] = 1
    sig[m.region_tag == 1, 0] = 1
    from paper_1212_3032_b200.workloads import face_center_element

    zm = np.flatnonzero(m.region_tag == 4)
    mid = int(zm[np.argmin(np.linalg.norm(m.centroids[zm] - np.array([1.5, 0.5, 0.0]), axis=1))])
    probes = [("tip_ux", 3 * face_center_element(m, 1), "displacement"),
              ("mid_ux", 3 * mid, "displacement"),
              ("root_tx", 3 * face_center_element(m, 0), "traction")]
    period, n = 0.0155, 8
    samples = [np.zeros(n), np.full(n, -1e6)]
    times, hists, stats, _ = O.sweep(m.vertices, m.triangles, STEEL0, kinds, sig.ravel(),
                                     samples, probes, period, n, 4.0, "hanning", 4, True, 1e-5)
    assert [s.iterations for s in stats] == list(g["tiny_its"])
    for name, _, _ in probes:
        assert rel_max(hists[name], g[f"tiny_h_{name}"]) <= 1e-9


# ----------------------------------------------------------------------
# live reference (build container only)
# ----------------------------------------------------------------------
def test_oracle_bitwise_equal_to_live_reference(reference):
    from ewbem.assembly import Assembler

    mesh = reference.generate_box_mesh((1, 1, 1), (2, 2, 2))
    mat = reference.Material.from_young_poisson(1.0, 0.25, 1.0)
    ra = Assembler(mesh, mat)
    oa = O.DenseOracle(mesh.vertices, mesh.triangles, O.Medium(mat.lam, mat.mu, mat.rho))
    for om in (0.0, -0.47j, 2.0 - 0.47j, 7.0 - 1.0j):
        t1, u1 = ra.assemble_tu(om)
        t2, u2 = oa.tu(om)
        assert np.array_equal(t1, t2) and np.array_equal(u1, u2)


def test_oracle_gmres_equal_to_live_reference(reference):
    from ewbem.linsolve import block_diag_precond, gmres

    rng = np.random.default_rng(2)
    a = rng.normal(size=(90, 90)) + 1j * rng.normal(size=(90, 90)) + 6 * np.eye(90)
    b = rng.normal(size=90) + 1j * rng.normal(size=90)
    x1, s1 = gmres(a, b, tol=1e-10, restart=15, precond=block_diag_precond(a))
    x2, s2 = O.gmres(a, b, tol=1e-10, restart=15, precond=O.block_precond(a)[0])
    assert s1.iterations == s2.iterations
    assert np.array_equal(x1, x2)
    assert s1.residual_history == s2.residual_history


def test_oracle_sampled_rows_equal_dense(reference):
    """The streaming row-sampled oracle (cfg5 checker) equals dense rows."""
    m = _ico(2)
    oa = O.DenseOracle(m.vertices, m.triangles, UNIT)
    om = 1.3 - 0.4j
    t, u = oa.tu(om)
    rng = np.random.default_rng(5)
    v = rng.normal(size=(m.n_dofs, 2)) + 1j * rng.normal(size=(m.n_dofs, 2))
    rows = np.array([0, 7, 100, 319])
    tv, uv, rs = O.sampled_row_operator(m.vertices, m.triangles, UNIT, rows, om, v, v,
                                        col_block=64)
    dof = (3 * rows[:, None] + np.arange(3)).ravel()
    assert rel_max(tv, t[dof] @ v) <= 1e-12
    assert rel_max(uv, u[dof] @ v) <= 1e-12
    assert rel_max(rs, oa.rowsums()[rows]) <= 1e-12
