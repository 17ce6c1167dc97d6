"""GPU: full-field reconstruction, CSV/manifest writers, exterior option,
SEM-off sweep, matrix-free sweep equals dense sweep."""

import numpy as np
import pytest

from conftest import rel_max

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    from test_gpu_solvers import _tiny_cfg

    return _tiny_cfg(**kw)


def test_full_field_histories_match_oracle_idft(cuda, tmp_path):
    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import emit_outputs, run_sweep

    cfg = _cfg(divisions=(2, 1, 1), n_omega=16)
    cfg.output_dir = tmp_path / "out"
    keep = []
    res = run_sweep(cfg, full_field=True, _sweep_out=keep)
    ds = keep[0]
    u_half = ds.displacement_field().cpu().numpy()          # (n_freq, N)
    field = res.full_field.cpu().numpy()                     # (N_omega, N)
    eta = O.eta_from_kappa(cfg.kappa, cfg.period)
    for d in (0, 5, cfg.mesh.n_dofs - 1):
        ref, _ = O.inverse_transform(O.conjugate_fill(u_half[:, d]), cfg.window, eta, cfg.period)
        assert rel_max(field[:, d], ref) <= 1e-12 or np.abs(ref).max() == 0.0
    # probe histories are the same columns
    p = cfg.probes[0]
    assert rel_max(res.histories[p.name], field[:, p.dof]) <= 1e-12
    written = emit_outputs(res, cfg)
    text = written["solve_stats"].read_text().splitlines()
    assert text[0] == "k,omega_re,omega_im,iterations,init_residual,final_residual,seconds"
    assert len(text) == 1 + cfg.n_omega // 2 + 1
    t, v = np.loadtxt(written[f"history_{p.name}"], delimiter=",", skiprows=1, unpack=True)
    assert np.array_equal(v, res.histories[p.name]) and np.array_equal(t, res.times)
    man = written["manifest"].read_text()
    assert f"n_elements = {cfg.mesh.n_elements}" in man and "gmres_tol = 1e-05" in man


def test_zero_load_and_linearity(cuda):
    from paper_1212_3032_b200 import TimeSignal, run_sweep

    cfg = _cfg()
    cfg.signals = [TimeSignal.zero(), TimeSignal.zero()]
    res = run_sweep(cfg)
    assert all(not np.any(h) for h in res.histories.values())
    cfg1 = _cfg()
    cfg2 = _cfg()
    cfg2.signals = [TimeSignal.zero(), TimeSignal.heaviside(-2e6)]
    r1, r2 = run_sweep(cfg1), run_sweep(cfg2)
    for name in r1.histories:
        assert rel_max(r2.histories[name], 2.0 * r1.histories[name]) <= 1e-6


def test_nonconverged_solves_poison_histories(cuda):
    from paper_1212_3032_b200 import run_sweep

    cfg = _cfg(maxiter=2, tol=1e-12)
    res = run_sweep(cfg)
    assert res.failed_frequencies
    assert all(np.isnan(h).all() for h in res.histories.values())


def test_exterior_option_shifts_t_diagonal_by_identity(cuda):
    from paper_1212_3032_b200 import Assembler, Material
    from paper_1212_3032_b200.workloads import cavity_mesh

    mesh = cavity_mesh(1)
    mat = Material.from_young_poisson(1.0, 0.25, 1.0)
    ti, _ = Assembler(mesh, mat).assemble_tu(1.2 - 0.3j, host=True)
    te, _ = Assembler(mesh, mat, exterior=True).assemble_tu(1.2 - 0.3j, host=True)
    d = te - ti
    assert np.abs(d - np.eye(mesh.n_dofs)).max() <= 1e-12


def test_matrix_free_sweep_equals_dense_sweep(cuda):
    from paper_1212_3032_b200 import run_sweep
    from paper_1212_3032_b200.workloads import sphere_pressure

    cfg = sphere_pressure(2, 16)
    dense = run_sweep(cfg, matrix_free=False)
    mf = run_sweep(cfg, matrix_free=True)
    for a, b in zip(dense.stats, mf.stats):
        assert abs(a.iterations - b.iterations) <= 1
    for name in dense.histories:
        h, href = mf.histories[name], dense.histories[name]
        assert np.linalg.norm(h - href) / np.linalg.norm(href) <= 1e-6
