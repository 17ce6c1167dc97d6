"""GPU parity: GMRES, block preconditioner, SEM, time reconstruction, sweeps."""

import numpy as np
import pytest

from conftest import golden, rel_max

pytestmark = pytest.mark.gpu


def test_gmres_random_system_matches_golden(cuda):
    from paper_1212_3032_b200 import gmres

    g = golden("linsolve")
    x, st = gmres(g["rand_A"], g["rand_b"], tol=1e-12, restart=20)
    # the golden run stalls at maxiter=1000 (restart 20 on a hard system);
    # our run must walk the same path: same count, same monotone cycles
    assert st.iterations == int(g["rand_its"])
    h = np.array(st.residual_history)
    ref = g["rand_hist"]
    assert len(h) == len(ref)
    assert np.abs(np.log10(h[:200]) - np.log10(ref[:200])).max() < 1e-3


def test_gmres_rod_bem_system_with_block_precond(cuda):
    from paper_1212_3032_b200 import block_diag_precond, gmres

    g = golden("linsolve")
    a, b = g["rod_A"], g["rod_b"]
    x, st = gmres(a, b, tol=1e-6, precond=block_diag_precond(a))
    assert st.converged
    assert abs(st.iterations - int(g["rod_its"])) <= 1
    x_direct = np.linalg.solve(a, b)
    assert np.abs(x.cpu().numpy() - x_direct).max() <= 1e-4 * np.abs(x_direct).max()


def test_gmres_nonconvergence_flagged(cuda):
    from paper_1212_3032_b200 import gmres

    g = golden("linsolve")
    x, st = gmres(g["nc_A"], g["nc_b"], tol=1e-14, restart=5, maxiter=10)
    assert not st.converged
    assert st.iterations == 10
    assert st.final_residual > 1e-14
    assert np.isfinite(x.cpu().numpy()).all()
    assert abs(st.final_residual - float(g["nc_final"])) <= 1e-10


def test_gmres_edge_cases(cuda):
    from paper_1212_3032_b200 import gmres

    rng = np.random.default_rng(0)
    b = rng.normal(size=30) + 1j * rng.normal(size=30)
    x, st = gmres(np.eye(30, dtype=complex), b, tol=1e-10)
    assert st.iterations == 1 and st.converged
    np.testing.assert_allclose(x.cpu().numpy(), b, rtol=1e-12)
    x, st = gmres(np.eye(5, dtype=complex), np.zeros(5, complex))
    assert st.iterations == 0 and not x.cpu().numpy().any()
    with pytest.raises(ValueError):
        gmres(np.eye(3, dtype=complex), np.ones(3, complex), tol=0.0)
    a = rng.normal(size=(64, 64)) + 1j * rng.normal(size=(64, 64)) + 10 * np.eye(64)
    bb = rng.normal(size=64) + 1j * rng.normal(size=64)
    xe = np.linalg.solve(a, bb)
    x, st = gmres(a, bb, x0=xe, tol=1e-6)
    assert st.iterations == 0 and st.init_residual <= 1e-12


def test_block_diag_precond_identity_and_singular(cuda):
    from paper_1212_3032_b200 import block_diag_precond

    rng = np.random.default_rng(5)
    n = 60
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)) + 4 * np.eye(n)
    pc = block_diag_precond(a)
    import torch

    pa = torch.stack([pc(torch.from_numpy(a[:, i]).cuda()) for i in range(n)], dim=1).cpu().numpy()
    for i in range(n // 3):
        assert np.abs(pa[3 * i:3 * i + 3, 3 * i:3 * i + 3] - np.eye(3)).max() <= 1e-13
    s = np.eye(6, dtype=complex)
    s[3:6, 3:6] = 0.0
    pc = block_diag_precond(s)
    v = np.arange(6.0).astype(complex)
    np.testing.assert_allclose(pc(torch.from_numpy(v).cuda()).cpu().numpy(), v)
    with pytest.raises(ValueError):
        block_diag_precond(np.eye(4, dtype=complex))


def test_sem_matches_golden(cuda):
    from paper_1212_3032_b200 import SolutionHistory, sem_initial_guess

    g = golden("linsolve")
    hist = SolutionHistory(4)
    X = g["sem_X"]
    for c in X.T[::-1]:
        hist.push(c)
    x0 = sem_initial_guess(hist, g["sem_A"], g["sem_b"]).cpu().numpy()
    assert rel_max(x0, g["sem_x0"]) <= 1e-10
    hist2 = SolutionHistory(3)
    for c in g["sem2_X"].T[::-1]:
        hist2.push(c)
    x0 = sem_initial_guess(hist2, g["sem_A"], g["sem2_b"]).cpu().numpy()
    a = g["sem_A"]
    assert np.linalg.norm(a @ x0 - g["sem2_b"]) <= 1e-9 * np.linalg.norm(g["sem2_b"])


def test_window_idft_matches_golden(cuda):
    import torch

    from paper_1212_3032_b200.transform import Spectrum, inverse_mft, windowed_inverse_device

    g = golden("transform")
    period, eta = float(g["period"]), float(g["eta"])
    half = g["half"]
    for w in ("rectangular", "hanning", "blackman"):
        out = inverse_mft(Spectrum(g["full"], period, eta), w, eta)
        assert rel_max(out, g[f"inv_{w}"]) <= 1e-12
    # many columns at once
    cols = np.stack([half, 2 * half, half * (1 - 1j)], axis=1)
    out, res = windowed_inverse_device(torch.from_numpy(cols).cuda(), "hanning", eta, period)
    out = out.cpu().numpy()
    assert rel_max(out[:, 0], g["inv_hanning"]) <= 1e-12
    assert rel_max(out[:, 1], 2 * g["inv_hanning"]) <= 1e-12
    assert float(res.max()) < 1e-12


def _tiny_cfg(**kw):
    from paper_1212_3032_b200 import (DIRICHLET, NEUMANN, BoundaryConditionSet, Material, Probe,
                                      SweepSpec, TimeSignal)
    from paper_1212_3032_b200.workloads import box_mesh, face_center_element

    divisions = kw.pop("divisions", (1, 1, 1))
    mesh = box_mesh((3.0, 1.0, 1.0), divisions)
    zm = np.flatnonzero(mesh.region_tag == 4)
    mid = int(zm[np.argmin(np.linalg.norm(mesh.centroids[zm] - np.array([1.5, 0.5, 0.0]),
                                          axis=1))])
    bcs = BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.set_region(mesh, 0, (0, 1, 2), DIRICHLET, 0)
    bcs.set_region(mesh, 1, (0,), NEUMANN, 1)
    args = dict(n_omega=8, kappa=4.0, window="hanning", sem_enabled=True, sem_depth=4, tol=1e-5)
    args.update(kw)
    return SweepSpec(
        mesh=mesh, material=Material.from_young_poisson(2.11e11, 0.0, 7850.0), bcs=bcs,
        signals=[TimeSignal.zero(), TimeSignal.heaviside(-1e6)], signal_names=["zero", "load"],
        probes=[Probe("tip_ux", face_center_element(mesh, 1), 0, "displacement"),
                Probe("mid_ux", mid, 0, "displacement"),
                Probe("root_tx", face_center_element(mesh, 0), 0, "traction")],
        period=0.0155, figures=False, **args)


def _check_sweep(res, g, prefix, its_tol=1, hist_tol=1e-6):
    its = np.array([s.iterations for s in res.stats])
    ref = g[f"{prefix}_its"]
    assert np.abs(its - ref).max() <= its_tol, (its, ref)
    for name in g[f"{prefix}_probes"]:
        h = res.histories[str(name)]
        href = g[f"{prefix}_h_{name}"]
        err = np.linalg.norm(h - href) / np.linalg.norm(href)
        assert err <= hist_tol, (name, err)


@pytest.mark.parametrize("prefix,kw", [("tiny", {}), ("tiny_nosem", {"sem_enabled": False}),
                                       ("rod622", {"divisions": (6, 2, 2), "n_omega": 32})])
def test_small_sweeps_match_golden(cuda, prefix, kw):
    from paper_1212_3032_b200 import run_sweep

    g = golden("sweeps")
    res = run_sweep(_tiny_cfg(**kw))
    _check_sweep(res, g, prefix)


def test_cfg1_stepwise_iterations_equal_reference(cuda):
    """BASELINE cfg1, every frequency: our SEM + GMRES fed the reference's own
    solution history reproduce the reference's iteration count (+-1) and its
    solution (1e-6).  This isolates per-solve parity from history drift."""
    import torch

    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.linsolve import gmres_device, sem_device
    from paper_1212_3032_b200.transform import eta_from_kappa, forward_mft, frequency_grid
    from paper_1212_3032_b200.workloads import cfg1

    g = golden("cfg1_solutions")
    cfg = cfg1()
    asm = Assembler(cfg.mesh, cfg.material)
    eta = eta_from_kappa(cfg.kappa, cfg.period)
    om = frequency_grid(cfg.period, cfg.n_omega, eta)
    spectra = np.stack([forward_mft(s, cfg.period, cfg.n_omega, eta).values for s in cfg.signals])
    sig = cfg.bcs.flat_signal()
    xref = g["x"]
    x = torch.zeros(cfg.mesh.n_dofs, dtype=torch.complex128, device="cuda")
    sysm = None
    diffs = []
    for k in range(len(om)):
        sysm = asm.assemble_system(om[k], cfg.bcs, spectra[sig, k], out=sysm)
        if k:
            hist = torch.from_numpy(xref[max(0, k - 2):k][::-1].copy()).cuda()
            sem_device(sysm.A, sysm.b, hist, 1e-10, x)
        st = gmres_device(sysm.A, sysm.b, x, k > 0, cfg.tol, cfg.restart, cfg.maxiter, sysm.pinv)
        diffs.append(st.iterations - int(g["its"][k]))
        assert abs(st.init_residual - g["init"][k]) <= 1e-6 * g["init"][k] + 1e-14
        assert rel_max(x.cpu().numpy(), xref[k]) <= 1e-6
    assert max(abs(d) for d in diffs) <= 1, diffs


def _reference_solver_chain(ds, cfg):
    """The reference's solver (the oracle: bitwise equal to linsolve.py's
    sem_initial_guess / block_diag_precond / gmres) run as the chained sweep
    (driver.py:128-153) on the SAME systems the device sweep assembled —
    re-assembled here in the sweep's own batches (bit-reproducible kernels)
    and read back.  Returns the per-k iteration counts."""
    from oracle import ewbem_oracle as O

    nb = ds.batch_size()
    hist = O.History(cfg.sem_depth)
    its = []
    batch = None
    for k0 in range(0, ds.n_freq, nb):
        ks = list(range(k0, min(ds.n_freq, k0 + nb)))
        batch = ds.asm.assemble_system_multi([ds.omegas[k] for k in ks], cfg.bcs,
                                             ds.P[ks[0]:ks[-1] + 1], out=batch, check=False)
        for f in range(len(ks)):
            m = batch.member(f)
            a, b = m.A.cpu().numpy(), m.b.cpu().numpy()
            x0 = O.sem_guess(hist, a, b) if len(hist) else None
            pc, _ = O.block_precond(a)
            x, st = O.gmres(a, b, x0=x0, tol=cfg.tol, restart=cfg.restart, maxiter=cfg.maxiter,
                            precond=pc)
            its.append(st.iterations)
            hist.push(x)
    return np.array(its)


def test_cfg1_sweep_matches_reference_run(cuda):
    """BASELINE cfg1 end to end (65 SEM-chained solves, tol 1e-8, K=2).

    Iterations +-1 on EVERY frequency against the reference's solver chained
    over the same assembled systems, on this box (the same-input comparison).
    Against the reference's own run (golden, reference-assembled matrices):
    histories 1e-6; counts differ by <= 2 at a few k.  That residue is the
    chain's sensitivity, not the solver: the reference's own solver chained
    over our matrices (which equal the reference's to 2.3e-15 of max|A|)
    shows the same deviation from the golden run (tools/diag_chain.py:
    k = 4 -> -2, k = 5 -> -1 for both)."""
    from paper_1212_3032_b200 import run_sweep
    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.workloads import cfg1

    g = golden("cfg1_sweep")
    cfg = cfg1()
    res = run_sweep(cfg)
    its = np.array([s.iterations for s in res.stats])
    ref_same = _reference_solver_chain(DeviceSweep(cfg), cfg)
    assert np.abs(its - ref_same).max() <= 1, (its - ref_same).tolist()
    d = np.abs(its - g["cfg1_its"])
    assert d.max() <= 2 and (d <= 1).mean() >= 0.95, d
    assert abs(its.sum() - g["cfg1_its"].sum()) <= 0.01 * g["cfg1_its"].sum()
    for name in g["cfg1_probes"]:
        h, href = res.histories[str(name)], g[f"cfg1_h_{name}"]
        assert np.linalg.norm(h - href) / np.linalg.norm(href) <= 1e-6
    assert not res.failed_frequencies


def test_cfg2_head_matches_reference(cuda):
    """BASELINE cfg2 (ico4, 15360 DOF): full-size T v / U v at k=1 and the first
    three SEM solves (iterations +-1, solutions 1e-6)."""
    import torch

    from paper_1212_3032_b200 import Assembler, BoundaryConditionSet, SolutionHistory
    from paper_1212_3032_b200.linsolve import gmres_device, sem_device
    from paper_1212_3032_b200.workloads import cfg2

    g = golden("cfg2_head")
    cfg = cfg2()
    asm = Assembler(cfg.mesh, cfg.material)
    t, u = asm.assemble_tu(complex(g["omegas"][1]))
    v = torch.from_numpy(g["v"]).cuda()
    assert rel_max((t @ v).cpu().numpy(), g["Tv_k1"]) <= 1e-10
    assert rel_max((u @ v).cpu().numpy(), g["Uv_k1"]) <= 1e-10
    assert np.abs(t[:3].cpu().numpy() - g["T_row0_k1"]).max() <= 1e-10 * float(g["Tmax_k1"])
    assert np.abs(u[:3].cpu().numpy() - g["U_row0_k1"]).max() <= 1e-10 * float(g["Umax_k1"])
    del t, u
    torch.cuda.empty_cache()
    bcs = BoundaryConditionSet.traction_free(cfg.mesh.n_elements)
    load = (-1.0 * cfg.mesh.normals).ravel()
    hist = torch.zeros((4, cfg.mesh.n_dofs), dtype=torch.complex128, device="cuda")
    x = torch.zeros(cfg.mesh.n_dofs, dtype=torch.complex128, device="cuda")
    sysm = None
    for k in range(3):
        p = load * g["unit_spec"][k]
        sysm = asm.assemble_system(complex(g["omegas"][k]), bcs, p, out=sysm)
        if k:
            sem_device(sysm.A, sysm.b, hist[:k], 1e-10, x)
        st = gmres_device(sysm.A, sysm.b, x, k > 0, 1e-8, 60, 1000, sysm.pinv)
        assert abs(st.iterations - int(g["its"][k])) <= 1, (k, st.iterations, g["its"][k])
        assert rel_max(x.cpu().numpy(), g["x"][k]) <= 1e-6
        hist[1:] = hist[:-1].clone()
        hist[0] = x


def test_cfg2_stepwise_iterations_equal_reference(cuda):
    """BASELINE cfg2 at k = 32, 64, 128 (low, middle, top of the sweep): fed the
    live reference's own four previous solutions (cfg2_sweep.npz), our SEM +
    GMRES reproduce the reference's iteration count (+-1), SEM initial
    residual and solution (1e-6)."""
    import torch

    from conftest import GOLDEN
    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.linsolve import gmres_device, sem_device
    from paper_1212_3032_b200.workloads import cfg2

    if not (GOLDEN / "cfg2_sweep.npz").exists():
        pytest.skip("cfg2_sweep.npz not generated")
    g = golden("cfg2_sweep")
    keep = {int(k): x for k, x in zip(g["keep_k"], g["keep_x"])}
    cfg = cfg2()
    ds = DeviceSweep(cfg, frequencies=[0])
    x = torch.zeros(ds.n, dtype=torch.complex128, device="cuda")
    sysm = None
    for k in (32, 64, 128):
        sysm = ds.asm.assemble_system(ds.omegas[k], cfg.bcs, ds.P[k], out=sysm)
        hist = torch.from_numpy(np.stack([keep[k - 1 - i] for i in range(4)])).cuda()
        sem_device(sysm.A, sysm.b, hist, 1e-10, x)
        st = gmres_device(sysm.A, sysm.b, x, True, cfg.tol, cfg.restart, cfg.maxiter, sysm.pinv)
        assert abs(st.iterations - int(g["cfg2_its"][k])) <= 1, (k, st.iterations, g["cfg2_its"][k])
        assert abs(st.init_residual - g["cfg2_init"][k]) <= 1e-4 * g["cfg2_init"][k], k
        assert rel_max(x.cpu().numpy(), keep[k]) <= 1e-6, k
        assert st.converged and st.final_residual <= cfg.tol


def test_cfg2_stepwise_all_frequencies(cuda):
    """BASELINE cfg2, all 129 frequencies, through the sweep's own
    multi-frequency assembly batches: each frequency fed the live reference's
    four previous solutions (tests/golden/cfg2_solutions.npz, a second run of
    the reference's run_sweep that keeps every solution) reproduces the
    reference's iteration count (+-1) and solution (1e-6), and the probe
    histories built from these per-frequency solutions match the reference's
    (1e-6 relative L2) — per-frequency parity without the chain's
    sensitivity (test_cfg2_full_sweep_matches_reference_run)."""
    import torch

    from conftest import GOLDEN
    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.linsolve import gmres_device, sem_device
    from paper_1212_3032_b200.transform import windowed_inverse_device
    from paper_1212_3032_b200.workloads import cfg2

    if not (GOLDEN / "cfg2_solutions.npz").exists():
        pytest.skip("cfg2_solutions.npz not generated")
    g = golden("cfg2_solutions")
    gs = golden("cfg2_sweep")
    xs, its_ref = g["x"], g["its"]
    cfg = cfg2()
    ds = DeviceSweep(cfg, frequencies=[0])
    nf, nb = ds.n_freq, 16
    assert xs.shape == (nf, ds.n)
    x = torch.zeros(ds.n, dtype=torch.complex128, device="cuda")
    half = torch.zeros((nf, len(cfg.probes)), dtype=torch.complex128, device="cuda")
    dofs = torch.tensor([p.dof for p in cfg.probes], device="cuda")
    d, sol_err, batch = [], 0.0, None
    for k0 in range(0, nf, nb):
        ks = list(range(k0, min(nf, k0 + nb)))
        batch = ds.asm.assemble_system_multi([ds.omegas[k] for k in ks], cfg.bcs,
                                             ds.P[ks[0]:ks[-1] + 1], out=batch, check=False)
        for f, k in enumerate(ks):
            m = batch.member(f)
            if k:
                hist = torch.from_numpy(np.stack([xs[k - 1 - i] for i in range(min(4, k))])).cuda()
                sem_device(m.A, m.b, hist, 1e-10, x)
            st = gmres_device(m.A, m.b, x, k > 0, cfg.tol, cfg.restart, cfg.maxiter, m.pinv)
            d.append(st.iterations - int(its_ref[k]))
            assert st.converged and st.final_residual <= cfg.tol, k
            sol_err = max(sol_err, rel_max(x.cpu().numpy(), xs[k]))
            half[k] = x[dofs]      # all-Neumann: the probe displacements are unknowns
    assert max(abs(v) for v in d) <= 1, d
    assert sol_err <= 1e-6, sol_err
    # histories: ours and the reference run's (its per-k probe values), both
    # through the same windowed IDFT (pinned separately against the golden)
    series, _ = windowed_inverse_device(half, cfg.window, ds.eta, cfg.period)
    ref_half = torch.from_numpy(np.ascontiguousarray(xs[:, [p.dof for p in cfg.probes]])).cuda()
    ref_series, _ = windowed_inverse_device(ref_half, cfg.window, ds.eta, cfg.period)
    series, ref_series = series.cpu().numpy(), ref_series.cpu().numpy()
    for c, p in enumerate(cfg.probes):
        href = ref_series[:, c]
        assert np.linalg.norm(series[:, c] - href) / np.linalg.norm(href) <= 1e-6, p.name
        # the reference's rerun (this golden) reproduces its first run's history
        assert (np.linalg.norm(href - gs[f"cfg2_h_{p.name}"]) /
                np.linalg.norm(gs[f"cfg2_h_{p.name}"])) <= 1e-7, p.name


def test_cfg2_full_sweep_matches_reference_run(cuda):
    """BASELINE cfg2 (the headline) end to end: all 129 SEM-chained solves of
    run_sweep against the live reference's own 129-frequency run
    (tests/golden/make_golden.py cfg2_sweep, driver.py:92-176).

    Per-frequency parity (identical inputs) is the stepwise test.  A chained
    sweep feeds each tol-1e-8 solution forward, so a 1e-15 difference in the
    assembled matrices moves later iteration counts and tol-level solution
    digits.  Measured (tools/diag_cfg2_chain.py, profiles/r02/
    cfg2_chain_gpu_vs_reference_solver.json): the reference's OWN solver
    chained over our systems differs from the reference's run by up to 3
    iterations (92 % of k within 1) and by 1.39e-6 in the e0_uz history
    (others <= 7e-8) — the same as our sweep (<= 5, 92 %, 1.38e-6), while our
    sweep and that chain agree to 1.2e-7 in every history.  The reference is
    no steadier against itself: its two golden runs (cfg2_sweep and
    cfg2_solutions, same machine, OPENBLAS_NUM_THREADS 4 vs 6) differ by up to
    4 iterations with 91.5 % of k within 1.  Any change of rounding moves
    this statistic (two of our solver builds that differ only in the row
    blocking of the dot products: 92 % and 90 % within 1, max 5 and 3).
    The e0_uz history is the one above 1e-6: the all-Neumann cavity operator
    (interior identity) has rigid-body near-null directions
    whose tiny eigenvalues are set by the assembly's rounding, and e0_uz is
    a small component (element 0's normal has n_z = -0.034: max |e0_uz| =
    0.11 against 3.1 for e0_uy), so a rigid z-drift far below the radial
    response shows up there relative to it; the reference's two runs (identical
    matrices) agree there to 2e-8, any other assembly (ours, at 2.3e-15 of
    max|A|) lands at ~1.4e-6.
    Bars here: every history within 2e-6 (three of four within 1e-6), counts
    within 5 and 85 % within 1, total within 1 %, no failed frequency,
    literal final residuals <= tol."""
    from conftest import GOLDEN
    from paper_1212_3032_b200 import run_sweep
    from paper_1212_3032_b200.workloads import cfg2

    if not (GOLDEN / "cfg2_sweep.npz").exists():
        pytest.skip("cfg2_sweep.npz not generated")
    g = golden("cfg2_sweep")
    res = run_sweep(cfg2())
    its = np.array([s.iterations for s in res.stats])
    d = np.abs(its - g["cfg2_its"])
    assert d.max() <= 5 and (d <= 1).mean() >= 0.85, d.tolist()
    assert abs(its.sum() - g["cfg2_its"].sum()) <= 0.01 * g["cfg2_its"].sum()
    errs = {}
    for name in g["cfg2_probes"]:
        h, href = res.histories[str(name)], g[f"cfg2_h_{name}"]
        errs[str(name)] = np.linalg.norm(h - href) / np.linalg.norm(href)
    assert max(errs.values()) <= 2e-6 and sorted(errs.values())[-2] <= 1e-6, errs
    assert not res.failed_frequencies and len(g["failed"]) == 0
    assert all(s.converged and s.final_residual <= 1e-8 for s in res.stats)


def test_sem_ax0_and_gmres_start_from_it(cuda):
    """SEM's A x0 (= Y s, ABI v2) equals A @ x0, and GMRES started from it
    takes the same iterations to the same solution as with b - A x0."""
    import torch

    from paper_1212_3032_b200 import block_diag_precond
    from paper_1212_3032_b200.linsolve import gmres_device, sem_device

    g = golden("linsolve")
    a = torch.from_numpy(g["rod_A"]).cuda()
    b = torch.from_numpy(g["rod_b"]).cuda()
    n = b.shape[0]
    rng = np.random.default_rng(5)
    xs = np.linalg.solve(g["rod_A"], g["rod_b"])
    cols = np.stack([xs + 1e-3 * (rng.normal(size=n) + 1j * rng.normal(size=n))
                     for _ in range(3)])
    X = torch.from_numpy(cols).cuda()
    x0 = torch.empty_like(b)
    ax0 = torch.empty_like(b)
    sem_device(a, b, X, 1e-10, x0, ax0_out=ax0)
    assert rel_max(ax0.cpu().numpy(), (a @ x0).cpu().numpy()) <= 1e-12
    pinv = block_diag_precond(a).pinv
    xa, xb = x0.clone(), x0.clone()
    sa = gmres_device(a, b, xa, True, 1e-9, 60, 1000, pinv, ax0=ax0)
    sb = gmres_device(a, b, xb, True, 1e-9, 60, 1000, pinv)
    assert sa.converged and sb.converged
    assert abs(sa.iterations - sb.iterations) <= 1
    if sa.iterations == sb.iterations:
        assert sb.matvecs - sa.matvecs == 1      # the skipped b - A x0 pass
    assert rel_max(xa.cpu().numpy(), xb.cpu().numpy()) <= 1e-7
    assert abs(sa.init_residual - sb.init_residual) <= 1e-12 * sb.init_residual


def test_solver_cta_budget_same_result(cuda):
    """ewb_set_solver_ctas: fewer CTAs, same algorithm (fixed-order sums over a
    different partition: results agree to rounding)."""
    import torch

    from paper_1212_3032_b200 import _lib, block_diag_precond
    from paper_1212_3032_b200.linsolve import gmres_device

    lib = _lib.load()
    g = golden("linsolve")
    a = torch.from_numpy(g["rod_A"]).cuda()
    b = torch.from_numpy(g["rod_b"]).cuda()
    pinv = block_diag_precond(a).pinv
    full = int(lib.ewb_solver_ctas())
    x1 = torch.zeros_like(b)
    s1 = gmres_device(a, b, x1, False, 1e-8, 30, 1000, pinv)
    try:
        _lib.check(lib.ewb_set_solver_ctas(37))
        assert lib.ewb_solver_ctas() == min(37, full)
        x2 = torch.zeros_like(b)
        s2 = gmres_device(a, b, x2, False, 1e-8, 30, 1000, pinv)
    finally:
        _lib.check(lib.ewb_set_solver_ctas(0))
    assert lib.ewb_solver_ctas() == full
    assert abs(s1.iterations - s2.iterations) <= 1
    assert rel_max(x1.cpu().numpy(), x2.cpu().numpy()) <= 1e-6
    with pytest.raises(ValueError):
        _lib.check(lib.ewb_set_solver_ctas(-1))


def test_cfg1_stepwise_iterations_with_batched_assembly(cuda):
    """As the stepwise test, with every system from the 16-member
    multi-frequency assembly the sweep uses (phase recurrence)."""
    import torch

    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.linsolve import gmres_device, sem_device
    from paper_1212_3032_b200.transform import eta_from_kappa, forward_mft, frequency_grid
    from paper_1212_3032_b200.workloads import cfg1

    g = golden("cfg1_solutions")
    cfg = cfg1()
    asm = Assembler(cfg.mesh, cfg.material)
    eta = eta_from_kappa(cfg.kappa, cfg.period)
    om = frequency_grid(cfg.period, cfg.n_omega, eta)
    spectra = np.stack([forward_mft(s, cfg.period, cfg.n_omega, eta).values for s in cfg.signals])
    sig = cfg.bcs.flat_signal()
    xref = g["x"]
    x = torch.zeros(cfg.mesh.n_dofs, dtype=torch.complex128, device="cuda")
    diffs = []
    batch = None
    for k0 in range(0, len(om), 16):
        ks = list(range(k0, min(len(om), k0 + 16)))
        P = np.stack([spectra[sig, k] for k in ks])
        batch = asm.assemble_system_multi([om[k] for k in ks], cfg.bcs, P, out=batch)
        for f, k in enumerate(ks):
            sysm = batch.member(f)
            if k:
                hist = torch.from_numpy(xref[max(0, k - 2):k][::-1].copy()).cuda()
                sem_device(sysm.A, sysm.b, hist, 1e-10, x)
            st = gmres_device(sysm.A, sysm.b, x, k > 0, cfg.tol, cfg.restart, cfg.maxiter,
                              sysm.pinv)
            diffs.append(st.iterations - int(g["its"][k]))
            assert rel_max(x.cpu().numpy(), xref[k]) <= 1e-6
    assert max(abs(d) for d in diffs) <= 1, diffs


def test_device_sweep_strided_frequencies_sem_off(cuda):
    """A rank's round-robin share (k = 1, 3, 5, ...: batches equispaced with
    step 2 dw) solved through the batched path equals per-frequency solves."""
    import dataclasses

    import torch

    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.linsolve import gmres_device
    from paper_1212_3032_b200.workloads import cfg1

    cfg = dataclasses.replace(cfg1(), sem_enabled=False)
    ks = list(range(1, 40, 2))
    ds = DeviceSweep(cfg, frequencies=ks)
    stats = ds.run()
    ref = DeviceSweep(cfg, assembler=ds.asm, frequencies=ks, assembly_batch=1)
    ref_stats = ref.run()
    for k in ks:
        assert abs(stats[k].iterations - ref_stats[k].iterations) <= 1
        assert rel_max(ds.sol[k].cpu().numpy(), ref.sol[k].cpu().numpy()) <= 1e-8
    x = torch.zeros_like(ds.sol[ks[3]])
    sysm = ds.asm.assemble_system(ds.omegas[ks[3]], cfg.bcs, ds.P[ks[3]])
    gmres_device(sysm.A, sysm.b, x, False, cfg.tol, cfg.restart, cfg.maxiter, sysm.pinv)
    assert rel_max(ds.sol[ks[3]].cpu().numpy(), x.cpu().numpy()) <= 1e-8


def test_concurrent_solves_equal_sequential(cuda):
    """gmres_device_concurrent: independent systems side by side on separate
    streams with 1/m of the SMs each == one after another (to rounding)."""
    import torch

    from paper_1212_3032_b200.linsolve import gmres_device, gmres_device_concurrent

    gen = torch.Generator(device="cuda")
    gen.manual_seed(9)
    n, m = 3000, 4
    As = [torch.randn((n, n), dtype=torch.complex128, device="cuda", generator=gen)
          for _ in range(m)]
    for a in As:
        a.diagonal().add_(2.5 * n ** 0.5)
    bs = [torch.randn(n, dtype=torch.complex128, device="cuda", generator=gen) for _ in range(m)]
    seq = []
    for a, b in zip(As, bs):
        x = torch.zeros_like(b)
        st = gmres_device(a, b, x, False, 1e-10, 30, 300, None)
        seq.append((x.cpu().numpy(), st.iterations))
    xs = [torch.zeros_like(b) for b in bs]
    stats = gmres_device_concurrent(As, bs, xs, 1e-10, 30, 300)
    for (xr, ir), x, st in zip(seq, xs, stats):
        assert abs(st.iterations - ir) <= 1 and st.converged
        assert rel_max(x.cpu().numpy(), xr) <= 1e-8


@pytest.mark.parametrize("nb", [1, 5, 32])
def test_cfg1_sweep_any_assembly_batch(cuda, nb):
    """The sweep with 1, 5 or 32 frequencies per assembly pass: iterations +-1
    on every k against the reference's solver chained over the same systems,
    histories 1e-6 against the reference's run (as the default-batch test)."""
    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.transform import windowed_inverse_device
    from paper_1212_3032_b200.workloads import cfg1

    g = golden("cfg1_sweep")
    cfg = cfg1()
    ds = DeviceSweep(cfg, assembly_batch=nb)
    assert ds.batch_size() == nb
    st = ds.run()
    its = np.array([st[k].iterations for k in sorted(st)])
    ref_same = _reference_solver_chain(ds, cfg)
    assert np.abs(its - ref_same).max() <= 1, (its - ref_same).tolist()
    d = np.abs(its - g["cfg1_its"])
    assert d.max() <= 2 and (d <= 1).mean() >= 0.95, d
    series, _ = windowed_inverse_device(ds.probe_half(cfg.probes), cfg.window, ds.eta, cfg.period)
    series = series.cpu().numpy()
    for c, p in enumerate(cfg.probes):
        href = g[f"cfg1_h_{p.name}"]
        assert np.linalg.norm(series[:, c] - href) / np.linalg.norm(href) <= 1e-6


# ----------------------------------------------------------------------
# exit semantics: every exit is decided on the literal b - A x
# (linsolve.py:200-205); restarts use the stored products
# ----------------------------------------------------------------------
def _literal(a, b, x):
    import torch

    return (torch.linalg.vector_norm(b - a @ x) / torch.linalg.vector_norm(b)).item()


def test_final_residual_is_literal_multicycle(cuda):
    """Several restart cycles (restart 7, tol 1e-11), block preconditioner:
    final_residual equals ||b - A x|| / ||b|| and meets tol."""
    torch = cuda
    from paper_1212_3032_b200 import block_diag_precond
    from paper_1212_3032_b200.linsolve import gmres_device

    gen = torch.Generator(device="cuda")
    gen.manual_seed(11)
    n = 1200
    a = torch.randn((n, n), dtype=torch.complex128, device="cuda", generator=gen)
    a.diagonal().add_(2.2 * n ** 0.5)
    b = torch.randn(n, dtype=torch.complex128, device="cuda", generator=gen)
    pinv = block_diag_precond(a).pinv
    x = torch.zeros_like(b)
    st = gmres_device(a, b, x, False, 1e-11, 7, 500, pinv)
    assert st.converged and st.iterations > 14             # >= 3 cycles
    lit = _literal(a, b, x)
    assert lit <= 1e-11 and abs(st.final_residual - lit) <= 1e-14
    # one literal pass per exit: iterations + the exit's b - A x
    assert st.matvecs == st.iterations + 1
    # restart from the solution with its A x supplied (SEM's Y s): a
    # 0-iteration exit is still confirmed by one literal pass
    x2 = x.clone()
    ax = a @ x2
    st2 = gmres_device(a, b, x2, True, 1e-10, 7, 500, pinv, ax0=ax)
    assert st2.iterations == 0 and st2.matvecs == 1 and st2.converged
    assert abs(st2.final_residual - _literal(a, b, x2)) <= 1e-14
    # maxiter exit is literal too
    x3 = torch.zeros_like(b)
    st3 = gmres_device(a, b, x3, False, 1e-14, 5, 12, pinv)
    assert not st3.converged and st3.iterations == 12
    assert abs(st3.final_residual - _literal(a, b, x3)) <= 1e-14


def test_cfg1_sweep_final_residuals_are_literal(cuda):
    """Every cfg1 solve of the device sweep: reported final residual =
    ||b - A x|| / ||b|| <= tol, recomputed on the re-assembled system."""
    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.workloads import cfg1

    cfg = cfg1()
    ds = DeviceSweep(cfg)
    stats = ds.run()
    sysm = None
    for k in sorted(stats):
        sysm = ds.asm.assemble_system(ds.omegas[k], cfg.bcs, ds.P[k], out=sysm)
        lit = _literal(sysm.A, sysm.b, ds.sol[k])
        assert stats[k].converged and lit <= cfg.tol, (k, lit)
        assert abs(stats[k].final_residual - lit) <= 1e-12 * max(1.0, lit / cfg.tol), k


def test_operator_gmres_multicycle_matches_dense(cuda):
    """Device operator GMRES (matrix-free, restart 5 -> several cycles) vs the
    dense kernel on the same system; a plain torch callable takes the same
    device kernels with a host-checked gate."""
    torch = cuda
    from paper_1212_3032_b200 import (Assembler, BoundaryConditionSet, MatrixFreeOperator,
                                      block_diag_precond, gmres)
    from paper_1212_3032_b200.workloads import cavity_mesh

    mesh = cavity_mesh(2)
    asm = Assembler(mesh, _unit())
    bcs = BoundaryConditionSet.traction_free(mesh.n_elements)
    load = (-1.0 * mesh.normals).ravel().astype(complex)
    om = 3.0 - 0.37j
    dense = asm.assemble_system(om, bcs, load)
    op = MatrixFreeOperator(asm, om, bcs)
    pc = op.block_preconditioner()
    x_d, st_d = gmres(dense.A, dense.b, tol=1e-10, restart=5, precond=block_diag_precond(dense.A))
    x_m, st_m = gmres(op, dense.b, tol=1e-10, restart=5, precond=pc)
    assert st_d.iterations > 10
    assert abs(st_m.iterations - st_d.iterations) <= 1 and st_m.converged
    assert rel_max(x_m.cpu().numpy(), x_d.cpu().numpy()) <= 1e-8
    assert abs(st_m.final_residual - _literal(dense.A, dense.b, x_m)) <= 1e-13
    A = dense.A
    x_c, st_c = gmres(lambda v: A @ v, dense.b, tol=1e-10, restart=5, precond=pc)
    assert abs(st_c.iterations - st_d.iterations) <= 1
    assert rel_max(x_c.cpu().numpy(), x_d.cpu().numpy()) <= 1e-8
    # warm start without A x0: the initial residual takes one application
    x_w, st_w = gmres(op, dense.b, x0=x_d, tol=1e-9, restart=5, precond=pc)
    assert st_w.iterations == 0 and st_w.matvecs == 1


def _unit():
    from paper_1212_3032_b200 import Material

    return Material.from_young_poisson(1.0, 0.25, 1.0)


@pytest.mark.parametrize("K,n", [(3, 1111), (4, 1111), (4, 513), (3, 40), (4, 2304)])
def test_sem_ring_staged_x_ragged_sizes(cuda, K, n):
    """SEM's Y = A X for K = 3, 4 stages the x chunks in the TMA ring next to 8
    rows of A (matvec_rows_wide<K, XS>): sizes with a ragged last column tile,
    a one-column second tile, fewer columns than one tile and the cfg1 size,
    against the oracle's least squares (linsolve.py:213-242) and, through the
    returned A x0, against numpy's product."""
    torch = cuda
    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200.linsolve import sem_device

    rng = np.random.default_rng(100 * K + n)
    A = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)) + 3 * np.sqrt(n) * np.eye(n)
    base = rng.normal(size=n) + 1j * rng.normal(size=n)
    X = np.stack([base * (1 + 0.1 * i) + 1e-2 * (rng.normal(size=n) + 1j * rng.normal(size=n))
                  for i in range(K)])
    b = A @ (base * 1.07) + 1e-3 * rng.normal(size=n)
    oh = O.History(K)
    for i in range(K - 1, -1, -1):
        oh.push(X[i])
    ref = O.sem_guess(oh, A, b)
    Ad = torch.from_numpy(A).cuda()
    x0 = torch.empty(n, dtype=torch.complex128, device="cuda")
    ax0 = torch.empty_like(x0)
    sem_device(Ad, torch.from_numpy(b).cuda(), torch.from_numpy(X).cuda(), 1e-10, x0, ax0_out=ax0)
    got = x0.cpu().numpy()
    assert rel_max(got, ref) <= 1e-9
    assert rel_max(ax0.cpu().numpy(), A @ got) <= 1e-12


@pytest.mark.parametrize("K", [5, 6, 8])
def test_sem_deep_history_vs_oracle(cuda, K):
    """SEM with K > 4 history columns (Y = A X in passes of 4; linsolve.py:213-242)
    for a dense matrix and for the matrix-free operator vs the oracle."""
    torch = cuda
    from oracle import ewbem_oracle as O
    from paper_1212_3032_b200 import (Assembler, MatrixFreeOperator, SolutionHistory,
                                      sem_initial_guess)
    from paper_1212_3032_b200.workloads import cavity_mesh

    mesh = cavity_mesh(1)
    asm = Assembler(mesh, _unit())
    om = 2.0 - 0.4j
    op = MatrixFreeOperator(asm, om)
    n = mesh.n_dofs
    A = op.apply_multi(torch.eye(n, dtype=torch.complex128, device="cuda")).T.contiguous()
    rng = np.random.default_rng(K)
    base = rng.normal(size=n) + 1j * rng.normal(size=n)
    hist, ohist = SolutionHistory(K), O.History(K)
    for i in range(K):
        c = base * (1 + 0.1 * i) + 1e-2 * (rng.normal(size=n) + 1j * rng.normal(size=n))
        hist.push(c)
        ohist.push(c)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    ref = O.sem_guess(ohist, A.cpu().numpy(), b)
    got_d = sem_initial_guess(hist, A, b).cpu().numpy()
    got_m = sem_initial_guess(hist, op, b).cpu().numpy()
    assert rel_max(got_d, ref) <= 1e-8
    assert rel_max(got_m, ref) <= 1e-8


def test_solver_rows_per_cta_capacity_rejected(cuda):
    """ewb_gmres refuses (ValueError, no launch) a CTA budget whose rows per
    CTA overflow the update phase's shared-memory scratch, instead of
    overrunning it; the same size with enough CTAs solves."""
    torch = cuda
    from paper_1212_3032_b200 import _lib
    from paper_1212_3032_b200.linsolve import gmres_device

    lib = _lib.load()
    cap = 12288                               # complex values the ring holds
    n_bad = 2 * (cap // 2 - 2) + 16           # 2 CTAs: rows per CTA + 2 > cap / 2
    a = torch.zeros((n_bad, n_bad), dtype=torch.complex128, device="cuda")
    a.diagonal().fill_(2.0)
    b = torch.ones(n_bad, dtype=torch.complex128, device="cuda")
    x = torch.zeros_like(b)
    try:
        _lib.check(lib.ewb_set_solver_ctas(2))
        with pytest.raises(ValueError, match="rows per solver CTA"):
            gmres_device(a, b, x, False, 1e-8, 10, 100, None)
    finally:
        _lib.check(lib.ewb_set_solver_ctas(0))
    st = gmres_device(a, b, x, False, 1e-8, 10, 100, None)
    assert st.converged and rel_max(x.cpu().numpy(), 0.5 * np.ones(n_bad)) <= 1e-14


def test_sem_depth_beyond_device_cap_rejected_up_front(cuda):
    """A reference config may ask for any SEM depth; the device SEM keeps up to
    8 columns and refuses a deeper one before any assembly or solve."""
    from dataclasses import replace

    from paper_1212_3032_b200.driver import MAX_SEM_DEPTH, DeviceSweep
    from paper_1212_3032_b200.workloads import cfg1

    cfg = replace(cfg1(n_omega=8, divisions=(2, 2, 2)), sem_depth=MAX_SEM_DEPTH + 1)
    with pytest.raises(ValueError, match="sem_depth"):
        DeviceSweep(cfg)
