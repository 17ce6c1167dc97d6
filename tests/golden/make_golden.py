"""Generate the golden fixtures from the LIVE reference (build container only).

Run from the repo root:
    python tests/golden/make_golden.py [section ...]
Sections: small, cfg1_rows, linsolve, transform, tiers, sweeps, cfg1_sweep,
cfg2_head.  No section list = all of them (cfg1_sweep takes ~5 min, cfg2_head
~7 min on the 8-core build container).

The reference package is imported from /root/reference/pkg/src — it does
not exist on the GPU box, which is why its outputs are frozen here as .npz
files (small, compressed).  Only the reference's public library API is
called (SURVEY.md Appendix A shows how each BASELINE config is expressed);
nothing of the reference is copied into the repo.
"""

from __future__ import annotations

import hashlib
import math
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import ewbem  # noqa: E402
from ewbem import assembly as R_asm  # noqa: E402
from ewbem import kernels as R_ker  # noqa: E402
from ewbem import linsolve as R_lin  # noqa: E402
from ewbem import mesh as R_mesh  # noqa: E402
from ewbem import quadrature as R_quad  # noqa: E402
from ewbem import transform as R_tr  # noqa: E402
from ewbem.config import Probe, SweepConfig  # noqa: E402

OUT = Path(__file__).resolve().parent
UNIT = ewbem.Material.from_young_poisson(1.0, 0.25, 1.0)
STEEL0 = ewbem.Material.from_young_poisson(2.11e11, 0.0, 7850.0)


def save(name, **arrays):
    path = OUT / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"wrote {path.name}: {path.stat().st_size / 1024:.0f} KiB", flush=True)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg1_omegas():
    c_s = UNIT.c_s
    period = 8.0 / c_s
    eta = R_tr.eta_from_kappa(6.0 / math.log(10.0), period)
    return R_tr.frequency_grid(period, 128, eta), period, eta


# ----------------------------------------------------------------------
def section_small():
    """Full T/U of small meshes at several frequencies + rule tables."""
    out = {}
    cube = R_mesh.generate_box_mesh((1, 1, 1), (2, 2, 2))
    asm = R_asm.Assembler(cube, UNIT)
    omegas = np.array([0.0, -0.47j, 2.0 - 0.47j, 10.0 - 0.47j, -3.0 - 0.2j])
    out["cube_vertices"] = cube.vertices
    out["cube_triangles"] = cube.triangles
    out["cube_omegas"] = omegas
    out["cube_rowsums"] = asm.static_offdiag_rowsums()
    for i, om in enumerate(omegas):
        t, u = asm.assemble_tu(complex(om))
        out[f"cube_T{i}"] = t
        out[f"cube_U{i}"] = u
    # steel rod box (32 elements) at the GMRES test frequency
    rod = R_mesh.generate_box_mesh((1, 1, 2), (2, 2, 1))
    t, u = R_asm.Assembler(rod, STEEL0).assemble_tu(2000.0 - 300.0j)
    out["rod32_T"], out["rod32_U"] = t, u
    # flipped icosphere L1 (cavity orientation, interior identity trap)
    ico = R_mesh.generate_icosphere((0, 0, 0), 1.0, 1, flip=True)
    t, u = R_asm.Assembler(ico, UNIT).assemble_tu(1.5 - 0.3j)
    out["ico1_T"], out["ico1_U"] = t, u
    # rule tables
    out["gauss3_pts"], out["gauss3_w"] = R_quad.gauss3().points, R_quad.gauss3().weights
    out["gauss7_pts"], out["gauss7_w"] = R_quad.gauss7().points, R_quad.gauss7().weights
    for lvl in range(1, 5):
        rule = R_quad.subdivided(R_quad.gauss7(), lvl)
        out[f"sub{lvl}_pts"], out[f"sub{lvl}_w"] = rule.points, rule.weights
    verts = R_mesh.element_vertices(cube, 5)
    y, w = R_quad.self_rule_points(verts, 8, 16)
    out["self_verts"], out["self_y"], out["self_w"] = verts, y, w
    # radial scalars across the series/closed seam
    r = np.geomspace(1e-3, 5.0, 400)
    ks, kp = R_ker.wavenumbers(UNIT, 3.0 - 0.4j)
    out["radial_r"] = r
    out["radial_k"] = np.array([ks, kp])
    out["radial_f"] = np.stack(R_ker.phi_psi(r, ks, kp))
    out["static_f"] = np.stack(R_ker.static_phi_psi(r, UNIT))
    save("small", **out)


def section_cfg1_rows():
    """cfg1 cube: sampled T/U rows, all diagonal blocks, and full matvecs."""
    mesh = R_mesh.generate_box_mesh((1, 1, 1), (8, 8, 8))
    asm = R_asm.Assembler(mesh, UNIT)
    omegas, _, _ = cfg1_omegas()
    rng = np.random.default_rng(1234)
    n = mesh.n_dofs
    v = rng.normal(size=n) + 1j * rng.normal(size=n)
    elems = np.array([0, 191, 400, 767])
    rows = (3 * elems[:, None] + np.arange(3)).ravel()
    out = dict(elements=elems, v=v, ks=np.array([1, 64]),
               rowsums=asm.static_offdiag_rowsums())
    for k in (1, 64):
        t, u = asm.assemble_tu(omegas[k])
        out[f"T_rows_k{k}"] = t[rows]
        out[f"U_rows_k{k}"] = u[rows]
        tb = t.reshape(768, 3, 768, 3)
        ub = u.reshape(768, 3, 768, 3)
        ids = np.arange(768)
        out[f"T_diag_k{k}"] = tb[ids, :, ids, :]
        out[f"U_diag_k{k}"] = ub[ids, :, ids, :]
        out[f"Tv_k{k}"] = t @ v
        out[f"Uv_k{k}"] = u @ v
        out[f"Tmax_k{k}"] = np.abs(t).max()
        out[f"Umax_k{k}"] = np.abs(u).max()
    save("cfg1_rows", **out)


def section_tiers():
    """Tier tables / near levels (the last-bit trap)."""
    out = {}
    for name, mesh in (("cfg1", R_mesh.generate_box_mesh((1, 1, 1), (8, 8, 8))),
                       ("rod", R_mesh.generate_box_mesh((3, 1, 1), (12, 4, 4))),
                       ("ico3", R_mesh.generate_icosphere((0, 0, 0), 1.0, 3, flip=True))):
        asm = R_asm.Assembler(mesh, UNIT)
        dist = np.linalg.norm(mesh.centroids[:, None, :] - mesh.centroids[None, :, :], axis=-1)
        tier = asm.quad.classify(dist / mesh.diameters[None, :])
        out[f"{name}_tier"] = np.packbits(np.stack([tier & 1, tier >> 1]).astype(np.uint8))
        out[f"{name}_n"] = np.array(mesh.n_elements)
        near_i, near_j, near_l = [], [], []
        for j in range(mesh.n_elements):
            for rows, w, r, d, drdn in asm._columns[j]:
                q = r.shape[1]
                if q in (28, 112, 448, 1792):
                    lvl = {28: 1, 112: 2, 448: 3, 1792: 4}[q]
                    near_i += list(rows)
                    near_j += [j] * len(rows)
                    near_l += [lvl] * len(rows)
        out[f"{name}_near"] = np.array([near_i, near_j, near_l], dtype=np.int32)
        out[f"{name}_geom_sha"] = np.array([sha(mesh.vertices), sha(mesh.centroids),
                                            sha(mesh.normals), sha(mesh.areas),
                                            sha(mesh.diameters)])
    for lvl in (4, 6):
        m = R_mesh.generate_icosphere((0, 0, 0), 1.0, lvl, flip=True)
        out[f"ico{lvl}_geom_sha"] = np.array([sha(m.vertices), sha(m.centroids),
                                              sha(m.normals), sha(m.areas),
                                              sha(m.diameters)])
    save("tiers", **out)


def section_linsolve():
    out = {}
    rng = np.random.default_rng(2)
    n = 150
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)) + 6.0 * np.eye(n)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    x, st = R_lin.gmres(a, b, tol=1e-12, restart=20)
    out.update(rand_A=a, rand_b=b, rand_x=x, rand_its=st.iterations,
               rand_hist=np.array(st.residual_history))
    # rod32 BEM system with block preconditioner (test_linsolve.py:49-62)
    rod = R_mesh.generate_box_mesh((1, 1, 2), (2, 2, 1))
    t, u = R_asm.Assembler(rod, STEEL0).assemble_tu(2000.0 - 300.0j)
    bcs = R_asm.BoundaryConditionSet.traction_free(rod.n_elements)
    bcs.set_region(rod, 0, (0, 1, 2), R_asm.DIRICHLET, 0)
    bcs.set_region(rod, 1, (0,), R_asm.NEUMANN, 1)
    p = np.zeros(rod.n_dofs, dtype=complex)
    p[3 * np.flatnonzero(rod.region_tag == 1)] = -1e6
    sysm = R_asm.apply_bcs(t, u, bcs, p)
    x, st = R_lin.gmres(sysm.A, sysm.b, tol=1e-6, precond=R_lin.block_diag_precond(sysm.A))
    out.update(rod_A=sysm.A, rod_b=sysm.b, rod_kind=bcs.flat_kind(), rod_p=p,
               rod_x=x, rod_its=st.iterations, rod_hist=np.array(st.residual_history))
    # SEM guess with a rank-deficient history
    rng = np.random.default_rng(9)
    n = 90
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)) + 10.0 * np.eye(n)
    cols = [rng.normal(size=n) + 1j * rng.normal(size=n) for _ in range(4)]
    hist = R_lin.SolutionHistory(4)
    for c in cols:
        hist.push(c)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    out.update(sem_A=a, sem_X=hist.matrix(), sem_b=b,
               sem_x0=R_lin.sem_initial_guess(hist, a, b))
    hist2 = R_lin.SolutionHistory(3)
    base = cols[0]
    for c in (base, base, base * (1 + 1e-15)):
        hist2.push(c)
    out.update(sem2_X=hist2.matrix(), sem2_b=a @ base,
               sem2_x0=R_lin.sem_initial_guess(hist2, a, a @ base))
    # non-convergence: restart 5 maxiter 10
    rng = np.random.default_rng(3)
    n = 100
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    x, st = R_lin.gmres(a, b, tol=1e-14, restart=5, maxiter=10)
    out.update(nc_A=a, nc_b=b, nc_x=x, nc_its=st.iterations,
               nc_final=st.final_residual, nc_hist=np.array(st.residual_history))
    save("linsolve", **out)


def section_transform():
    out = {}
    period, n = 0.0155, 128
    eta = R_tr.eta_from_kappa(4.0, period)
    out.update(period=period, n=n, eta=eta)
    out["grid"] = R_tr.frequency_grid(period, n, eta)
    out["fwd_heaviside"] = R_tr.forward_mft(R_tr.TimeSignal.heaviside(-1e6), period, n, eta).values
    tab = R_tr.TimeSignal.tabulated([0.0, 0.004, 0.01, 0.0155], [0.0, 1.0, -0.5, 0.25])
    out["fwd_tab"] = R_tr.forward_mft(tab, period, n, eta).values
    rng = np.random.default_rng(11)
    half = rng.normal(size=n // 2 + 1) + 1j * rng.normal(size=n // 2 + 1)
    out["half"] = half
    spec = R_tr.conjugate_fill(half, period, eta)
    out["full"] = spec.values
    for w in ("rectangular", "hanning", "blackman"):
        out[f"inv_{w}"] = R_tr.inverse_mft(spec, w, eta)
        out[f"win_{w}"] = R_tr.window_weights(w, n)
    save("transform", **out)


def tiny_cfg(divisions=(1, 1, 1), n_omega=8, kappa=4.0, sem=True, tol=1e-5, window="hanning"):
    """The reference tests' rod fixture builder, restated (rod_fixtures.py:47-77)."""
    mesh = R_mesh.generate_box_mesh((3.0, 1.0, 1.0), divisions)

    def face_center(tag):
        m = np.flatnonzero(mesh.region_tag == tag)
        c = mesh.centroids[m].mean(axis=0)
        return int(m[np.argmin(np.linalg.norm(mesh.centroids[m] - c, axis=1))])

    zm = np.flatnonzero(mesh.region_tag == 4)
    mid = int(zm[np.argmin(np.linalg.norm(mesh.centroids[zm] - np.array([1.5, 0.5, 0.0]), axis=1))])
    bcs = R_asm.BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.set_region(mesh, 0, (0, 1, 2), R_asm.DIRICHLET, 0)
    bcs.set_region(mesh, 1, (0,), R_asm.NEUMANN, 1)
    return SweepConfig(
        mesh=mesh, material=STEEL0, bcs=bcs,
        signals=[R_tr.TimeSignal.zero(), R_tr.TimeSignal.heaviside(-1e6)],
        signal_names=["zero", "load"],
        probes=[Probe("tip_ux", face_center(1), 0, "displacement"),
                Probe("mid_ux", mid, 0, "displacement"),
                Probe("root_tx", face_center(0), 0, "traction")],
        period=0.0155, n_omega=n_omega, kappa=kappa, window=window,
        sem_enabled=sem, sem_depth=4, tol=tol, figures=False)


def _dump_sweep(prefix, res, out):
    out[f"{prefix}_its"] = np.array([s.iterations for s in res.stats])
    out[f"{prefix}_init"] = np.array([s.init_residual for s in res.stats])
    out[f"{prefix}_final"] = np.array([s.final_residual for s in res.stats])
    out[f"{prefix}_times"] = res.times
    names = sorted(res.histories)
    out[f"{prefix}_probes"] = np.array(names)
    for nm in names:
        out[f"{prefix}_h_{nm}"] = res.histories[nm]
        out[f"{prefix}_s_{nm}"] = res.half_spectra[nm]


def section_sweeps():
    out = {}
    from ewbem.driver import run_sweep
    _dump_sweep("tiny", run_sweep(tiny_cfg()), out)
    _dump_sweep("tiny_nosem", run_sweep(tiny_cfg(sem=False)), out)
    _dump_sweep("rod622", run_sweep(tiny_cfg(divisions=(6, 2, 2), n_omega=32)), out)
    save("sweeps", **out)


def cfg1_reference_config():
    mesh = R_mesh.generate_box_mesh((1, 1, 1), (8, 8, 8))
    _, period, _ = cfg1_omegas()
    bcs = R_asm.BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.set_region(mesh, 4, (0, 1, 2), R_asm.DIRICHLET, 0)   # z- all displacement zero
    bcs.set_region(mesh, 5, (2,), R_asm.NEUMANN, 1)          # z+ z traction load

    def face_center(tag):
        m = np.flatnonzero(mesh.region_tag == tag)
        c = mesh.centroids[m].mean(axis=0)
        return int(m[np.argmin(np.linalg.norm(mesh.centroids[m] - c, axis=1))])

    return SweepConfig(
        mesh=mesh, material=UNIT, bcs=bcs,
        signals=[R_tr.TimeSignal.zero(), R_tr.TimeSignal.heaviside(-1.0)],
        signal_names=["zero", "load"],
        probes=[Probe("top_uz", face_center(5), 2, "displacement"),
                Probe("bottom_tz", face_center(4), 2, "traction")],
        period=period, n_omega=128, kappa=6.0 / math.log(10.0), window="hanning",
        sem_enabled=True, sem_depth=2, tol=1e-8, restart=60, maxiter=1000, figures=False)


def section_cfg1_sweep():
    from ewbem.driver import run_sweep
    t0 = time.perf_counter()
    res = run_sweep(cfg1_reference_config())
    out = {"seconds": time.perf_counter() - t0}
    _dump_sweep("cfg1", res, out)
    save("cfg1_sweep", **out)


def section_cfg1_solutions():
    """cfg1 per-frequency solutions a_k, (b_k norm) and SEM initial residuals.

    The loop restates run_sweep's sequential branch (driver.py:123-153) with
    the reference's own functions so the per-k solution vectors can be kept:
    a GPU solve fed the reference's history must reproduce each count.
    """
    cfg = cfg1_reference_config()
    eta = R_tr.eta_from_kappa(cfg.kappa, cfg.period)
    omegas = R_tr.frequency_grid(cfg.period, cfg.n_omega, eta)
    spectra = np.stack([R_tr.forward_mft(s, cfg.period, cfg.n_omega, eta).values[:len(omegas)]
                        for s in cfg.signals])
    asm = R_asm.Assembler(cfg.mesh, cfg.material)
    asm.static_offdiag_rowsums()
    hist = R_lin.SolutionHistory(cfg.sem_depth)
    xs, its, init = [], [], []
    for k in range(len(omegas)):
        t, u = asm.assemble_tu(omegas[k])
        p = spectra[cfg.bcs.flat_signal(), k]
        sysm = R_asm.apply_bcs(t, u, cfg.bcs, p)
        x0 = R_lin.sem_initial_guess(hist, sysm.A, sysm.b) if len(hist) else None
        x, st = R_lin.gmres(sysm.A, sysm.b, x0=x0, tol=cfg.tol, restart=cfg.restart,
                            maxiter=cfg.maxiter, precond=R_lin.block_diag_precond(sysm.A))
        hist.push(x)
        xs.append(x)
        its.append(st.iterations)
        init.append(st.init_residual)
    save("cfg1_solutions", x=np.array(xs), its=np.array(its), init=np.array(init))


def section_cfg2_head():
    """cfg2 sphere (ico4 cavity, 15360 DOF): first 3 frequencies of the sweep.

    All-Neumann pressure load t = -p n_e with p = 1 (unit step), SEM K=4,
    tol 1e-8, restart 60; expressed through the library API.
    """
    mesh = R_mesh.generate_icosphere((0, 0, 0), 1.0, 4, flip=True)
    period = 16.0 / UNIT.c_s
    eta = R_tr.eta_from_kappa(6.0 / math.log(10.0), period)
    omegas = R_tr.frequency_grid(period, 256, eta)
    unit_spec = R_tr.forward_mft(R_tr.TimeSignal.heaviside(1.0), period, 256, eta).values
    load = (-1.0 * mesh.normals).ravel()
    bcs = R_asm.BoundaryConditionSet.traction_free(mesh.n_elements)
    t0 = time.perf_counter()
    asm = R_asm.Assembler(mesh, UNIT)
    asm.static_offdiag_rowsums()
    out = {"setup_seconds": time.perf_counter() - t0}
    rng = np.random.default_rng(77)
    v = rng.normal(size=mesh.n_dofs) + 1j * rng.normal(size=mesh.n_dofs)
    out["v"] = v
    hist = R_lin.SolutionHistory(4)
    its, init, final, secs, xs = [], [], [], [], []
    for k in range(3):
        t1 = time.perf_counter()
        t, u = asm.assemble_tu(omegas[k])
        if k == 1:
            out["Tv_k1"], out["Uv_k1"] = t @ v, u @ v
            out["T_row0_k1"], out["U_row0_k1"] = t[:3], u[:3]
            out["Tmax_k1"], out["Umax_k1"] = np.abs(t).max(), np.abs(u).max()
        p = load * unit_spec[k]
        sysm = R_asm.apply_bcs(t, u, bcs, p)
        del t, u
        x0 = R_lin.sem_initial_guess(hist, sysm.A, sysm.b) if len(hist) else None
        x, st = R_lin.gmres(sysm.A, sysm.b, x0=x0, tol=1e-8, restart=60, maxiter=1000,
                            precond=R_lin.block_diag_precond(sysm.A))
        hist.push(x)
        its.append(st.iterations)
        init.append(st.init_residual)
        final.append(st.final_residual)
        xs.append(x)
        secs.append(time.perf_counter() - t1)
        print(f"cfg2 k={k}: its={st.iterations} init={st.init_residual:.3e} "
              f"{secs[-1]:.1f}s", flush=True)
    out.update(its=np.array(its), init=np.array(init), final=np.array(final),
               seconds=np.array(secs), x=np.array(xs), omegas=omegas[:3], unit_spec=unit_spec)
    save("cfg2_head", **out)


def ref_sphere_pressure(level: int, n_omega: int, sem_depth: int = 4):
    """cfg2/cfg5 through the reference's own SweepConfig:
    flipped icosphere, all-Neumann, per-DOF step signals t = -p n_e, p = 1.
    Mirrors paper_1212_3032_b200/workloads.py:sphere_pressure field by field."""
    mesh = R_mesh.generate_icosphere((0, 0, 0), 1.0, level, flip=True)
    load = (-1.0 * mesh.normals).ravel()
    signals = [R_tr.TimeSignal.zero()] + [R_tr.TimeSignal.heaviside(a) for a in load]
    bcs = R_asm.BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.signal_index[:] = (1 + np.arange(mesh.n_dofs)).reshape(-1, 3).astype(np.int32)
    probes = [Probe("e0_ux", 0, 0, "displacement"), Probe("e0_uy", 0, 1, "displacement"),
              Probe("e0_uz", 0, 2, "displacement"),
              Probe("emid_ux", mesh.n_elements // 2, 0, "displacement")]
    return SweepConfig(
        mesh=mesh, material=UNIT, bcs=bcs, signals=signals,
        signal_names=["zero"] + [f"p{k}" for k in range(mesh.n_dofs)], probes=probes,
        period=16.0 / UNIT.c_s, n_omega=n_omega, kappa=6.0 / math.log(10.0),
        window="hanning", sem_enabled=True, sem_depth=sem_depth, tol=1e-8, restart=60,
        maxiter=1000, figures=False, allow_floating=True)


# per-k solution vectors kept for the "fed reference history" GPU tests
CFG2_KEEP = tuple(range(28, 33)) + tuple(range(60, 65)) + tuple(range(124, 129))
CFG2_KEEP_ALL = False   # cfg2_solutions: every k (the full stepwise test), 31 MB


def section_cfg2_sweep():
    """cfg2 full 129-frequency sweep through the LIVE reference run_sweep
    (driver.py:92-176), unmodified.  The module-level names run_sweep calls
    (Assembler.assemble_tu, apply_bcs, sem_initial_guess, gmres) are wrapped
    only to OBSERVE: per-k timings and a few solution vectors are recorded,
    every call is forwarded with its arguments untouched.  ~4 h on 8 cores."""
    from ewbem import driver as R_drv
    rec = {"asm_s": [], "bcs_s": [], "sem_s": [], "gmres_s": [], "x": {}, "x0": {}}
    orig_asm, orig_bcs = R_asm.Assembler.assemble_tu, R_drv.apply_bcs
    orig_sem, orig_gmres = R_drv.sem_initial_guess, R_drv.gmres

    def timed(key, fn):
        def wrap(*a, **kw):
            t0 = time.perf_counter()
            out = fn(*a, **kw)
            rec[key].append(time.perf_counter() - t0)
            return out
        return wrap

    def gmres_rec(*a, **kw):
        t0 = time.perf_counter()
        x, st = orig_gmres(*a, **kw)
        rec["gmres_s"].append(time.perf_counter() - t0)
        k = len(rec["gmres_s"]) - 1
        if CFG2_KEEP_ALL or k in CFG2_KEEP:
            rec["x"][k] = x.copy()
        print(f"cfg2 k={k}: its={st.iterations} init={st.init_residual:.3e} "
              f"final={st.final_residual:.3e} asm={rec['asm_s'][-1]:.1f}s", flush=True)
        return x, st

    R_asm.Assembler.assemble_tu = timed("asm_s", orig_asm)
    R_drv.apply_bcs = timed("bcs_s", orig_bcs)
    R_drv.sem_initial_guess = timed("sem_s", orig_sem)
    R_drv.gmres = gmres_rec
    try:
        t0 = time.perf_counter()
        res = R_drv.run_sweep(ref_sphere_pressure(4, 256))
        wall = time.perf_counter() - t0
    finally:
        R_asm.Assembler.assemble_tu = orig_asm
        R_drv.apply_bcs, R_drv.sem_initial_guess, R_drv.gmres = orig_bcs, orig_sem, orig_gmres
    out = {"seconds": wall, "asm_s": np.array(rec["asm_s"]), "bcs_s": np.array(rec["bcs_s"]),
           "sem_s": np.array(rec["sem_s"]), "gmres_s": np.array(rec["gmres_s"]),
           "keep_k": np.array(sorted(rec["x"])),
           "keep_x": np.array([rec["x"][k] for k in sorted(rec["x"])]),
           "failed": np.array(res.failed_frequencies, dtype=np.int64)}
    _dump_sweep("cfg2", res, out)
    out["cfg2_hist_len"] = np.array([len(s.residual_history) for s in res.stats])
    out["cfg2_hist_cat"] = np.concatenate([np.asarray(s.residual_history, float)
                                           for s in res.stats])
    if CFG2_KEEP_ALL:
        save("cfg2_solutions", k=out["keep_k"], x=out["keep_x"], its=out["cfg2_its"],
             init=out["cfg2_init"])
        return
    save("cfg2_sweep", **out)


def section_cfg2_solutions():
    """The same live-reference cfg2 run, keeping every per-k solution (the
    stepwise test feeds each frequency the reference's own history)."""
    global CFG2_KEEP_ALL
    CFG2_KEEP_ALL = True
    try:
        section_cfg2_sweep()
    finally:
        CFG2_KEEP_ALL = False


SECTIONS = dict(small=section_small, cfg1_rows=section_cfg1_rows, tiers=section_tiers,
                linsolve=section_linsolve, transform=section_transform,
                sweeps=section_sweeps, cfg1_sweep=section_cfg1_sweep,
                cfg1_solutions=section_cfg1_solutions,
                cfg2_head=section_cfg2_head, cfg2_sweep=section_cfg2_sweep,
                cfg2_solutions=section_cfg2_solutions)

if __name__ == "__main__":
    names = sys.argv[1:] or list(SECTIONS)
    for nm in names:
        t0 = time.perf_counter()
        SECTIONS[nm]()
        print(f"[{nm}] {time.perf_counter() - t0:.1f}s", flush=True)
