"""The BASELINE.json configurations, built through this package's API.

cfg1  unit cube, 768 triangles / 2304 DOF, T = 8/c_s, N = 128 -> 65 solves,
      z- clamped, z+ unit step normal traction, SEM K = 2, tol 1e-8.
cfg2  flipped icosphere L4 (5120 / 15360 DOF), all-Neumann unit step
      pressure t = -p n_e, T = 16/c_s, N = 256 -> 129 solves, SEM K = 4.
cfg3  2^14 random points x 2^14 random triangles x 16 frequencies
      (pair-kernel microbenchmark; seeded).
cfg4  dense complex GMRES, N in {4096, 8192, 16384}, 8 systems, restart 50.
cfg5  flipped icosphere L6 (81920 / 245760 DOF), matrix-free, N = 64 -> 33.

eta = 6/T throughout (kappa = 6/ln 10).

Meshes are the reference's own (generate_box_mesh / generate_icosphere,
mesh.py:279-404), frozen in tests/golden/meshes.npz by
tests/golden/make_golden_scale.py: nothing here regenerates geometry.
"""

from __future__ import annotations

import math
from functools import lru_cache
from pathlib import Path

import numpy as np

from .assembly import DIRICHLET, NEUMANN, BoundaryConditionSet
from .material import Material
from .spec import Probe, SweepSpec
from .surface import SurfaceMesh
from .transform import TimeSignal

UNIT = Material.from_young_poisson(1.0, 0.25, 1.0)
KAPPA_6 = 6.0 / math.log(10.0)
MESH_FILE = Path(__file__).resolve().parents[1] / "tests" / "golden" / "meshes.npz"


@lru_cache(maxsize=None)
def _mesh_arrays():
    if not MESH_FILE.exists():
        raise FileNotFoundError(f"{MESH_FILE} (reference-generated meshes) is missing")
    return dict(np.load(MESH_FILE, allow_pickle=False))


def mesh_names():
    return sorted({k.split("__")[0] for k in _mesh_arrays()})


def load_mesh(name: str) -> SurfaceMesh:
    """A reference-generated mesh: ``box_<L>_<D>`` (e.g. box_1x1x1_8x8x8) or
    ``ico<level>`` (flipped unit icosphere, a cavity)."""
    a = _mesh_arrays()
    if f"{name}__vertices" not in a:
        raise KeyError(f"no mesh {name!r}; have {mesh_names()}")
    return SurfaceMesh(a[f"{name}__vertices"], a[f"{name}__triangles"],
                       a[f"{name}__region_tag"])


def box_mesh(lengths, divisions) -> SurfaceMesh:
    (lx, ly, lz), (nx, ny, nz) = lengths, divisions
    return load_mesh(f"box_{lx:g}x{ly:g}x{lz:g}_{nx}x{ny}x{nz}")


def cavity_mesh(level: int) -> SurfaceMesh:
    return load_mesh(f"ico{level}")


def face_center_element(mesh, tag: int) -> int:
    m = np.flatnonzero(mesh.region_tag == tag)
    c = mesh.centroids[m].mean(axis=0)
    return int(m[np.argmin(np.linalg.norm(mesh.centroids[m] - c, axis=1))])


def cfg1(n_omega: int = 128, divisions=(8, 8, 8)) -> SweepSpec:
    mesh = box_mesh((1, 1, 1), divisions)
    bcs = BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.set_region(mesh, 4, (0, 1, 2), DIRICHLET, 0)
    bcs.set_region(mesh, 5, (2,), NEUMANN, 1)
    return SweepSpec(
        mesh=mesh, material=UNIT, bcs=bcs,
        signals=[TimeSignal.zero(), TimeSignal.heaviside(-1.0)], signal_names=["zero", "load"],
        probes=[Probe("top_uz", face_center_element(mesh, 5), 2, "displacement"),
                Probe("bottom_tz", face_center_element(mesh, 4), 2, "traction")],
        period=8.0 / UNIT.c_s, n_omega=n_omega, kappa=KAPPA_6, window="hanning",
        sem_enabled=True, sem_depth=2, tol=1e-8, restart=60, maxiter=1000, figures=False)


def sphere_pressure(level: int, n_omega: int, sem_depth: int = 4, mesh=None) -> SweepSpec:
    """Pressurised flipped icosphere: per-DOF step signals t = -p n_e, p = 1."""
    mesh = cavity_mesh(level) if mesh is None else mesh
    load = (-1.0 * mesh.normals).ravel()
    signals = [TimeSignal.zero()] + [TimeSignal.heaviside(a) for a in load]
    bcs = BoundaryConditionSet.traction_free(mesh.n_elements)
    bcs.signal_index[:] = (1 + np.arange(mesh.n_dofs)).reshape(-1, 3).astype(np.int32)
    probes = [Probe("e0_ux", 0, 0, "displacement"), Probe("e0_uy", 0, 1, "displacement"),
              Probe("e0_uz", 0, 2, "displacement"),
              Probe("emid_ux", mesh.n_elements // 2, 0, "displacement")]
    return SweepSpec(
        mesh=mesh, material=UNIT, bcs=bcs, signals=signals,
        signal_names=["zero"] + [f"p{k}" for k in range(mesh.n_dofs)], probes=probes,
        period=16.0 / UNIT.c_s, n_omega=n_omega, kappa=KAPPA_6, window="hanning",
        sem_enabled=True, sem_depth=sem_depth, tol=1e-8, restart=60, maxiter=1000,
        figures=False, allow_floating=True)


def cfg2(n_omega: int = 256, mesh=None) -> SweepSpec:
    return sphere_pressure(4, n_omega, mesh=mesh)


def cfg5(n_omega: int = 64, mesh=None) -> SweepSpec:
    return sphere_pressure(6, n_omega, mesh=mesh)


def cfg3_inputs(n_points: int = 1 << 14, n_tris: int = 1 << 14, n_freq: int = 16,
                seed: int = 3032):
    """Seeded cfg3 inputs: points U[-1,1]^3, triangles (area >= 1e-4), omega_r - 2i."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1.0, 1.0, size=(n_points, 3))
    tris = []
    while len(tris) < n_tris:
        v = rng.uniform(-1.0, 1.0, size=(max(64, n_tris - len(tris)) * 2, 3, 3))
        a = 0.5 * np.linalg.norm(np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), axis=1)
        tris.extend(v[a >= 1e-4])
    tris = np.ascontiguousarray(np.array(tris[:n_tris]))
    omegas = rng.uniform(0.0, 50.0, size=n_freq) - 2.0j
    xv = rng.normal(size=(n_tris, 3)) + 1j * rng.normal(size=(n_tris, 3))
    return x, tris, omegas, xv


def cfg4_random_system(n: int, seed: int):
    """A = (G + iG')/sqrt2 + 3 sqrt(N) I, b ~ CN(0, 1)."""
    rng = np.random.default_rng(seed)
    a = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))) / math.sqrt(2.0)
    a[np.diag_indices(n)] += 3.0 * math.sqrt(n)
    b = (rng.normal(size=n) + 1j * rng.normal(size=n)) / math.sqrt(2.0)
    return a, b


def cfg4_assembled():
    """cfg4-ii: BEM operators of the nearest mesh sizes —
    ico3 cavity (3,840 DOF), box 16 x 16 x 12 (7,680 DOF), ico4 cavity
    (15,360 DOF) — at 8 consecutive sweep frequencies, SEM off."""
    out = []
    for name, cfg in (("ico3", sphere_pressure(3, 256)),
                      ("box16x16x12", cfg1(divisions=(16, 16, 12))),
                      ("ico4", sphere_pressure(4, 256))):
        cfg.sem_enabled = False
        out.append((name, cfg))
    return out
