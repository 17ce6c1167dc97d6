"""GPU parity at the BASELINE sizes (cfg3, cfg4, cfg5) against fixtures of the
live reference (tests/golden/make_golden_scale.py).

cfg5 (ico6 cavity, 81,920 elements): 4,096 seeded rows of T and U applied to a
seeded vector and to the pressure load at the sweep's first 2 frequencies,
built column by column with the reference's own functions; the tier and
near-level census of those rows; and the sampled-row residual of the GPU
solution of the first 2 sweep frequencies.
cfg3: the 512 x 512 x 16 pair-kernel subsample.
cfg4: the batched GEMV on all 8 systems and GMRES iteration counts of the
reference's gmres (restart 50, tol 1e-8) at N = 4096 and 8192.
"""

import numpy as np
import pytest

from conftest import golden, rel_max

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ico6(cuda):
    from paper_1212_3032_b200 import Assembler
    from paper_1212_3032_b200.workloads import UNIT, load_mesh

    mesh = load_mesh("ico6")
    return mesh, Assembler(mesh, UNIT)


def test_cfg5_row_census_vs_reference(ico6):
    """Tier / near-level decisions of the 4,096 sampled rows over all 81,920
    columns equal the reference's classify / point_triangle_distance /
    near_level (assembly.py:132-161)."""
    mesh, asm = ico6
    g = golden("cfg5_rows")
    rows = g["rows"]
    pl = asm.pair_lists()
    mid_ref, near_ref = g["mid"], g["near"]
    n_e = mesh.n_elements
    for r_i, i in enumerate(rows):
        gm = set(mid_ref[mid_ref[:, 0] == i, 1].tolist())
        mm = set(pl["mid_j"][pl["mid_ptr"][i]:pl["mid_ptr"][i + 1]].tolist())
        assert gm == mm, f"row {i}: mid columns differ"
        sel = near_ref[:, 0] == i
        gn = set(zip(near_ref[sel, 1].tolist(), near_ref[sel, 2].tolist()))
        a, b = pl["near_ptr"][i], pl["near_ptr"][i + 1]
        nn = set(zip(pl["near_j"][a:b].tolist(), pl["near_lvl"][a:b].tolist()))
        assert gn == nn, f"row {i}: near (column, level) pairs differ"
        assert n_e - 1 - len(mm) - len(nn) == g["n_far"][r_i]


def _cfg5_vectors(mesh):
    rng = np.random.default_rng(int(golden("cfg5_rows")["vecs_seed"]))
    n = mesh.n_dofs
    v = rng.normal(size=n) + 1j * rng.normal(size=n)
    load = (-1.0 * mesh.normals).ravel().astype(complex)
    return np.stack([v, load])


def test_cfg5_sampled_rows_vs_reference(ico6, cuda):
    """(T V)[rows] and (U V)[rows] of the matrix-free kernels vs the reference's
    column-by-column assembly, first 2 sweep frequencies (<= 1e-10)."""
    torch = cuda
    from paper_1212_3032_b200 import MatrixFreeOperator

    mesh, asm = ico6
    g = golden("cfg5_rows")
    dof = (3 * g["rows"][:, None] + np.arange(3)).ravel()
    V = torch.from_numpy(_cfg5_vectors(mesh)).cuda()
    for f, om in enumerate(g["omegas"]):
        op = MatrixFreeOperator(asm, complex(om))          # all-Neumann: A = T
        tv = op.apply_multi(V).cpu().numpy()                # (2, N) = T V
        uv = np.stack([op.rhs_and_apply(V[c])[0].cpu().numpy() for c in range(2)])  # U V
        for c in range(2):
            assert rel_max(tv[c][dof], g["tv"][f][:, c]) <= 1e-10, (f, c)
            assert rel_max(uv[c][dof], g["uv"][f][:, c]) <= 1e-10, (f, c)


def test_cfg5_first_two_frequencies_sampled_residual(ico6, cuda):
    """The GPU matrix-free sweep's first 2 solutions satisfy the reference's
    equations on the sampled rows: b_R (reference) - (A x)_R within tol."""
    torch = cuda
    from paper_1212_3032_b200 import MatrixFreeOperator
    from paper_1212_3032_b200.driver import DeviceSweep
    from paper_1212_3032_b200.workloads import cfg5

    mesh, asm = ico6
    g = golden("cfg5_rows")
    cfg = cfg5(mesh=mesh)
    ds = DeviceSweep(cfg, assembler=asm, frequencies=[0, 1])
    ds.matrix_free = True
    stats = ds.run()
    dof = (3 * g["rows"][:, None] + np.arange(3)).ravel()
    for f, k in enumerate(g["ks"]):
        st = stats[int(k)]
        assert st.converged and st.final_residual <= cfg.tol
        x = ds.sol[int(k)]
        op = MatrixFreeOperator(asm, complex(g["omegas"][f]))
        ax = op(x).cpu().numpy()
        b_full = (g["unit_spec"][f] * op.rhs_and_apply(
            torch.from_numpy((-1.0 * mesh.normals).ravel().astype(complex)).cuda())[0]
        ).cpu().numpy()
        b_ref = g["unit_spec"][f] * g["uv"][f][:, 1]       # U p on the sampled rows
        assert rel_max(b_full[dof], b_ref) <= 1e-10
        r = b_ref - ax[dof]
        assert np.linalg.norm(r) <= 1.001 * cfg.tol * np.linalg.norm(b_full)


def test_cfg3_subsample_vs_reference(cuda):
    """ewb_pair_kernels_blocks / _reduce on the seeded 512 x 512 x 16 cfg3
    subsample vs reference pair_geometry + integrated_blocks (<= 1e-10)."""
    torch = cuda
    from paper_1212_3032_b200 import _lib
    from paper_1212_3032_b200.workloads import UNIT, cfg3_inputs

    g = golden("cfg3_sub")
    P, M = int(g["P"]), int(g["M"])
    x, tris, om, xv = cfg3_inputs()
    x, tris, xv = x[:P], tris[:M], xv[:M]
    assert np.array_equal(om, g["omegas"])
    F = len(om)
    lib = _lib.load()
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(tris.reshape(M, 9).copy()).cuda()
    omh = np.ascontiguousarray(np.stack([om.real, om.imag], axis=1))
    u = torch.empty((F, P, M, 3, 3), dtype=torch.complex128, device="cuda")
    t = torch.empty_like(u)
    _lib.check(lib.ewb_pair_kernels_blocks(_lib.ptr(xd), P, _lib.ptr(td), M, omh.ctypes.data, F,
                                           UNIT.lam, UNIT.mu, UNIT.rho, _lib.ptr(u), _lib.ptr(t),
                                           _lib.stream_handle()))
    s = g["samp"]
    us = u[s[:, 0], s[:, 1], s[:, 2]].cpu().numpy()
    ts = t[s[:, 0], s[:, 1], s[:, 2]].cpu().numpy()
    assert rel_max(us, g["u_samp"]) <= 1e-10
    assert rel_max(ts, g["t_samp"]) <= 1e-10
    for f in range(F):   # per-frequency max |K| over all 262,144 blocks
        assert abs(u[f].abs().max().item() - g["umax"][f]) <= 1e-10 * g["umax"][f]
        assert abs(t[f].abs().max().item() - g["tmax"][f]) <= 1e-10 * g["tmax"][f]
    xvd = torch.from_numpy(xv.copy()).cuda()
    yu = torch.einsum("fpmab,mb->fpa", u, xvd).cpu().numpy()
    assert rel_max(yu, g["yu"]) <= 1e-10
    del u, t
    yu = torch.empty((F, P, 3), dtype=torch.complex128, device="cuda")
    yt = torch.empty_like(yu)
    wsb = int(lib.ewb_pair_kernels_workspace_bytes(P, M, F))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.ewb_pair_kernels_reduce(_lib.ptr(xd), P, _lib.ptr(td), M, _lib.ptr(xvd),
                                           omh.ctypes.data, F, UNIT.lam, UNIT.mu, UNIT.rho,
                                           _lib.ptr(yu), _lib.ptr(yt), _lib.ptr(ws), wsb,
                                           _lib.stream_handle()))
    assert rel_max(yu.cpu().numpy(), g["yu"]) <= 1e-10
    assert rel_max(yt.cpu().numpy(), g["yt"]) <= 1e-10


_CFG4 = {}


def _cfg4_systems(n):
    """The 8 seeded cfg4-i systems of size n (host arrays, built once per run)."""
    from paper_1212_3032_b200.workloads import cfg4_random_system

    if n not in _CFG4:
        _CFG4[n] = [cfg4_random_system(n, seed) for seed in range(8)]
    return _CFG4[n]


CFG4_SIZES = [4096, 8192, 16384]   # BASELINE cfg4


@pytest.mark.parametrize("n", CFG4_SIZES)
def test_cfg4_gemv_batched_vs_numpy(cuda, n):
    """ewb_gemv_batched on the 8 seeded cfg4-i systems vs numpy (<= 1e-12)."""
    torch = cuda
    from paper_1212_3032_b200 import _lib

    lib = _lib.load()
    sys_ = _cfg4_systems(n)
    A = torch.from_numpy(np.stack([a for a, _ in sys_])).cuda()
    X = torch.from_numpy(np.stack([b for _, b in sys_])).cuda()
    Y = torch.empty_like(X)
    _lib.check(lib.ewb_gemv_batched(_lib.ptr(A), _lib.ptr(X), _lib.ptr(Y), n, 8,
                                    _lib.stream_handle()))
    Yh = Y.cpu().numpy()
    for i, (a, b) in enumerate(sys_):
        assert rel_max(Yh[i], a @ b) <= 1e-12


@pytest.mark.parametrize("n", CFG4_SIZES)
def test_cfg4_gmres_vs_reference(cuda, n):
    """GMRES (restart 50, tol 1e-8, no preconditioner) on the 8 seeded cfg4-i
    systems: iteration counts within +-1 of the reference's gmres, solutions
    1e-8, final residual = literal ||b - A x|| / ||b||."""
    torch = cuda
    from paper_1212_3032_b200 import gmres

    g = golden("cfg4_gmres")
    if f"n{n}_its" not in g:
        pytest.skip(f"no reference golden for n = {n}")
    its_ref, x_ref = g[f"n{n}_its"], g[f"n{n}_x"]
    for seed, (a, b) in enumerate(_cfg4_systems(n)):
        ad = torch.from_numpy(a).cuda()
        x, st = gmres(ad, b, tol=1e-8, restart=50, maxiter=1000)
        assert abs(st.iterations - int(its_ref[seed])) <= 1
        assert rel_max(x.cpu().numpy(), x_ref[seed]) <= 1e-8
        bd = torch.from_numpy(b).cuda()
        lit = (torch.linalg.vector_norm(bd - ad @ x) / torch.linalg.vector_norm(bd)).item()
        assert st.final_residual <= 1e-8 and abs(st.final_residual - lit) <= 1e-13
