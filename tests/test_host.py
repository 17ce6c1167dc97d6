"""Host-side code without a GPU: mesh fixtures and derived geometry, rule
tables, workloads, the C-ABI library exports, and the multi-rank frequency
sharding (gloo)."""

import hashlib
import os
import re
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name,key", [("cfg1", "box_1x1x1_8x8x8"), ("rod", "box_3x1x1_12x4x4"),
                                      ("ico3", "ico3"), ("ico4", "ico4"), ("ico6", "ico6")])
def test_mesh_geometry_bit_identical_to_reference(name, key):
    """SurfaceMesh's derived geometry of the reference-generated meshes equals
    the reference's own (hashes written by the live reference, mesh.py:88-106)."""
    from paper_1212_3032_b200.workloads import load_mesh

    m = load_mesh(key)
    ref = golden("tiers")[f"{name}_geom_sha"]
    got = [_sha(m.vertices), _sha(m.centroids), _sha(m.normals), _sha(m.areas),
           _sha(m.diameters)]
    assert got == list(ref)


def test_mesh_fixture_derived_geometry_bitwise():
    from paper_1212_3032_b200.workloads import load_mesh, mesh_names

    g = golden("meshes")
    for name in mesh_names():
        m = load_mesh(name)
        assert np.array_equal(m.areas, g[f"{name}__areas"]), name
        assert np.array_equal(m.diameters, g[f"{name}__diameters"]), name


def test_mesh_fixtures_equal_live_reference(reference):
    """tests/golden/meshes.npz is what the reference's generators produce."""
    from ewbem import mesh as R

    from paper_1212_3032_b200.workloads import load_mesh, mesh_names

    for name in mesh_names():
        if name.startswith("box_"):
            ls, ds = name[4:].split("_")
            ref = R.generate_box_mesh(tuple(float(v) for v in ls.split("x")),
                                              tuple(int(v) for v in ds.split("x")))
        else:
            ref = R.generate_icosphere((0, 0, 0), 1.0, int(name[3:]), flip=True)
        m = load_mesh(name)
        for f in ("vertices", "triangles", "region_tag", "centroids", "normals", "areas",
                  "diameters"):
            assert np.array_equal(getattr(m, f), getattr(ref, f)), (name, f)


def test_device_rule_tables_bitwise():
    from paper_1212_3032_b200.quadrature import device_rule_tables

    g = golden("small")
    flat, off, q = device_rule_tables()
    names = ["gauss3", "gauss7"] + [f"sub{L}" for L in range(1, 5)]
    for k, nm in enumerate(names):
        Q = q[k]
        b = flat[off[k]:off[k] + 3 * Q].reshape(Q, 3)
        w = flat[off[k] + 3 * Q:off[k] + 4 * Q]
        assert np.array_equal(b, g[f"{nm}_pts"]) and np.array_equal(w, g[f"{nm}_w"])


def test_workloads_config_values():
    from paper_1212_3032_b200.transform import eta_from_kappa
    from paper_1212_3032_b200.workloads import cfg1, cfg2, cfg3_inputs

    c = cfg1()
    assert c.mesh.n_elements == 768 and c.n_omega == 128
    assert eta_from_kappa(c.kappa, c.period) == 6.0 / c.period
    c2 = cfg2()
    assert c2.mesh.n_elements == 5120 and len(c2.signals) == 15361
    x, tris, om, xv = cfg3_inputs(64, 64, 4)
    area = 0.5 * np.linalg.norm(np.cross(tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 0]), axis=1)
    assert (area >= 1e-4).all() and x.shape == (64, 3) and np.all(om.imag == -2.0)


# ----------------------------------------------------------------------
# C ABI
# ----------------------------------------------------------------------
def _declared_symbols():
    text = (ROOT / "include" / "ewbem_b200.h").read_text()
    return sorted(set(re.findall(r"^(?:int|int32_t|int64_t|const char\*)\s+(ewb_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1212_3032_b200 import _lib
    from paper_1212_3032_b200.build import build

    build()
    lib = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 20
    assert sorted(_lib.EXPORTS) == declared
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.ewb_abi_version() == _lib.ABI_VERSION == 6
    out = subprocess.run(["nm", "-D", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf" T {name}$", out, re.M), name


def test_cubin_is_sm100a():
    from paper_1212_3032_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_compute_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1212_3032_b200 import Assembler, Material, NativeUnavailable
    from paper_1212_3032_b200.workloads import box_mesh

    with pytest.raises(NativeUnavailable):
        Assembler(box_mesh((1, 1, 1), (1, 1, 1)), Material.from_young_poisson(1, 0.25, 1))


def test_argument_validation_without_gpu():
    """Invalid arguments are rejected before any device work."""
    import ctypes

    from paper_1212_3032_b200 import _lib

    lib = _lib.load()
    assert lib.ewb_gmres(None, None, None, None, 0, None, 0, 1e-5, 60, 1000, None, 0, None, 0,
                         None, None) == _lib.EWB_ERR_INVALID
    assert b"bad argument" in lib.ewb_last_error()
    assert lib.ewb_blockdiag_inverse(ctypes.c_void_p(16), 4, ctypes.c_void_p(16),
                                     ctypes.c_void_p(16), None) == _lib.EWB_ERR_INVALID
    assert b"divisible by 3" in lib.ewb_last_error()
    # multi-frequency entry point
    v = ctypes.c_void_p(16)
    assert lib.ewb_assemble_system_multi(None, 4, v, v, v, v, v, v, v, v, None) == \
        _lib.EWB_ERR_INVALID
    assert b"null argument" in lib.ewb_last_error()
    assert lib.ewb_set_solver_ctas(-1) == _lib.EWB_ERR_INVALID


# ----------------------------------------------------------------------
# multi-rank sharding (gloo, world size 2, CPU)
# ----------------------------------------------------------------------
def test_shard_frequencies_partition():
    from paper_1212_3032_b200.driver import shard_frequencies

    for nf in (5, 33, 65, 129):
        for w in (1, 2, 3, 8):
            got = sorted(k for r in range(w) for k in shard_frequencies(nf, r, w))
            assert got == list(range(nf))


_GLOO_SCRIPT = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch.distributed as dist
from paper_1212_3032_b200.driver import gather_frequency_results, shard_frequencies
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
nf, width = 9, 3
local = {k: (np.arange(width) * (k + 1) + 1j * k, (k, 0.5 * k, 1e-9, 0.1, 1.0, 0.0))
         for k in shard_frequencies(nf, r, w)}
vals, meta = gather_frequency_results(local, nf, width, dist)
for k in range(nf):
    assert np.array_equal(vals[k], np.arange(width) * (k + 1) + 1j * k)
    assert meta[k][0] == k
print("ok", r)
dist.destroy_process_group()
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_two_rank_gather(tmp_path):
    script = tmp_path / "g.py"
    script.write_text(_GLOO_SCRIPT)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()),
               WORLD_SIZE="2")
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, str(script), str(ROOT)], env=e,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=120)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    assert all("ok" in o for o in outs)


def test_forward_transform_batch_equals_per_signal():
    """forward_mft_batch (linearity for steps, one FFT for tabulated signals)
    equals the per-signal transform (transform.py:206-211) to 1 ulp."""
    from paper_1212_3032_b200.transform import TimeSignal, forward_mft, forward_mft_batch

    period, n, eta = 12.5, 128, 0.37
    sigs = [TimeSignal.zero(), TimeSignal.heaviside(-1.0), TimeSignal.heaviside(0.3137),
            TimeSignal.tabulated([0.0, 2.0, 5.0, 12.0], [0.0, 1.0, -0.5, 0.25]),
            TimeSignal.heaviside(1e-7)]
    ref = np.stack([forward_mft(s, period, n, eta).values for s in sigs])
    got = forward_mft_batch(sigs, period, n, eta)
    assert np.abs(got - ref).max() <= 4e-16 * np.abs(ref).max()
    np.testing.assert_array_equal(got[3], ref[3])          # tabulated: same FFT
    assert not got[0].any()
    part = forward_mft_batch(sigs, period, n, eta, n_keep=n // 2 + 1)
    np.testing.assert_array_equal(part, got[:, : n // 2 + 1])
