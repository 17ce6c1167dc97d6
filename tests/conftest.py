import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def have_reference() -> bool:
    return (REFERENCE_SRC / "ewbem" / "__init__.py").exists()


@pytest.fixture(scope="session")
def reference():
    """The live reference package (build container only)."""
    if not have_reference():
        pytest.skip("reference not present (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import ewbem

    return ewbem


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1212_3032_b200 import _lib

    _lib.require_cuda()
    return torch


def rel_max(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def pytest_sessionfinish(session, exitstatus):
    """Debug-check build (EWB_LIBRARY=.../variants/debug.so):
    fail the session if any device-side invariant check fired."""
    if not os.environ.get("EWB_LIBRARY"):
        return
    try:
        import ctypes

        import torch

        if not torch.cuda.is_available():
            return
        from paper_1212_3032_b200 import _lib

        lib = _lib.load()
        fails, site = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.ewb_debug_checks(ctypes.byref(fails), ctypes.byref(site), 0))
    except Exception as exc:  # pragma: no cover - reporting only
        print(f"\n[ewb debug checks] could not read: {exc}")
        return
    print(f"\n[ewb debug checks] library={os.environ['EWB_LIBRARY']} "
          f"failures={fails.value} first_site={site.value}")
    if fails.value > 0:   # -1: a release build (no checks compiled in)
        session.exitstatus = 1
