"""Per-iteration GMRES cost vs the pure TMA GEMV (N = 15360, fixed iteration counts)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib  # noqa: E402
from paper_1212_3032_b200.linsolve import _Workspace, gmres_device  # noqa: E402

lib = _lib.load()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 15360
g = torch.Generator(device="cuda")
g.manual_seed(0)
A = torch.randn((n, n), dtype=torch.complex128, device="cuda", generator=g)
A.diagonal().add_(0.5 * n ** 0.5)
b = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
y = torch.empty_like(b)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


gemv = timed(lambda: _lib.check(lib.ewb_gemv_batched(_lib.ptr(A), _lib.ptr(b), _lib.ptr(y), n, 1,
                                                     _lib.stream_handle())), 10)
print(f"gemv {gemv:.4f} ms  {16 * n * n / gemv / 1e6:.1f} GB/s")
import os  # noqa: E402
pinv = None
if os.environ.get("PC"):
    pinv = torch.eye(3, dtype=torch.complex128, device="cuda").repeat(n // 3, 1, 1)
    pinv += 0.01 * torch.randn(pinv.shape, dtype=torch.complex128, device="cuda", generator=g)
ws = _Workspace()
for m in (1, 10, 30, 59):
    x = torch.zeros(n, dtype=torch.complex128, device="cuda")
    stats = {}

    def run():
        x.zero_()
        stats["st"] = gmres_device(A, b, x, False, 1e-300 if False else 1e-15, 60, m, pinv, ws=ws,
                                   sync=False)

    ms = timed(run)
    print(f"its={m:3d}  {ms:8.3f} ms  per-pass {ms / (m + 1):.4f} ms  overhead/iter "
          f"{(ms - (m + 1) * gemv) / m * 1e3:.1f} us")
