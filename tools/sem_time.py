"""Time one SEM initial guess (Y = A X pass + QR) at N = 15360, K = 1..4."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.load(sys.argv[1])
from paper_1212_3032_b200.linsolve import sem_device  # noqa: E402

n = 15360
g = torch.Generator(device="cuda")
g.manual_seed(0)
A = torch.randn((n, n), dtype=torch.complex128, device="cuda", generator=g)
b = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
X = torch.randn((4, n), dtype=torch.complex128, device="cuda", generator=g)
x0 = torch.empty_like(b)
for K in (1, 2, 3, 4):
    for _ in range(2):
        sem_device(A, b, X[:K], 1e-10, x0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        sem_device(A, b, X[:K], 1e-10, x0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    # check: x0 minimises |A X s - b| -> residual orthogonal to A X
    Y = (A @ X[:K].T)
    r = b - A @ x0
    orth = float((Y.conj().T @ r).abs().max() / (Y.abs().max() * r.abs().max() * n))
    print(f"K={K}: {ms:.3f} ms per SEM guess  ({16 * n * n / ms / 1e6:.0f} GB/s for one A pass)  "
          f"orthogonality {orth:.1e}")
