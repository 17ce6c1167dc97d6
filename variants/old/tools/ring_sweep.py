"""Time the TMA GEMV for one library variant: python tools/ring_sweep.py LIB.so"""
import math
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib  # noqa: E402

lib = _lib.load(sys.argv[1])
out = {}
for n, batch in ((15360, 1), (16384, 8)):
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    A = torch.randn((batch, n, n), dtype=torch.complex128, device="cuda", generator=g)
    x = torch.randn((batch, n), dtype=torch.complex128, device="cuda", generator=g)
    y = torch.empty_like(x)

    def step():
        _lib.check(lib.ewb_gemv_batched(_lib.ptr(A), _lib.ptr(x), _lib.ptr(y), n, batch,
                                        _lib.stream_handle()))

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    err = float((y[0] - A[0] @ x[0]).abs().max() / (A[0] @ x[0]).abs().max())
    out[(n, batch)] = (round(batch * 16 * n * n / ms / 1e6, 1), err)
    del A
    torch.cuda.empty_cache()
print(sys.argv[1].split("/")[-1], out)
