"""Time one matrix-free operator application (K=1 and K=5) on an icosphere.

python tools/mf_time.py [level] [lib.so]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib  # noqa: E402

if len(sys.argv) > 2:
    _lib.load(sys.argv[2])
from paper_1212_3032_b200 import Assembler, MatrixFreeOperator  # noqa: E402
from paper_1212_3032_b200.workloads import sphere_pressure  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cfg = sphere_pressure(level, 64)
asm = Assembler(cfg.mesh, cfg.material)
pe = asm.point_evals()
res = []
for om in (0.25 - 0.375j * 0.632, 8.0 - 0.237j):
    op = MatrixFreeOperator(asm, om)
    for K in (1, 5):
        v = torch.randn((K, asm.n), dtype=torch.complex128, device="cuda")
        op.apply_multi(v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply_multi(v)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res.append((round(om.real, 2), K, round(ms, 1), round(pe / ms / 1e6, 2)))
print(sys.argv[2].split("/")[-1] if len(sys.argv) > 2 else "default",
      "(omega_re, K, ms, Gpoint/s):", res)
