"""One matrix-free application (K=1) on an icosphere of the given level, for ncu."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import Assembler, MatrixFreeOperator  # noqa: E402
from paper_1212_3032_b200.workloads import sphere_pressure  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = sphere_pressure(level, 64)
asm = Assembler(cfg.mesh, cfg.material)
op = MatrixFreeOperator(asm, 8.0 - 0.237j)
v = torch.randn((1, asm.n), dtype=torch.complex128, device="cuda")
op.apply_multi(v)
torch.cuda.synchronize()
print("done")
