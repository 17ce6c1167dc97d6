"""Time the fused dense assembly (ewb_assemble_system) for cfg2 at a few k.

python tools/asm_time.py [LIB.so]
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.load(sys.argv[1])
from paper_1212_3032_b200 import Assembler  # noqa: E402
from paper_1212_3032_b200.transform import eta_from_kappa, frequency_grid  # noqa: E402
from paper_1212_3032_b200.workloads import cfg2  # noqa: E402

cfg = cfg2()
asm = Assembler(cfg.mesh, cfg.material)
eta = eta_from_kappa(cfg.kappa, cfg.period)
om = frequency_grid(cfg.period, cfg.n_omega, eta)
p = torch.ones(cfg.mesh.n_dofs, dtype=torch.complex128, device="cuda")
sysm = None
out = []
for k in (1, 32, 64, 128):
    sysm = asm.assemble_system(om[k], cfg.bcs, p, out=sysm, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        asm.assemble_system(om[k], cfg.bcs, p, out=sysm, check=False)
    e1.record()
    torch.cuda.synchronize()
    out.append((k, round(e0.elapsed_time(e1) / 5, 3)))
ref = sysm.A[:3, :6].cpu().numpy()
print((sys.argv[1].split("/")[-1] if len(sys.argv) > 1 else "default"), out,
      "checksum", float(np.abs(sysm.A.sum().item())))
