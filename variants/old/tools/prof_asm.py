"""Profiling driver for the dense assembly: cfg2 context + assemble_system at k.

python tools/prof_asm.py [k] [repeats]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import Assembler  # noqa: E402
from paper_1212_3032_b200.transform import eta_from_kappa, frequency_grid  # noqa: E402
from paper_1212_3032_b200.workloads import cfg2  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = cfg2()
asm = Assembler(cfg.mesh, cfg.material)
om = frequency_grid(cfg.period, cfg.n_omega, eta_from_kappa(cfg.kappa, cfg.period))
p = torch.ones(cfg.mesh.n_dofs, dtype=torch.complex128, device="cuda")
sysm = None
for _ in range(reps):
    sysm = asm.assemble_system(om[k], cfg.bcs, p, out=sysm, check=False)
torch.cuda.synchronize()
print("ok", k)
