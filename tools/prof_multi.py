"""One cfg2 multi-frequency assembly (nf=8 at k0=60) and one single-frequency
assembly at k=60, for ncu launch lists / captures of the assembly kernels."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.load(sys.argv[1])
from paper_1212_3032_b200 import Assembler  # noqa: E402
from paper_1212_3032_b200.transform import eta_from_kappa, frequency_grid  # noqa: E402
from paper_1212_3032_b200.workloads import cfg2  # noqa: E402

cfg = cfg2()
asm = Assembler(cfg.mesh, cfg.material)
om = frequency_grid(cfg.period, cfg.n_omega, eta_from_kappa(cfg.kappa, cfg.period))
n = cfg.mesh.n_dofs
P = torch.ones((8, n), dtype=torch.complex128, device="cuda")
asm.assemble_system_multi(om[60:68], cfg.bcs, P, check=False)
asm.assemble_system(om[60], cfg.bcs, P[0], check=False)
torch.cuda.synchronize()
print("done")
