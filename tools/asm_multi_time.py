"""cfg2: multi-frequency fused assembly (ewb_assemble_system_multi) vs the
single-frequency kernels — time per frequency and max member deviation.

python tools/asm_multi_time.py [LIB.so]
"""
import os
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
tag = sys.argv[1].split("/")[-1] if len(sys.argv) > 1 else "default"


def timed(fn, reps=5 if os.environ.get('ASM_QUICK') == '1' else 3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


P = torch.ones((32, n), dtype=torch.complex128, device="cuda")
single = asm.assemble_system(om[1], cfg.bcs, P[0], check=False)
batch = None
QUICK = os.environ.get("ASM_QUICK") == "1"   # one batch position, nf = 16 only
for k0 in ((60,) if QUICK else (1, 60, 96)):
    t1 = timed(lambda: asm.assemble_system(om[k0], cfg.bcs, P[0], out=single, check=False))
    row = [f"k0={k0} single {t1:.3f} ms"]
    for nf in ((16,) if QUICK else (8, 16, 24, 32)):
        if batch is not None and batch.A.shape[0] < nf:
            batch = None
            torch.cuda.empty_cache()
        batch = asm.assemble_system_multi(om[k0:k0 + nf], cfg.bcs, P[:nf], out=batch, check=False)
        tb = timed(lambda: asm.assemble_system_multi(om[k0:k0 + nf], cfg.bcs, P[:nf], out=batch,
                                                     check=False))
        dev = 0.0
        for f in (0, nf - 1):
            s = asm.assemble_system(om[k0 + f], cfg.bcs, P[0], out=single, check=False)
            amax = torch.abs(s.A).max().item()
            dev = max(dev, torch.abs(batch.A[f] - s.A).max().item() / amax)
        row.append(f"nf={nf} {tb / nf:.3f} ms/freq (dev {dev:.1e})")
    print(tag, " | ".join(row), flush=True)
