"""K = 5 matrix-free pass (b + 4 SEM columns) with and without the
per-vector T / U masks, all-Neumann icosphere.  python tools/mf_mask_time.py [level]"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import Assembler, MatrixFreeOperator  # noqa: E402
from paper_1212_3032_b200.workloads import sphere_pressure  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = sphere_pressure(level, 64)
asm = Assembler(cfg.mesh, cfg.material)
n = asm.n
for om in (0.25 - 0.237j, 8.0 - 0.237j):
    op = MatrixFreeOperator(asm, om)
    V = torch.randn((4, n), dtype=torch.complex128, device="cuda")
    p = torch.randn(n, dtype=torch.complex128, device="cuda")
    vt = torch.cat([V, torch.zeros((1, n), dtype=V.dtype, device="cuda")]).contiguous()
    vu = torch.cat([torch.zeros_like(V), p[None]]).contiguous()
    res = {}
    for name, masks in (("unmasked", None), ("masked", (0b01111, 0b10000))):
        y = op._apply_tu(vt, vu, True, masks)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            y = op._apply_tu(vt, vu, True, masks)
        e1.record()
        torch.cuda.synchronize()
        res[name] = (e0.elapsed_time(e1) / 3, y.clone())
    d = (res["masked"][1] - res["unmasked"][1]).abs().max() / res["unmasked"][1].abs().max()
    print(f"omega {om}: unmasked {res['unmasked'][0]:.1f} ms  masked {res['masked'][0]:.1f} ms  "
          f"max rel diff {float(d):.1e}")
