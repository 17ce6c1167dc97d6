"""cfg5 (ico6 cavity, 81,920 el / 245,760 DOF) matrix-free: setup, one operator
application, and the first `nk` frequencies of the sweep.

python tools/cfg5_probe.py [nk]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib  # noqa: E402
from paper_1212_3032_b200.driver import DeviceSweep  # noqa: E402
from paper_1212_3032_b200.matfree import MatrixFreeOperator  # noqa: E402
from paper_1212_3032_b200.workloads import cfg5  # noqa: E402

nk = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = cfg5()
t0 = time.perf_counter()
ds = DeviceSweep(cfg, frequencies=list(range(nk)))
torch.cuda.synchronize()
setup = time.perf_counter() - t0
pc = ds.asm.pair_counts()
op = MatrixFreeOperator(ds.asm, complex(ds.omegas[1]))
v = torch.randn((1, ds.n), dtype=torch.complex128, device="cuda")
op.apply_multi(v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
op.apply_multi(v)
e1.record()
torch.cuda.synchronize()
t1 = e0.elapsed_time(e1)
v5 = torch.randn((5, ds.n), dtype=torch.complex128, device="cuda")
e0.record()
op.apply_multi(v5)
e1.record()
torch.cuda.synchronize()
t5 = e0.elapsed_time(e1)
ds.matrix_free = True
t2 = time.perf_counter()
stats = ds.run()
sweep_part = time.perf_counter() - t2
pe = ds.asm.point_evals()
out = dict(setup_s=setup, pairs=pc, point_evals_per_application=pe, apply_ms_k1=t1,
           apply_ms_k5=t5, point_evals_per_s=pe / (t1 * 1e-3),
           first_freqs={k: (s.iterations, s.init_residual, s.final_residual, s.matvecs,
                            round(s.seconds, 3)) for k, s in stats.items()},
           first_freqs_seconds=sweep_part)
print(json.dumps(out))
