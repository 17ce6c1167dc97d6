"""Profiling driver: cfg2 context + one frequency (assembly, SEM, GMRES).

Used under ncu (launch list and --set full on the top kernels); small enough
that ncu's per-kernel replay stays bounded.
    python tools/prof_cfg2.py [k]
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import Assembler  # noqa: E402
from paper_1212_3032_b200.driver import DeviceSweep  # noqa: E402
from paper_1212_3032_b200.workloads import cfg2  # noqa: E402

k_stop = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cfg = cfg2()
ds = DeviceSweep(cfg, frequencies=list(range(k_stop)))
stats = ds.run()
torch.cuda.synchronize()
print({k: (s.iterations, s.matvecs) for k, s in stats.items()})
