"""Phase trace (CTA 0, %globaltimer) of the LAST GMRES solve of a full cfg2
sweep, i.e. under the sweep's own clocks and power state (tools/gmres_trace.py
traces a standalone solve).  python tools/sweep_trace.py"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

probe = torch.zeros(1 << 16, dtype=torch.int64, device="cuda")
os.environ["EWB_GMRES_PROBE"] = str(probe.data_ptr())
from paper_1212_3032_b200 import workloads  # noqa: E402
from paper_1212_3032_b200.driver import DeviceSweep  # noqa: E402

ds = DeviceSweep(workloads.cfg2())
ds.run()
probe.zero_()
st = ds.run(timing=True)
torch.cuda.synchronize()
k_last = max(st)
p = probe.cpu().numpy()[:32768].astype(np.uint64)
p = p[p != 0]
ids = (p >> np.uint64(56)).astype(int)
ts = (p & np.uint64((1 << 56) - 1)).astype(np.int64)
acc = {}
for a_, b_, d in zip(ids[:-1], ids[1:], np.diff(ts)):
    acc.setdefault((a_, b_), []).append(d)
print(f"k={k_last} its={st[k_last].iterations} traced {(ts[-1] - ts[0]) / 1e3:.1f} us; "
      f"sweep solve {ds.phase['solve_ms']:.0f} ms, {ds.phase['matvecs']} passes")
for (a_, b_), v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f"{a_:3d} -> {b_:3d}  n={len(v):3d}  mean {np.mean(v) / 1e3:8.2f} us  "
          f"total {sum(v) / 1e3:9.1f} us")
