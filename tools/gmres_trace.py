"""Phase trace of one k_gmres launch (CTA 0, %globaltimer): where the time goes."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 15360
m = int(sys.argv[2]) if len(sys.argv) > 2 else 30
probe = torch.zeros(1 << 16, dtype=torch.int64, device="cuda")
os.environ["EWB_GMRES_PROBE"] = str(probe.data_ptr())
from paper_1212_3032_b200.linsolve import _Workspace, gmres_device  # noqa: E402

g = torch.Generator(device="cuda")
g.manual_seed(0)
A = torch.randn((n, n), dtype=torch.complex128, device="cuda", generator=g)
A.diagonal().add_(0.5 * n ** 0.5)
b = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
x = torch.zeros(n, dtype=torch.complex128, device="cuda")
ws = _Workspace()
gmres_device(A, b, x, False, 1e-15, 60, m, None, ws=ws)
probe.zero_()
x.zero_()
gmres_device(A, b, x, False, 1e-15, 60, m, None, ws=ws)
torch.cuda.synchronize()
p = probe.cpu().numpy().astype(np.uint64)
p = p[p != 0]
ids = (p >> np.uint64(56)).astype(int)
ts = (p & np.uint64((1 << 56) - 1)).astype(np.int64)
dt = np.diff(ts)
acc = {}
for a_, b_, d in zip(ids[:-1], ids[1:], dt):
    acc.setdefault((a_, b_), []).append(d)
names = {2: "iter start", 3: "matvec done (CTA0)", 4: "after grid.sync", 5: "dots+reduce",
         6: "tri solve + w update", 7: "norm grid_sum", 8: "givens", 9: "v/z phase",
         10: "iter end sync", 11: "x update", 12: "residual matvec", 13: "slice_dots", 14: "dots sync"}
tot = ts[-1] - ts[0]
print(f"n={n} its={m} traced {tot / 1e3:.1f} us")
for (a_, b_), v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f"{names.get(a_, a_):>22s} -> {names.get(b_, b_):<22s} n={len(v):3d} "
          f"mean {np.mean(v) / 1e3:8.2f} us  total {sum(v) / 1e3:9.1f} us")
mv = [int(d) for a_, b_, d in zip(ids[:-1], ids[1:], dt) if a_ == 2 and b_ == 3]
dd = [int(d) for a_, b_, d in zip(ids[:-1], ids[1:], dt) if a_ == 4 and b_ == 5]
print("matvec us by j:", [round(v / 1e3) for v in mv])
print("dots us by j:", [round(v / 1e3, 1) for v in dd])
