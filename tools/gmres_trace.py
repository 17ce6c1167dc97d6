"""Phase trace of one k_gmres launch (CTA 0, %globaltimer).

python tools/gmres_trace.py [n] [iterations] [lib.so]
Prints the mean duration between consecutive probe ids.
"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 15360
m = int(sys.argv[2]) if len(sys.argv) > 2 else 30
probe = torch.zeros(1 << 16, dtype=torch.int64, device="cuda")
os.environ["EWB_GMRES_PROBE"] = str(probe.data_ptr())
from paper_1212_3032_b200 import _lib  # noqa: E402

if len(sys.argv) > 3:
    _lib.load(sys.argv[3])
from paper_1212_3032_b200.linsolve import _Workspace, gmres_device  # noqa: E402

g = torch.Generator(device="cuda")
g.manual_seed(0)
A = torch.randn((n, n), dtype=torch.complex128, device="cuda", generator=g)
A.diagonal().add_(0.5 * n ** 0.5)
b = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
x = torch.zeros(n, dtype=torch.complex128, device="cuda")
ws = _Workspace()
if os.environ.get("TRACE_BALANCE"):
    from paper_1212_3032_b200.linsolve import calibrate_row_balance

    print("row balance stats (us):", calibrate_row_balance(A))
gmres_device(A, b, x, False, 1e-15, 60, m, None, ws=ws)
probe.zero_()
x.zero_()
gmres_device(A, b, x, False, 1e-15, 60, m, None, ws=ws)
torch.cuda.synchronize()
p = probe.cpu().numpy()[:32768].astype(np.uint64)
p = p[p != 0]
ids = (p >> np.uint64(56)).astype(int)
ts = (p & np.uint64((1 << 56) - 1)).astype(np.int64)
acc = {}
for a_, b_, d in zip(ids[:-1], ids[1:], np.diff(ts)):
    acc.setdefault((a_, b_), []).append(d)
print(f"n={n} its={m} traced {(ts[-1] - ts[0]) / 1e3:.1f} us")
for (a_, b_), v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f"{a_:3d} -> {b_:3d}  n={len(v):3d}  mean {np.mean(v) / 1e3:8.2f} us  "
          f"total {sum(v) / 1e3:9.1f} us")

# per-CTA matvec finish times (first cycle), relative to the earliest CTA
P = probe.cpu().numpy()[32768:].astype(np.int64)
G = 148
rows = []
for j in range(min(m, 100)):
    t = P[j * G:(j + 1) * G]
    if (t == 0).any():
        break
    rows.append(t - t.min())
if rows:
    R = np.array(rows) / 1e3
    print(f"matvec finish spread per step: mean max-min {R.max(1).mean():.2f} us, "
          f"median CTA lag {np.median(R, 1).mean():.2f} us")
    lag = R[1:].mean(0)
    order = np.argsort(-lag)
    print("slowest CTAs (mean lag us):", [(int(b), round(float(lag[b]), 2)) for b in order[:12]])
    print("fastest CTAs:", [(int(b), round(float(lag[b]), 2)) for b in order[-6:]])

    sm = P[100 * G:101 * G]
    print("smid of the 12 slowest CTAs:", [int(sm[b]) for b, _ in sorted(enumerate(lag), key=lambda t: -t[1])[:12]])
    np.save(os.environ.get("TRACE_OUT", "/tmp/trace_lag.npy"), np.stack([np.arange(G), sm, lag]))
