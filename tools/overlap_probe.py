"""Concurrency probe: one GMRES solve (stream A) with the next frequency's
assembly (stream B) started once the solver is resident.

python tools/overlap_probe.py [lib.so] [its]
Prints standalone and overlapped times of both.
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    _lib.load(sys.argv[1])
its = int(sys.argv[2]) if len(sys.argv) > 2 else 40
from paper_1212_3032_b200 import workloads  # noqa: E402
from paper_1212_3032_b200.assembly import Assembler  # noqa: E402
from paper_1212_3032_b200.linsolve import gmres_device  # noqa: E402
from paper_1212_3032_b200.driver import DeviceSweep  # noqa: E402

cfg = workloads.cfg2()
sw = DeviceSweep(cfg)
asm = sw.asm
k1, k2 = 20, 21
s1 = asm.assemble_system(sw.omegas[k1], cfg.bcs, sw.P[k1])
s2 = asm.assemble_system(sw.omegas[k2], cfg.bcs, sw.P[k2])
x = torch.zeros(sw.n, dtype=torch.complex128, device="cuda")
torch.cuda.synchronize()


def ev():
    return torch.cuda.Event(enable_timing=True)


def solve():
    x.zero_()
    gmres_device(s1.A, s1.b, x, False, 1e-15, 60, its, s1.pinv, sync=False)


def assemble():
    asm.assemble_system(sw.omegas[k2], cfg.bcs, sw.P[k2], out=s2, check=False)


for _ in range(2):
    solve()
    assemble()
torch.cuda.synchronize()
e = [ev() for _ in range(4)]
e[0].record(); solve(); e[1].record()
e[2].record(); assemble(); e[3].record()
torch.cuda.synchronize()
t_solve, t_asm = e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])
print(f"standalone: solve {t_solve:.2f} ms  assembly {t_asm:.2f} ms  sum {t_solve + t_asm:.2f}")

sa = torch.cuda.Stream(priority=-1)
sb = torch.cuda.Stream(priority=0)
for delay in (0.0, 0.002):
    torch.cuda.synchronize()
    f = [ev() for _ in range(4)]
    with torch.cuda.stream(sa):
        f[0].record(sa)
        solve()
        f[1].record(sa)
    time.sleep(delay)
    with torch.cuda.stream(sb):
        f[2].record(sb)
        assemble()
        f[3].record(sb)
    torch.cuda.synchronize()
    ts, ta = f[0].elapsed_time(f[1]), f[2].elapsed_time(f[3])
    tot = max(f[0].elapsed_time(f[1]), f[0].elapsed_time(f[3]))
    print(f"overlap (host delay {delay * 1e3:.0f} ms): solve {ts:.2f} ms  assembly {ta:.2f} ms  "
          f"span {tot:.2f} ms  asm start after solve start {f[0].elapsed_time(f[2]):.2f} ms")
