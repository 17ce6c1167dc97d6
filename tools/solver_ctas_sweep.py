"""Sweep solve-phase time vs the solver CTA budget (SMs left free for
concurrent work).  python tools/solver_ctas_sweep.py [cfg1|cfg2] 148 140 136 132 128"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib, workloads  # noqa: E402
from paper_1212_3032_b200.driver import DeviceSweep  # noqa: E402

lib = _lib.load()
args = sys.argv[1:]
wl = args.pop(0) if args and args[0].startswith("cfg") else "cfg2"
ds = DeviceSweep(getattr(workloads, wl)())
ds.run()
for g in [int(a) for a in args]:
    _lib.check(lib.ewb_set_solver_ctas(g))
    ds.run(timing=True)
    st = ds.run(timing=True)
    print(f"ctas={lib.ewb_solver_ctas()} solve_ms={ds.phase['solve_ms']:.0f} "
          f"asm_ms={ds.phase['assembly_ms']:.0f} its={sum(s.iterations for s in st.values())}",
          flush=True)
_lib.check(lib.ewb_set_solver_ctas(0))
