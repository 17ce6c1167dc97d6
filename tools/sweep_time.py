"""cfg2 sweep time (device-resident DeviceSweep.run) for a library variant."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.load(sys.argv[1])
from paper_1212_3032_b200 import workloads  # noqa: E402
from paper_1212_3032_b200.driver import DeviceSweep  # noqa: E402

ds = DeviceSweep(workloads.cfg2())
ds.run()
for _ in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = ds.run(timing=True)
    e1.record()
    torch.cuda.synchronize()
    its = sum(s.iterations for s in st.values())
    print(f"{sys.argv[1] if len(sys.argv) > 1 else 'default'}: sweep {e0.elapsed_time(e1):.1f} ms  "
          f"asm {ds.phase['assembly_ms']:.0f}  solve {ds.phase['solve_ms']:.0f}  its {its}  "
          f"passes {ds.phase['matvecs']}")
