"""Where run_sweep's setup time goes on cfg2 (context creation, spectra,
uploads): cProfile of DeviceSweep(cfg2()) after a warm-up construction."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1212_3032_b200.driver import DeviceSweep  # noqa: E402
from paper_1212_3032_b200.workloads import cfg2  # noqa: E402

cfg = cfg2()
ds = DeviceSweep(cfg)
torch.cuda.synchronize()
del ds
for _ in range(2):
    t0 = time.perf_counter()
    ds = DeviceSweep(cfg)
    torch.cuda.synchronize()
    print("DeviceSweep(cfg2) %.1f ms" % ((time.perf_counter() - t0) * 1e3))
    del ds
pr = cProfile.Profile()
pr.enable()
ds = DeviceSweep(cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
