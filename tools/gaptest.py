"""Sweep wall/GPU time with and without the bench's clock sampler and outputs."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_1212_3032_b200 import workloads  # noqa: E402
from paper_1212_3032_b200.driver import DeviceSweep  # noqa: E402
from paper_1212_3032_b200.transform import windowed_inverse_device  # noqa: E402

cfg = workloads.cfg2()
ds = DeviceSweep(cfg)


def step(outputs):
    ds.run(timing=True)
    if outputs:
        half = ds.probe_half(cfg.probes)
        windowed_inverse_device(half, cfg.window, ds.eta, cfg.period)


for sampler in (False, True):
    for outputs in (False, True):
        step(outputs)
        torch.cuda.synchronize()
        cs = ClockSampler(0) if sampler else None
        t0 = time.perf_counter()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        step(outputs)
        s1.record()
        torch.cuda.synchronize()
        if cs:
            cs.stop()
        p = ds.phase
        print(f"sampler={sampler} outputs={outputs}: wall {time.perf_counter() - t0:.3f}s "
              f"gpu {s0.elapsed_time(s1):.1f} ms asm {p['assembly_ms']:.0f} solve "
              f"{p['solve_ms']:.0f} gaps {p.get('gap_ms', 0):.1f}")
