"""Dump per-frequency GMRES residual histories of the GPU cfg1 sweep."""
import sys, json
sys.path.insert(0, ".")
import numpy as np
from paper_1212_3032_b200 import run_sweep
from paper_1212_3032_b200.workloads import cfg1
res = run_sweep(cfg1())
out = {str(s.k): dict(its=s.iterations, init=s.init_residual, final=s.final_residual,
                      hist=s.residual_history) for s in res.stats}
json.dump(out, open("gpurun_out/cfg1_stats.json", "w"))
print("elapsed", res.manifest["elapsed_seconds"])
