"""Build a compile-time variant of the library for A/B timing on the GPU box.

python tools/build_variant.py NAME -DFLAG[=V] ...   ->  paper_1212_3032_b200/variants/NAME.so
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1212_3032_b200.build import ARCH, CSRC, PKG, SOURCES, nvcc  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = PKG / "variants"
tmp = out_dir / f"{name}.o.d"
tmp.mkdir(parents=True, exist_ok=True)
procs, objs = [], []
for src in SOURCES:
    obj = tmp / (src + ".o")
    objs.append(str(obj))
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
           "-diag-suppress", "177", *defs, "-c", str(CSRC / src), "-o", str(obj)]
    procs.append(subprocess.Popen(cmd))
assert all(p.wait() == 0 for p in procs)
so = out_dir / f"{name}.so"
subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(so), *objs], check=True)
print(so)
