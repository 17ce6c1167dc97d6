"""Instruction mix of a kernel's hottest loop from an ncu report's SASS
source page.  python tools/ncu_hotloop.py REPORT.ncu-rep [frac]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) >= len(h)]


def op(src):
    t = src.split()
    if not t:
        return ""
    o = t[1] if t[0].startswith("@") else t[0]
    return o.split(".")[0]


n = [float(r[ix["Instructions Executed"]] or 0) for r in data]
tot = sum(n)
mix = collections.Counter()
for r, c in zip(data, n):
    mix[op(r[ix["Source"]].strip())] += c
print(f"total warp instructions {tot:.3e}")
print("whole kernel:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in mix.most_common(12)))
mx = max(n)
body = [(r, c) for r, c in zip(data, n) if c >= frac * mx]
cnt = collections.Counter(op(r[ix["Source"]].strip()) for r, _ in body)
fp64 = sum(v for k, v in cnt.items() if k in ("DFMA", "DMUL", "DADD"))
print(f"hot body (exec >= {frac} x max = {mx:.3e}): {len(body)} instructions, FP64 {fp64}")
print("  ", ", ".join(f"{k} {v}" for k, v in cnt.most_common(20)))
