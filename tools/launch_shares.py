"""Per-kernel totals and shares of an ncu launch list (--metrics
gpu__time_duration.sum --csv).  python tools/launch_shares.py FILE [regex-exclude]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
excl = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "s": 1e6, "second": 1e6}
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= mi or not r[mi]:
        continue
    name = r[ki].split("(")[0]
    if excl and excl.search(name):
        continue
    tot[name] += float(r[mi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T / 1e3:.1f} ms over {sum(cnt.values())} launches")
for k, v in tot.most_common(25):
    print(f"{k:58s} {cnt[k]:6d} {v / 1e3:10.2f} ms {100 * v / T:6.2f} %")
