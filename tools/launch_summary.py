"""Summarise an ncu --metrics gpu__time_duration.sum launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("knng::", "").strip()
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':22s} {'launches':>8s} {'total ms':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:22s} {cnt[k]:8d} {v:9.3f} {100 * v / T:5.1f}%")
print(f"{'total':22s} {sum(cnt.values()):8d} {T:9.3f}")
