"""Opcode histogram (instructions executed, stall samples) of an ncu report's SASS page.
Usage: python tools/ncu_sass_ops.py rep.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
S, E, A = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter()
st = collections.Counter()
for r in rows[1:]:
    src = r[S].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += float(r[E] or 0)
    st[op] += float(r[A] or 0)
T = sum(ops.values())
TS = sum(st.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"total warp instructions {T:.3e}")
for op, v in ops.most_common(top):
    print(f"{op:12s} {v:14.0f} {100 * v / T:5.1f}%  stall-samples {100 * st[op] / max(TS, 1):5.1f}%")
