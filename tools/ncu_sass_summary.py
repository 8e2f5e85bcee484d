"""Summarise an ncu report's SASS source page: executed instructions and
stall samples by opcode, plus the hottest instructions.  Usage:
  python tools/ncu_sass_summary.py gpurun_out/x.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
iS, iSt, iEx = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
by_op = collections.defaultdict(lambda: [0.0, 0.0])
inst = []
for idx, r in enumerate(rows[1:]):
    try:
        st, ex = float(r[iSt] or 0), float(r[iEx] or 0)
    except ValueError:
        continue
    src = r[iS].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    by_op[op][0] += st
    by_op[op][1] += ex
    inst.append((st, ex, idx, src[:90]))
TS = sum(v[0] for v in by_op.values()) or 1
TE = sum(v[1] for v in by_op.values()) or 1
print(f"total stall samples {TS:.0f}; executed warp instructions {TE:.4e}")
print("-- by opcode (stall %, inst %)")
for op, (st, ex) in sorted(by_op.items(), key=lambda x: -x[1][1])[:25]:
    print(f"  {op:10s} {100*st/TS:5.1f}% {100*ex/TE:5.1f}%  {ex:.3e}")
print("-- hottest instructions by stall samples")
for st, ex, idx, src in sorted(inst, reverse=True)[:top]:
    print(f"  {100*st/TS:5.1f}% st {ex:10.3e} ex  #{idx:5d} {src}")


def top_by(col, k=12):
    j = h.index(col)
    items = []
    for idx, r in enumerate(rows[1:]):
        try:
            items.append((float(r[j] or 0), idx, r[iS].strip()[:80], float(r[iEx] or 0)))
        except ValueError:
            pass
    items.sort(reverse=True)
    tot = sum(x[0] for x in items) or 1
    print(f"-- top by {col} (total {tot:.0f})")
    for v, idx, src, ex in items[:k]:
        print(f"  {100*v/tot:5.1f}%  #{idx:5d} ex {ex:10.3e}  {src}")


if len(sys.argv) > 3:
    for c in sys.argv[3].split(","):
        top_by(c)
