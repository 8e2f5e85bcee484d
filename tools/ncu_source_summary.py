"""Summarise an ncu report's source page: per CUDA source line, executed
instructions and stall samples (needs -lineinfo).  Usage:
  python tools/ncu_source_summary.py gpurun_out/x.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# skip the "Kernel Name" preamble line(s)
start = next(i for i, l in enumerate(lines) if l.startswith('"#"') or l.startswith('"Line"') or l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
def col(name):
    for i, x in enumerate(h):
        if x.startswith(name):
            return i
    return None
ci = {k: col(k) for k in ["#", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed"]}
data = []
for r in rows[1:]:
    try:
        ex = float(r[ci["Instructions Executed"]] or 0)
        st = float(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, TypeError, IndexError):
        continue
    data.append((st, ex, r[ci["#"]] if ci["#"] is not None else "", r[ci["Source"]].strip()[:110]))
TS = sum(d[0] for d in data) or 1
TE = sum(d[1] for d in data) or 1
print(f"total stall samples {TS:.0f}, executed instructions {TE:.3e}")
for st, ex, ln, src in sorted(data, reverse=True)[:top]:
    print(f"{100*st/TS:5.1f}% stall {100*ex/TE:5.1f}% inst  L{ln:>5s}  {src}")
