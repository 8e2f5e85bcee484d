"""Executed warp instructions and stall samples of one kernel per CUDA source
line: the ncu report's SASS page (per-instruction counts, in address order)
aligned with `nvdisasm -g` of the same build's cubin (line annotations).
Usage: python tools/ncu_lines.py gpurun_out/x.ncu-rep <mangled kernel name> [top]
(the cubin is extracted from paper_2103_15386_b200/lib/libknng.so; the report
must come from the same build)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(out) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(out[start:]))))
h = rows[0]
E, A = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
counts = [(float(r[E] or 0), float(r[A] or 0)) for r in rows[1:]]

with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2103_15386_b200/lib/libknng.so")],
                   cwd=td, capture_output=True)
    cubin = next(os.path.join(td, f) for f in os.listdir(td) if f.endswith(".cubin"))
    sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
i0 = next(i for i, l in enumerate(sass) if l.startswith(".text." + fn + ":"))
line = None
lines = []
for l in sass[i0 + 1:]:
    if l.startswith(".text.") or l.startswith("\t.section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        lines.append(line)
if len(lines) != len(counts):
    print(f"warning: {len(lines)} SASS instructions vs {len(counts)} profiled (different build?)")
agg = collections.defaultdict(lambda: [0.0, 0.0])
for ln, (ex, st) in zip(lines, counts):
    agg[ln][0] += ex
    agg[ln][1] += st
TE = sum(v[0] for v in agg.values()) or 1
TS = sum(v[1] for v in agg.values()) or 1
print(f"{'source line':34s} {'inst %':>7s} {'stall %':>8s}")
for ln, (ex, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{str(ln):34s} {100 * ex / TE:7.2f} {100 * st / TS:8.2f}")
