"""Executed warp instructions, stall samples (with the top stall reasons) and
shared-memory wavefronts of one kernel per CALL SITE: like ncu_lines.py, but
an inlined helper's instructions are charged to the outermost source line
that called it (nvdisasm -gi "inlined at"), so e.g. a barrier wait is split
by the role that waits.  Usage:
  python tools/ncu_callsites.py gpurun_out/x.ncu-rep <mangled kernel> [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(out) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(out[start:]))))
h = rows[0]
E, A = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
WF, WI = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
SR = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]


def f(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2103_15386_b200/lib/libknng.so")],
                   cwd=td, capture_output=True)
    cubin = next(os.path.join(td, x) for x in os.listdir(td) if x.endswith(".cubin"))
    sass = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.splitlines()
if fn == "auto":
    # the report's demangled kernel name -> the cubin's mangled one
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    want = rr[2][rr[0].index("Kernel Name")]
    names = [l[len(".text."):-1] for l in sass if l.startswith(".text.") and l.endswith(":")]
    dem = subprocess.run(["cu++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    def norm(x):  # name and template arguments only (ncu prints parameters as T1, ...)
        x = re.sub(r"\((?:int|bool|unsigned int|long|unsigned long)\)", "", x).split("(")[0]
        return re.sub(r"\s+|void|knng::|\(anonymous namespace\)::", "", x).replace("true", "1").replace("false", "0")
    cand = [m for m, dm in zip(names, dem) if norm(dm) == norm(want)]
    if not cand:
        sys.exit(f"no cubin function matches {want!r}")
    fn = cand[0]
i0 = next(i for i, l in enumerate(sass) if l.startswith(".text." + fn + ":"))
site = None
sites = []
for l in sass[i0 + 1:]:
    if l.startswith(".text.") or l.startswith("\t.section"):
        break
    if l.lstrip().startswith("//## File"):
        locs = re.findall(r'"([^"]+)", line (\d+)', l)
        fl, ln = locs[-1]  # outermost call site
        site = f"{os.path.basename(fl)}:{ln}"
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        sites.append(site)
if len(sites) != len(rows) - 1:
    print(f"warning: {len(sites)} SASS instructions vs {len(rows) - 1} profiled (different build?)")
agg = collections.defaultdict(lambda: {"ex": 0.0, "st": 0.0, "wf": 0.0, "wi": 0.0, "sr": collections.Counter()})
for s, r in zip(sites, rows[1:]):
    a = agg[s]
    a["ex"] += f(r[E])
    a["st"] += f(r[A])
    a["wf"] += f(r[WF])
    a["wi"] += f(r[WI])
    for i, c in SR:
        a["sr"][c[6:]] += f(r[i])
TE = sum(v["ex"] for v in agg.values()) or 1
TS = sum(v["st"] for v in agg.values()) or 1
print(f"{'call site':28s} {'inst %':>7s} {'stall %':>8s} {'smem wf/ideal':>14s}  top stall reasons")
for s, v in sorted(agg.items(), key=lambda x: -x[1]["st"])[:top]:
    tot = sum(v["sr"].values()) or 1
    reasons = ", ".join(f"{k} {100 * c / tot:.0f}%" for k, c in v["sr"].most_common(3) if c > 0)
    wf = f"{v['wf'] / v['wi']:.2f}" if v["wi"] else "-"
    print(f"{str(s):28s} {100 * v['ex'] / TE:7.2f} {100 * v['st'] / TS:8.2f} {wf:>14s}  {reasons}")
