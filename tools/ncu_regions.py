"""Region x stall-reason table of an ncu report (SASS page), regions split at
barrier/wait instructions given as index boundaries.  Usage:
  python tools/ncu_regions.py rep.ncu-rep            -> list sync markers
  python tools/ncu_regions.py rep.ncu-rep a:b:name,c:d:name2"""
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
data = rows[1:]
S, Ex, A = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
if len(sys.argv) < 3:
    for i, r in enumerate(data):
        s = r[S]
        if any(k in s for k in ("TRYWAIT", "BAR.SYNC", "EXIT", "ARRIVE", "LDGSTS", "ATOMG", "STG")):
            print(i, s.strip()[:70], r[Ex], r[A])
    sys.exit(0)
cols = ["stall_long_sb", "stall_wait", "stall_short_sb", "stall_barrier", "stall_sleep", "stall_selected",
        "stall_not_selected", "stall_dispatch", "stall_math", "stall_no_inst", "stall_lg", "stall_mio"]
ci = [h.index(c) for c in cols]
T = sum(float(r[A] or 0) for r in data)
E = sum(float(r[Ex] or 0) for r in data)
print("region            samp%  inst%  " + " ".join(c.replace("stall_", "")[:7].rjust(7) for c in cols))
for spec in sys.argv[2].split(","):
    lo, hi, name = spec.split(":")
    lo, hi = int(lo), (int(hi) if hi else len(data))
    a = sum(float(r[A] or 0) for r in data[lo:hi])
    e = sum(float(r[Ex] or 0) for r in data[lo:hi])
    parts = [sum(float(r[j] or 0) for r in data[lo:hi]) for j in ci]
    print(f"{name:16s} {100*a/T:5.1f} {100*e/E:5.1f}  " + " ".join(f"{100*p/T:7.1f}" for p in parts))
