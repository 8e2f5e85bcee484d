"""One-page summary of an `ncu --set full` report for profiles/: key raw
metrics (duration, DRAM bytes, issue/pipe utilisation, occupancy) and the
executed-instruction histogram by opcode.  Usage:
  python tools/ncu_report.py gpurun_out/x.ncu-rep "title" > profiles/....txt"""
import collections
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
METRICS = [
    "Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tmem_cycles_active.avg.pct_of_peak_sustained_active",
]
print(f"# ncu --set full --clock-control none: {title}")
for m in METRICS:
    if m in h:
        i = h.index(m)
        print(f"{m}: {v[i]} {u[i]}".rstrip())
for i, m in enumerate(h):
    if "pipe_tensor" in m and "pct_of_peak_sustained_active" in m and m not in METRICS:
        print(f"{m}: {v[i]} {u[i]}")
stalls = []
for i, m in enumerate(h):
    if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued"):
        try:
            stalls.append((float(v[i].replace(",", "")), m.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
T = sum(x for x, _ in stalls) or 1
print("-- stall samples: " + ", ".join(f"{n} {100 * x / T:.1f}%" for x, n in sorted(stalls, reverse=True)[:8]))

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
try:
    start = next(i for i, l in enumerate(src) if l.startswith('"Address"'))
    srows = list(csv.reader(io.StringIO("\n".join(src[start:]))))
    sh = srows[0]
    S, E = sh.index("Source"), sh.index("Instructions Executed")
    ops = collections.Counter()
    for r in srows[1:]:
        s = r[S].strip()
        op = s.split()[0] if s else "?"
        if op.startswith("@"):
            op = s.split()[1]
        ops[op.split(".")[0]] += float(r[E] or 0)
    TE = sum(ops.values()) or 1
    print("-- executed warp instructions by opcode: " +
          ", ".join(f"{o} {100 * c / TE:.1f}%" for o, c in ops.most_common(14)))
except StopIteration:
    pass
