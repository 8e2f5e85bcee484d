# End-of-round GPU evidence: parity tests, smoke, bench (N=1), launch list and
# ncu --set full captures of the main kernels, all from the current build.
# The .ncu-rep files are summarised ON THE BOX (tools/ncu_report.py,
# tools/ncu_callsites.py) and only the join's report is kept: gpurun copies
# back at most 64 MiB.
T=${1:-final}
make all >/dev/null || exit 1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/${T}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/prof_build.py --iters 7 > /dev/null 2>&1
bash tools/prof_kernels.sh ${T}
for K in k_join k_merge_sample k_rev_select k_rev_scatter; do
  R=gpurun_out/${T}_$K.ncu-rep
  [ -f $R ] || continue
  python tools/ncu_report.py $R "$K, C2 build (${T})" > gpurun_out/${T}_ncu_$K.txt 2>&1
  timeout 300 python tools/ncu_callsites.py $R auto 40 >> gpurun_out/${T}_ncu_$K.txt 2>&1
  [ $K = k_join ] || rm -f $R
done
