make all >/dev/null
for K in k_merge_sample k_rev_select k_join; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/s11_$K python tools/prof_build.py --iters 7 > /dev/null 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s11_launches.csv python tools/prof_build.py --iters 7 > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/s11_tests.log
