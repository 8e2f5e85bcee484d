make all >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/s24_tests.log
timeout 300 python tools/kernel_times.py --ns 1000000 > gpurun_out/s24_kt.log 2>&1
timeout 600 python bench.py > gpurun_out/s24_bench.json 2> gpurun_out/s24_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s24_launches.csv python tools/prof_build.py --iters 7 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_join -s 3 -c 1 -o gpurun_out/s24_join python tools/prof_build.py --iters 7 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_merge_sample -s 4 -c 1 -o gpurun_out/s24_ms python tools/prof_build.py --iters 7 > /dev/null 2>&1
