make all >/dev/null || exit 1
T=s3c
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_join -s 3 -c 1 -o gpurun_out/${T}_k_join python tools/prof_build.py --iters 7 > gpurun_out/${T}_ncu.log 2>&1
python tools/ncu_report.py gpurun_out/${T}_k_join.ncu-rep "k_join, C2 build (${T})" > gpurun_out/${T}_ncu_k_join.txt 2>&1
timeout 300 python tools/ncu_callsites.py gpurun_out/${T}_k_join.ncu-rep auto 60 >> gpurun_out/${T}_ncu_k_join.txt 2>&1
timeout 300 python tools/ncu_lines.py gpurun_out/${T}_k_join.ncu-rep auto 60 > gpurun_out/${T}_lines_k_join.txt 2>&1
ncu -i gpurun_out/${T}_k_join.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_sass.csv 2>/dev/null
