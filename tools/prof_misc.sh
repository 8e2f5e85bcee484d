timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_merge_sample -s 4 -c 1 -o gpurun_out/merge_v16 python tools/prof_build.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rev_select -s 3 -c 1 -o gpurun_out/revsel_v16 python tools/prof_build.py > /dev/null 2>&1
ls gpurun_out
