# ncu --set full captures of the non-join kernels of one C2 build (tag = $1)
T=${1:-x}
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_merge_sample -s 4 -c 1 -o gpurun_out/merge_$T python tools/prof_build.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rev_select -s 3 -c 1 -o gpurun_out/revsel_$T python tools/prof_build.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rev_scatter -s 3 -c 1 -o gpurun_out/revsc_$T python tools/prof_build.py > /dev/null 2>&1
ls gpurun_out
