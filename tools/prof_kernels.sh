# ncu --set full captures of the C2 build's main kernels (current build), tag = $1
T=${1:-x}
for K in k_join k_merge_sample k_rev_select k_rev_scatter; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/${T}_$K python tools/prof_build.py --iters 7 > /dev/null 2>&1
done
