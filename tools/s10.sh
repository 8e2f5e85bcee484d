make all >/dev/null
timeout 300 python tools/join_compare.py --shape deep > gpurun_out/s10_cmp.log 2>&1
timeout 300 python tools/join_compare.py --shape c1 --d 16 >> gpurun_out/s10_cmp.log 2>&1
timeout 300 python tools/join_compare.py --shape deep --d 32 >> gpurun_out/s10_cmp.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_join -s 3 -c 1 -o gpurun_out/s10_tcf_deep python tools/join_compare.py --shape deep --opts 0 > /dev/null 2>&1
