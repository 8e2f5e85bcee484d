VARS=";-DTC_PMIN=1;;-DTC_PMIN=1" bash tools/ab.sh > gpurun_out/s3p_ab.log 2>&1
make all >/dev/null
timeout 600 ncu --set full --clock-control none -k regex:k_merge_sample -s 12 -c 1 -o gpurun_out/s3p_merge_deep20m python tools/deep_kt.py --n 20000000 > gpurun_out/s3p_ncu.log 2>&1
python tools/ncu_report.py gpurun_out/s3p_merge_deep20m.ncu-rep "k_merge_sample, DEEP-shaped 20M build (s3p)" > gpurun_out/s3p_ncu_merge_deep20m.txt 2>&1
timeout 300 python tools/ncu_callsites.py gpurun_out/s3p_merge_deep20m.ncu-rep auto 30 >> gpurun_out/s3p_ncu_merge_deep20m.txt 2>&1
rm -f gpurun_out/s3p_merge_deep20m.ncu-rep
