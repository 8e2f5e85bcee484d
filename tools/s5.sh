make all >/dev/null
KNNG_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --rows 500000 --steps 2 --warmup 3 > gpurun_out/s5_bench2.json 2> gpurun_out/s5_bench2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_launches.csv python tools/prof_build.py --iters 7 > /dev/null 2>&1
for K in k_merge_sample k_rev_select k_rev_scatter; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/s5_$K python tools/prof_build.py --iters 7 > /dev/null 2>&1
done
ls gpurun_out
