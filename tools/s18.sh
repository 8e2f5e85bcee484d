make all >/dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "u8_match" 2>&1 | tail -3 > gpurun_out/s18_tests.log
timeout 300 python tools/join_compare.py --shape sift --opts 0,5,6,0 > gpurun_out/s18_cmp.log 2>&1
timeout 1200 python tools/configs_run.py c5 --iters 7,10,13,16 > gpurun_out/s18_c5.log 2>&1
timeout 1200 python tools/configs_run.py c4 --iters 7,10,13 --merge-iters 8 > gpurun_out/s18_c4.log 2>&1
timeout 900 python tools/configs_run.py c3 --iters 10,14 > gpurun_out/s18_c3.log 2>&1
