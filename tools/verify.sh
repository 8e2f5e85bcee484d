# GPU verification round: parity tests + per-kernel times of the C2 build (+ optional extra command)
make all >/dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/${TAG}_tests.log
timeout 300 python tools/kernel_times.py --ns 1000000 > gpurun_out/${TAG}_kt.log 2>&1
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
