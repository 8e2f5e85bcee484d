# C2 build kernel times (two runs) + the u8 join's parity tests
make all >/dev/null || exit 1
for i in 1 2; do timeout 300 python tools/kernel_times.py --ns 1000000 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_build"], {k: v["ms_per_build"] for k, v in d["kernels"].items() if v["ms_per_build"] > 0.5})'; done
timeout 600 python -m pytest tests -m gpu -x -q -k "u8 or ggm or distributed or c2_full or sift or teacher" 2>&1 | tail -2
