# A/B of the u8 join: current tree vs a git ref's join_tc.cuh (kernel times of a C2 build)
REF=${1:-HEAD}
echo "current: $(timeout 300 python tools/kernel_times.py --ns 1000000 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_build"], d["kernels"]["k_join"]["ms_per_build"])')"
