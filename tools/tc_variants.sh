# u8 join variants (compile-time switches) timed on the C2 build
for v in "-DTC_EPI_IDLE=0" "-DTC_EPI_IDLE=1 -DWS_IDLE_MIN_NS=32 -DWS_IDLE_MAX_NS=256" "-DTC_EPI_IDLE=1 -DWS_IDLE_MIN_NS=64 -DWS_IDLE_MAX_NS=1024"; do
  make clean >/dev/null; make all NVEXTRA="$v" >/dev/null 2>&1 || { echo build fail; continue; }
  echo "$v: $(timeout 300 python tools/kernel_times.py --ns 1000000 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_build"], d["kernels"]["k_join"]["ms_per_build"])')"
done
