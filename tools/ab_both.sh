# A/B of compile-time variants (VARS, ';'-separated) on a C2 build (kernel
# times, twice) and a DEEP-shaped 20M build generated on the GPU (once).
kt() { timeout 300 python tools/kernel_times.py --ns 1000000 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_build"], " ".join("%s=%.3f" % (n, k[n]["ms_per_build"]) for n in ("k_init","k_join","k_merge_sample","k_rev_select","k_rev_scatter") if n in k))'; }
IFS=';' read -ra VV <<< "$VARS"
for v in "${VV[@]}"; do
  make clean >/dev/null; make all NVEXTRA="$v" >/dev/null 2>&1 || { echo "[$v] build fail"; continue; }
  echo "[$v] C2: $(kt)"; echo "[$v] C2: $(kt)"
  echo "[$v] DEEP: $(timeout 600 python tools/deep_kt.py --n ${DEEP_N:-20000000} 2>&1 | tail -1)"
done
make clean >/dev/null; make all >/dev/null
