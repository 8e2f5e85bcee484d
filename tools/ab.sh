# A/B of compile-time variants on the C2 build's kernel times.
#   REFS="HEAD" (baselines: trees staged here with
#     mkdir -p ab_ref/HEAD && git archive HEAD paper_2103_15386_b200/csrc include | tar -x -C ab_ref/HEAD
#     -- the GPU box gets no .git)
#   VARS=";-DTC_PLANS=8" (NVEXTRA variants of the working tree, ';'-separated)
# Each build is timed twice (kernel_times.py, CUDA events per launch).
kt() { timeout 300 python tools/kernel_times.py --ns 1000000 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(d["ms_per_build"], " ".join("%s=%.3f" % (n, k[n]["ms_per_build"]) for n in ("k_join","k_merge_sample","k_rev_select","k_rev_scatter") if n in k))'; }
for R in $REFS; do
  [ -d ab_ref/$R ] || { echo "no ab_ref/$R"; continue; }
  mkdir -p paper_2103_15386_b200/lib
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC -shared -ldl -Iab_ref/$R/include \
    -o paper_2103_15386_b200/lib/libknng.so ab_ref/$R/paper_2103_15386_b200/csrc/knng_api.cu || continue
  echo "ref $R: $(kt)"; echo "ref $R: $(kt)"
done
IFS=';' read -ra VV <<< "$VARS"
for v in "${VV[@]}"; do
  make clean >/dev/null; make all NVEXTRA="$v" >/dev/null 2>&1 || { echo "[$v] build fail"; continue; }
  echo "[$v]: $(kt)"; echo "[$v]: $(kt)"
done
make clean >/dev/null; make all >/dev/null
