# float join stage-count variants (compile-time) on DEEP 1M (L2, cosine) and GIST 200k
for v in "-DWS_STG=3 -DWS_STP=3" "-DWS_STG=4 -DWS_STP=4" "-DWS_STG=5 -DWS_STP=2"; do
  make clean >/dev/null; make all NVEXTRA="$v" >/dev/null 2>&1 || { echo "$v build fail"; continue; }
  echo "== $v"
  timeout 300 python tools/join_compare.py --shape deep --n 1000000 --opts 2,3 | cut -c1-60
  timeout 300 python tools/join_compare.py --shape deep --n 1000000 --opts 2,3 --metric cosine | cut -c1-60
  timeout 300 python tools/join_compare.py --shape gist --n 200000 --opts 2,3 | cut -c1-60
done
make clean >/dev/null; make all >/dev/null
