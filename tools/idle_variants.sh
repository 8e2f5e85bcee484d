# build variants of the idle back-off and time the DEEP float join
for v in "64 1024" "32 512" "128 2048" "256 4096"; do
  set -- $v
  make clean >/dev/null; make all NVEXTRA="-DWS_IDLE_MIN_NS=$1 -DWS_IDLE_MAX_NS=$2" >/dev/null 2>&1 || { echo build fail; continue; }
  echo "idle $1..$2 ns"; timeout 300 python tools/join_compare.py --shape deep --n 1000000 --opts 0
done
