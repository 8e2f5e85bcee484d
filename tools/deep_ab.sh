for v in "" "-DKNNG_REV_CURSOR=0"; do
  make clean >/dev/null; make all NVEXTRA="$v" >/dev/null 2>&1 || { echo "[$v] build fail"; continue; }
  echo "[$v] $(timeout 600 python tools/deep_kt.py --n 20000000 2>&1 | tail -1)"
done
make clean >/dev/null; make all >/dev/null
