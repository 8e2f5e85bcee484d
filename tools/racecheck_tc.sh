# racecheck of the u8 tensor-core join: the default build,
# whose plan ring is handed off with mbarriers only, and the KNNG_TC_LOCKSTEP
# build, where the planning warp also meets the epilogue warps at a CTA
# barrier per batch (an ordering racecheck models).  Same graphs expected.
OUT=gpurun_out/racecheck
mkdir -p $OUT
make clean >/dev/null; make all >/dev/null || exit 1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_one.py > $OUT/default.txt 2>&1
python tools/sanitize_one.py > $OUT/default_digest.txt 2>&1
make clean >/dev/null; make all NVEXTRA=-DKNNG_TC_LOCKSTEP >/dev/null || exit 1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_one.py > $OUT/lockstep.txt 2>&1
python tools/sanitize_one.py > $OUT/lockstep_digest.txt 2>&1
make clean >/dev/null; make all >/dev/null
for f in default lockstep; do echo "$f: $(grep -c 'Race reported\|hazard' $OUT/$f.txt) hazard lines; $(tail -2 $OUT/$f.txt | tr '\n' ' ')"; cat $OUT/${f}_digest.txt; done
