# What the driver runs at round end, timed: smoke, default bench, reference arm.
set -x
OUT=${OUT:-gpurun_out/final}
mkdir -p $OUT
/usr/bin/time -v python __graft_entry__.py smoke > $OUT/smoke.txt 2> $OUT/smoke.err; echo "smoke rc=$?"; tail -3 $OUT/smoke.txt; grep Elapsed $OUT/smoke.err
/usr/bin/time -v python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; grep Elapsed $OUT/bench.err; head -c 300 $OUT/bench.json
/usr/bin/time -v python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; grep Elapsed $OUT/bench_ref.err; cat $OUT/bench_ref.json
