# What the driver runs at round end, timed: smoke, default bench, reference arm.
set -x
OUT=${OUT:-gpurun_out/final}
mkdir -p $OUT
t0=$(date +%s); python __graft_entry__.py smoke > $OUT/smoke.txt 2> $OUT/smoke.err; echo "smoke rc=$? $(( $(date +%s) - t0 )) s"; tail -3 $OUT/smoke.txt
t0=$(date +%s); python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$? $(( $(date +%s) - t0 )) s"; tail -2 $OUT/bench.err; head -c 300 $OUT/bench.json
t0=$(date +%s); python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$? $(( $(date +%s) - t0 )) s"; tail -2 $OUT/bench_ref.err; cat $OUT/bench_ref.json
