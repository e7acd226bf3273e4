# tests -> tuning -> bench in one box session.  OUT=gpurun_out/<tag>
set -x
OUT=${OUT:-gpurun_out/round}
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest.txt 2>&1; rc=$?
tail -5 $OUT/pytest.txt
[ $rc = 0 ] || exit $rc
OUT=$OUT/tune timeout 3000 bash tools/tune_all.sh > $OUT/tune_log.txt 2>&1
tail -3 $OUT/tune_log.txt
timeout 900 python bench.py --wisdom $OUT/tune/wisdom > $OUT/bench.json 2> $OUT/bench.err
tail -2 $OUT/bench.err; head -c 1500 $OUT/bench.json
