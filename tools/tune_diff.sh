# diff_uvw: full GPU tests, TMA-family surrogate tuning at every size the bench / BASELINE configs use,
# keep-best merge with earlier wisdom (BASE), then the bench line.   OUT=gpurun_out/<tag> BASE=<wisdom dir>
set -x
OUT=${OUT:-gpurun_out/diff}
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest.txt 2>&1; rc=$?
tail -5 $OUT/pytest.txt
[ $rc = 0 ] || exit $rc
tune() {  # precision grid evals
  timeout 900 python -m paper_2303_12374_b200.autotune --kernel diff_uvw --precision $1 --grid $2 --strategy surrogate \
    --budget-evals $3 --budget-seconds 400 --family TMA --wisdom $OUT/wisdom --sessions $OUT/sessions \
    --json-out $OUT/summary.jsonl 2>&1 | tail -1 | cut -c1-400
}
tune fp32 1024,1024,1024 120
tune fp32 1024,1024,512 60
tune fp32 1024,1024,256 60
tune fp32 1024,1024,128 60
tune fp32 1024,1024,1 30
tune fp32 1024,1024,64 40
tune fp32 512,512,512 60
tune fp64 512,512,512 80
tune fp64 64,64,64 60
mkdir -p $OUT/merged
for f in $OUT/wisdom/*.wisdom; do
  b=$(basename $f)
  if [ -n "$BASE" ] && [ -f $BASE/$b ]; then python -m paper_2303_12374_b200.cli wisdom merge $OUT/merged/$b $f $BASE/$b; else cp $f $OUT/merged/$b; fi
done
for f in ${EXTRA:-}; do cp $f $OUT/merged/; done
timeout 900 python bench.py --wisdom $OUT/merged > $OUT/bench.json 2> $OUT/bench.err
tail -2 $OUT/bench.err; head -c 600 $OUT/bench.json
