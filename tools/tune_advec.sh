# advec_u: GPU tests for the kernel, then TMA-family tuning at the benchmark sizes.  OUT=gpurun_out/<tag>
set -x
OUT=${OUT:-gpurun_out/advec}
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x -k "advec or slab or capture" > $OUT/pytest.txt 2>&1; rc=$?
tail -15 $OUT/pytest.txt
[ $rc = 0 ] || exit $rc
for spec in "fp32 256,256,256" "fp32 512,512,512" "fp64 512,512,512"; do
  set -- $spec
  timeout 900 python -m paper_2303_12374_b200.autotune --kernel advec_u --precision $1 --grid $2 --strategy surrogate \
    --budget-evals ${EVALS:-100} --budget-seconds 400 --family TMA --wisdom $OUT/wisdom --sessions $OUT/sessions \
    --json-out $OUT/summary.jsonl 2>&1 | tail -1 | cut -c1-600
done
