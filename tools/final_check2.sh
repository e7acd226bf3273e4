# Round-end validation of the committed state: GPU suite, smoke, default bench, reference arm.
OUT=${OUT:-gpurun_out/final2}
mkdir -p $OUT
t0=$(date +%s); timeout 1800 python -m pytest tests -q -m gpu -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$? $(( $(date +%s) - t0 )) s"; tail -3 $OUT/pytest.txt
OUT=$OUT bash tools/final_check.sh 2>&1 | grep -E "rc=|smoke|value" | cut -c1-300
