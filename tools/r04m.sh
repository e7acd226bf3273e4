# GPU suite at HEAD (full-volume bench parity, rk3 vector path tests) + memcheck of the rk3 vector/scalar paths
OUT=gpurun_out/r04m; mkdir -p $OUT
export KL_PARITY_LOG=$OUT/parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA --durations=15 > $OUT/pytest.txt 2>&1
echo pytest rc $?
timeout 900 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python -m pytest tests/test_gpu_family.py -q -x -k "rk3_pass or rk3_vector" \
  > $OUT/memcheck_rk3.txt 2>&1
echo "memcheck rk3 rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/memcheck_rk3.txt | tr '\n' ' ')"
