# late round-2 evidence run on one box: GPU tests, smoke, default bench, reference arm, 2-rank bench, dispatch,
# and memcheck of the rk3_uvw vector path on ragged grids
T=${1:-r04j}
bash tools/r02_final.sh $T
timeout 900 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python -m pytest tests/test_gpu_family.py -q -x -k "rk3_pass or rk3_vector" \
  > gpurun_out/${T}_memcheck_rk3.txt 2>&1
echo "memcheck rk3 rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/${T}_memcheck_rk3.txt | tr '\n' ' ')"
