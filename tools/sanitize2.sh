# compute-sanitizer over this session's changed paths: evisc_smag TMA (per-level
# factors by warp shuffle) in both precisions, and the CUDA-graph tests.
OUT=${OUT:-gpurun_out/san2}
mkdir -p $OUT
P="python tools/profile_kernel.py --launches 1 --config wisdom"
run() {  # tool kernel precision grid
  timeout 900 compute-sanitizer --tool $1 --print-limit 20 $P --kernel $2 --precision $3 --grid $4 > $OUT/$1_$2_$3.txt 2>&1
  echo "$1 $2 $3 $4 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/$1_$2_$3.txt | tr '\n' ' ')"
}
for tool in memcheck racecheck synccheck; do
  run $tool evisc_smag fp32 150,70,45
  run $tool evisc_smag fp64 90,50,45
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_graph.py -q -x > $OUT/memcheck_graph.txt 2>&1
echo "memcheck graph tests rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/memcheck_graph.txt | tr '\n' ' ')"
