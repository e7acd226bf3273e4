# full-volume oracle parity of the benchmarked kernels (every interior cell, C restatement in z-chunks)
OUT=gpurun_out/r04h; mkdir -p $OUT
nproc > $OUT/nproc.txt; free -g >> $OUT/nproc.txt
export KL_PARITY_LOG=$OUT/parity.jsonl
timeout 1500 python -m pytest tests/test_gpu_bench_parity.py -q -p no:cacheprovider -rA --durations=20 > $OUT/pytest.txt 2>&1
echo rc $?
