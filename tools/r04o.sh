# full-volume parity of every benchmarked kernel incl. the §8f family and the unfused rk3 pass at 512^3
OUT=gpurun_out/r04o; mkdir -p $OUT
export KL_PARITY_LOG=$OUT/parity.jsonl
timeout 1800 python -m pytest tests/test_gpu_bench_parity.py -q -p no:cacheprovider -rA --durations=30 > $OUT/pytest.txt 2>&1
echo rc $?
