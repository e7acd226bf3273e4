# config-5 runtime-selected kernels at shapes without a record: full-volume parity
OUT=gpurun_out/r04p; mkdir -p $OUT
export KL_PARITY_LOG=$OUT/parity.jsonl
timeout 1200 python -m pytest tests/test_gpu_bench_parity.py -q -p no:cacheprovider -rA -k "config5 or 192 or 384 or 768 or 320" > $OUT/pytest.txt 2>&1
echo rc $?
