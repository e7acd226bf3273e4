# r02s: fp64 fast square root — precision test, evisc parity, record timing with KL_SQRT64 = 1 (new default) vs 0
timeout 900 python -m pytest tests/test_gpu_fastmath.py tests/test_gpu_family.py -q -p no:cacheprovider -rA -s -k "sqrt or evisc" > gpurun_out/r02s_pytest.txt 2>&1
echo pytest rc $?
timeout 900 python tools/ysplit_probe.py --kernel evisc_smag --precision fp64 --grid 512,512,512 --reps 21 \
  --case '{}' --case '{"defines": {"KL_SQRT64": 0}}' --case '{}' --case '{"defines": {"KL_SQRT64": 0}}' \
  --json-out gpurun_out/r02s_sqrt.jsonl > gpurun_out/r02s_sqrt.log 2>&1
echo probe rc $?
