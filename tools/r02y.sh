# r02y: fused halo, advec_u short last chunk (prologue planes above the slab) — GPU tests
timeout 1500 python -m pytest tests/test_gpu_slab.py tests/test_gpu_multiproc.py -q -p no:cacheprovider -rA -k "fused" \
  > gpurun_out/r02y_pytest.txt 2>&1
echo pytest rc $?
