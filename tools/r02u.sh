# r02u: fused halo after the per-field-set detach fix — GPU tests (incl. a shared exchanger), both bench halo modes
timeout 1200 python -m pytest tests/test_gpu_slab.py tests/test_gpu_multiproc.py -q -p no:cacheprovider -rA \
  > gpurun_out/r02u_pytest.txt 2>&1
echo pytest rc $?
for h in fused exchange; do
KL_DEVICE_ORDINAL=0 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-suite --e2e-steps 1 --halo $h \
  > gpurun_out/r02u_bench2_$h.json 2> gpurun_out/r02u_bench2_$h.err
echo bench2 $h rc $?
done
