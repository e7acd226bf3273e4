# r02x: fused halo for advec_u as well — GPU tests (virtual ranks + IPC processes, both kernels), per-rank probe
timeout 1500 python -m pytest tests/test_gpu_slab.py tests/test_gpu_multiproc.py -q -p no:cacheprovider -rA -k "fused" \
  > gpurun_out/r02x_pytest.txt 2>&1
echo pytest rc $?
timeout 1200 python tools/fused_halo_probe.py --kernel advec_u --precision fp32 --grid 1024,1024,1024 --ranks 2,4,8 \
  --json-out gpurun_out/r02x_fused.jsonl > gpurun_out/r02x_fused.log 2>&1
echo probe rc $?
