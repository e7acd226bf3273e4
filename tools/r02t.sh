# r02t: fused z-slab halo (diff_uvw_peer) — GPU tests (virtual ranks, IPC processes), per-rank step of the
# middle rank at N = 2/4/8 vs the exchange variant (tools/fused_halo_probe.py), bench with 2 ranks on one GPU
timeout 1200 python -m pytest tests/test_gpu_slab.py tests/test_gpu_multiproc.py -q -p no:cacheprovider -rA -k "fused" \
  > gpurun_out/r02t_pytest.txt 2>&1
echo pytest rc $?
timeout 1200 python tools/fused_halo_probe.py --precision fp32 --grid 1024,1024,1024 --ranks 2,4,8 \
  --json-out gpurun_out/r02t_fused.jsonl > gpurun_out/r02t_fused.log 2>&1
echo probe rc $?
for h in exchange fused; do
KL_DEVICE_ORDINAL=0 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-suite --e2e-steps 1 --halo $h \
  > gpurun_out/r02t_bench2_$h.json 2> gpurun_out/r02t_bench2_$h.err
echo bench2 $h rc $?
done
