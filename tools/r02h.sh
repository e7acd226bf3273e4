# r02h: head-to-head rebase of advec_u fp32 256^3 (ysplit session vs current record); ysplit tuning at 128^3;
# step_host copy-stream tests; e2e with 1/2/3 copy streams per direction
python tools/rebase_wisdom.py --kernel advec_u --precision fp32 --grid 256,256,256 \
  --sessions gpurun_out/r02g_sessions/*.klsession --top 8 --rounds 5 --json-out gpurun_out/r02h_rebase.jsonl > gpurun_out/r02h_rebase256.log 2>&1
echo rebase256 rc $?
FOC='unravel == "XYZ" && min_blocks == 1 && (zchunk == 32 || zchunk == 64 || zchunk == 128) && depth <= 2 && block_x * tile_x >= 32 && ysplit > 0'
timeout 1500 python -m paper_2303_12374_b200.autotune --kernel advec_u --precision fp32 --grid 128,128,128 \
  --family TMA --strategy exhaustive --budget-evals 2000 --budget-seconds 1400 --restrict "$FOC" \
  --wisdom gpurun_out/r02h_scratch_wisdom --sessions gpurun_out/r02h_sessions --json-out gpurun_out/r02h_tune.jsonl > gpurun_out/r02h_tune128.log 2>&1
echo tune128 rc $?
python tools/rebase_wisdom.py --kernel advec_u --precision fp32 --grid 128,128,128 \
  --sessions gpurun_out/r02h_sessions/*.klsession --top 8 --rounds 5 --json-out gpurun_out/r02h_rebase.jsonl > gpurun_out/r02h_rebase128.log 2>&1
echo rebase128 rc $?
cp wisdom/advec_u_fp32-*.wisdom gpurun_out/
timeout 600 python -m pytest tests/test_gpu_slab.py -q -p no:cacheprovider > gpurun_out/r02h_slab.txt 2>&1
echo slab rc $?
for n in 1 2 3; do
  timeout 400 python bench.py --no-suite --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 3 --e2e-streams $n > gpurun_out/r02h_e2e_s$n.json 2>/dev/null
  echo e2e $n rc $?
done
