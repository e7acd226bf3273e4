# r02i: head-to-head rebase of advec_u fp32 256^3 (ysplit session vs current record), then GPU tests touched since r02b
python tools/rebase_wisdom.py --kernel advec_u --precision fp32 --grid 256,256,256 \
  --sessions profiles/sessions_r02/advec_u_fp32_256x256x256.exhaustive.tma.restricted.seed0.klsession --top 8 --rounds 5 \
  --json-out gpurun_out/r02i_rebase.jsonl > gpurun_out/r02i_rebase256.log 2>&1
echo rebase256 rc $?
cp wisdom/advec_u_fp32-*.wisdom gpurun_out/
timeout 900 python -m pytest tests/test_gpu_stencils.py tests/test_gpu_graph.py tests/test_gpu_capture_tune.py tests/test_gpu_bench_parity.py -q -p no:cacheprovider > gpurun_out/r02i_pytest.txt 2>&1
echo pytest rc $?
