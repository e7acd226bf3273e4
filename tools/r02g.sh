# r02g: PDL trigger-at-exit graph rows; ysplit sub-space tuning of advec_u fp32 256^3 (config 2)
python - > gpurun_out/r02g_graph.json 2> gpurun_out/r02g_graph.err <<'PY'
import json, sys
sys.argv = ["bench.py"]
import bench
from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
ctx = open_device(0)
peak, _ = bench.peaks()
print(json.dumps(bench.graph_measure(ctx, NvrtcCompiler(ctx), bench.ROOT / "wisdom", peak)))
PY
echo graph rc $?
FOC='unravel == "XYZ" && min_blocks == 1 && (zchunk == 32 || zchunk == 64 || zchunk == 128) && depth <= 2 && block_x * tile_x >= 32 && ysplit > 0'
timeout 2400 python -m paper_2303_12374_b200.autotune --kernel advec_u --precision fp32 --grid 256,256,256 \
  --family TMA --strategy exhaustive --budget-evals 2000 --budget-seconds 2200 --restrict "$FOC" \
  --wisdom wisdom --sessions gpurun_out/r02g_sessions --json-out gpurun_out/r02g_tune.jsonl > gpurun_out/r02g_tune.log 2>&1
echo tune rc $?
cp wisdom/advec_u_fp32-*.wisdom gpurun_out/
