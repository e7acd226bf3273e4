set -x
mkdir -p gpurun_out/e4
python -m pytest tests -q -m gpu -x 2>&1 | tail -8
for spec in "diff_uvw fp32 512,512,512" "diff_uvw fp64 512,512,512" "advec_u fp32 512,512,512" "advec_u fp64 512,512,512"; do
  set -- $spec
  timeout 900 python -m paper_2303_12374_b200.autotune --kernel $1 --precision $2 --grid $3 --strategy random --budget-evals 80 --budget-seconds 400 --wisdom gpurun_out/e4/wisdom --sessions gpurun_out/e4/sessions --json-out gpurun_out/e4/summary.jsonl --family TMA 2>&1 | tail -2
done
CFG='{"staging":"TMA","block_x":32,"block_y":8,"tile_x":1,"tile_y":2,"zchunk":32,"block_z":1,"tile_z":1,"depth":2}'
timeout 300 ncu --set full --clock-control none --import-source on -k regex:diff_uvw -s 1 -c 1 -o gpurun_out/e4/diff_tma python tools/profile_kernel.py --kernel diff_uvw --precision fp32 --grid 512,512,512 --config "$CFG" --launches 2 2>&1 | tail -2
timeout 300 ncu --set full --clock-control none --import-source on -k regex:advec_u -s 1 -c 1 -o gpurun_out/e4/advec_tma python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 512,512,512 --config "$CFG" --launches 2 2>&1 | tail -2
