# config 2: plain-load z-march traversal vs chunk length; exhaustive advec_u TMA session at zchunk 8/16 (never enumerated)
OUT=gpurun_out/r04t; mkdir -p $OUT
timeout 300 python tools/floor_probe.py > $OUT/floor_probe.json 2> $OUT/floor_probe.err; echo floor rc $?
cp -r wisdom $OUT/wisdom
R='unravel == "XYZ" && min_blocks == 1 && (zchunk == 8 || zchunk == 16) && depth <= 2 && block_x * tile_x >= 32'
timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl \
  --kernel advec_u --precision fp32 --grid 256,256,256 --family TMA --strategy exhaustive --budget-evals 4000 --budget-seconds 1200 \
  --restrict "$R" 2>&1 | tail -1 | cut -c1-300
timeout 900 python tools/rebase_wisdom.py --kernel advec_u --precision fp32 --grid 256,256,256 --wisdom $OUT/wisdom \
  --sessions $OUT/sessions/advec_u_fp32_256x256x256*.klsession --top 8 --rounds 5 --json-out $OUT/rebase.jsonl 2>&1 | tail -2
