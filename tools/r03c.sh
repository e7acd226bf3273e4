# r03c: evisc_smag fp32 row-pair march with the register cap that keeps the scalar march's occupancy (min_blocks)
R='"defines": {"KL_ROWPACK": 1}'
cases=(--case '{}')
for c in '{"block_x": 128, "block_y": 2, "tile_y": 4, "zchunk": 64, "depth": 2, "xshare": 0' \
         '{"block_x": 128, "block_y": 2, "tile_y": 4, "zchunk": 64, "depth": 2, "xshare": 0, "min_blocks": 3' \
         '{"block_x": 64, "block_y": 4, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0, "min_blocks": 3' \
         '{"block_x": 64, "block_y": 2, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0, "min_blocks": 6' \
         '{"block_x": 32, "block_y": 4, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0, "min_blocks": 6' \
         '{"block_x": 64, "block_y": 4, "tile_y": 4, "zchunk": 64, "depth": 1, "xshare": 0, "min_blocks": 3'; do
  cases+=(--case "$c}" --case "$c, $R}")
done
timeout 1200 python tools/ysplit_probe.py --kernel evisc_smag --precision fp32 --grid 512,512,512 --reps 21 "${cases[@]}" \
  --json-out gpurun_out/r03c_rowpack.jsonl > gpurun_out/r03c.log 2>&1
echo probe rc $?
