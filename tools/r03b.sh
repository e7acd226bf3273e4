# r03b: evisc_smag fp32 row-pair packed march (KL_ROWPACK=1) on aligned (xshare = 0) layouts vs the xshare record
C='{"block_x": 128, "block_y": 2, "tile_y": 4, "zchunk": 64, "depth": 2, "xshare": 0}'
D='{"block_x": 64, "block_y": 2, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0}'
E='{"block_x": 64, "block_y": 4, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0}'
F='{"block_x": 32, "block_y": 4, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0}'
G='{"block_x": 128, "block_y": 2, "tile_y": 2, "zchunk": 64, "depth": 2, "xshare": 0}'
R='"defines": {"KL_ROWPACK": 1}'
cases=(--case '{}')
for c in "$C" "$D" "$E" "$F" "$G"; do cases+=(--case "$c" --case "${c%\}}, $R}"); done
timeout 1200 python tools/ysplit_probe.py --kernel evisc_smag --precision fp32 --grid 512,512,512 --reps 21 "${cases[@]}" \
  --json-out gpurun_out/r03b_rowpack.jsonl > gpurun_out/r03b.log 2>&1
echo probe rc $?
