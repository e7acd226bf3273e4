# r03d: evisc_smag fp32 aligned x-edge sharing (-D KL_XSHARE=2 on xshare = 0 layouts) vs no sharing and the helper record
X='"defines": {"KL_XSHARE": 2}'
cases=(--case '{}')
for c in '{"block_x": 128, "block_y": 2, "tile_y": 4, "zchunk": 64, "depth": 2, "xshare": 0' \
         '{"block_x": 64, "block_y": 4, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0' \
         '{"block_x": 64, "block_y": 2, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0' \
         '{"block_x": 32, "block_y": 4, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0' \
         '{"block_x": 32, "block_y": 8, "tile_y": 4, "zchunk": 32, "depth": 2, "xshare": 0'; do
  cases+=(--case "$c}" --case "$c, $X}")
done
for p in fp32 fp64; do
timeout 1200 python tools/ysplit_probe.py --kernel evisc_smag --precision $p --grid 512,512,512 --reps 21 "${cases[@]}" \
  --json-out gpurun_out/r03d_xalign.jsonl > gpurun_out/r03d_$p.log 2>&1
echo probe $p rc $?
done
