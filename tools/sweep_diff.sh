# diff_uvw fp32 1024^3 TMA: tile shape x launch order x depth around the tuned point
set -x
OUT=${OUT:-gpurun_out/sweep}
mkdir -p $OUT
S="python tools/sweep.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 --json-out $OUT/diff.jsonl"
timeout 600 $S --vary unravel=XZY,XYZ,YXZ --vary block_y=1,2,4 --vary depth=1,2 --set min_blocks=1
timeout 600 $S --vary unravel=XZY,XYZ --vary block_y=1,2,4,8 --vary tile_y=2 --vary depth=1,2 --set min_blocks=1
timeout 600 $S --vary unravel=XZY,XYZ --vary block_x=32,128 --vary block_y=1,2,4 --vary depth=1,2 --set min_blocks=1
timeout 600 $S --vary unravel=XYZ --vary block_y=2,4 --vary zchunk=32,128 --vary min_blocks=1,2,3
