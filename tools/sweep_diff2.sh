# diff_uvw TMA column tiles (tile_x consecutive columns) x block shapes, XYZ order, 1024^3 fp32 + 512^3 fp64
set -x
OUT=${OUT:-gpurun_out/sweep2}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_stencils.py -q -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"; tail -15 $OUT/pytest.txt
B='{"staging":"TMA","block_x":64,"block_y":1,"tile_y":4,"unravel":"XYZ","depth":1,"zchunk":64,"min_blocks":1,"contiguous_x":false}'
for prec_grid in fp32:1024,1024,1024 fp64:512,512,512; do
  p=${prec_grid%%:*}; g=${prec_grid##*:}
  S="python tools/sweep.py --kernel diff_uvw --precision $p --grid $g --base $B --json-out $OUT/diff_$p.jsonl"
  for bt in 64:1:false 128:1:false 32:2:true 64:2:true 16:4:true 32:4:true; do
    bx=$(echo $bt | cut -d: -f1); tx=$(echo $bt | cut -d: -f2); cx=$(echo $bt | cut -d: -f3)
    timeout 600 $S --set block_x=$bx --set tile_x=$tx --set contiguous_x=$cx --vary block_y=1,2,4 --vary tile_y=2,4 --vary depth=1,2
  done
done
