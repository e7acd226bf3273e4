# balanced y split probe for advec_u fp32 256^3 (config 2)
P="python tools/ysplit_probe.py --kernel advec_u --precision fp32 --grid 256,256,256 --json-out gpurun_out/r02d_ysplit.jsonl"
C=""
for c in '{}' '{"ysplit":18}' \
  '{"block_y":8,"tile_y":1,"zchunk":128,"depth":4}' '{"block_y":8,"tile_y":1,"zchunk":128,"depth":4,"ysplit":37}' \
  '{"block_y":8,"tile_y":1,"zchunk":128,"depth":6,"ysplit":37}' '{"block_y":8,"tile_y":1,"zchunk":128,"depth":2,"ysplit":37}' \
  '{"block_y":4,"tile_y":2,"zchunk":128,"depth":4,"ysplit":37}' '{"block_y":4,"tile_y":2,"zchunk":128,"depth":6,"ysplit":37}' \
  '{"block_y":4,"tile_y":1,"zchunk":128,"depth":3,"ysplit":74}' '{"block_y":4,"tile_y":1,"zchunk":128,"depth":5,"ysplit":74}' \
  '{"block_y":4,"tile_y":1,"zchunk":64,"depth":2,"ysplit":74}' '{"block_y":8,"tile_y":1,"zchunk":64,"depth":2,"ysplit":37}' \
  '{"block_y":8,"tile_y":1,"zchunk":64,"depth":3,"ysplit":37}' \
  '{"block_y":4,"tile_y":1,"tile_x":2,"block_x":64,"zchunk":128,"depth":4,"ysplit":74}' \
  '{"block_y":2,"tile_y":2,"zchunk":128,"depth":4,"ysplit":74}' '{"block_y":2,"tile_y":2,"zchunk":64,"depth":2,"ysplit":74}' \
  '{"block_y":8,"tile_y":1,"zchunk":32,"depth":2,"ysplit":37}' '{"block_y":4,"tile_y":1,"zchunk":32,"depth":2,"ysplit":74}'; do
  C="$C --case $c"
done
timeout 900 $P $C > gpurun_out/r02d_probe.log 2>&1
echo probe rc $?
