# config 2: where the skeleton's extra DRAM reads come from (ncu DRAM bytes of KL_SKEL=3 under tiling changes)
OUT=gpurun_out/r04e; mkdir -p $OUT
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
i=0
for cfg in '{}' '{"zchunk": 128}' '{"zchunk": 256, "ysplit": 0}' '{"block_x": 32, "block_y": 2, "ysplit": 0}' '{"block_x": 16, "block_y": 8, "tile_y": 1, "ysplit": 0}'; do
  for v in KL_SKEL=3 KL_SKEL=1 ""; do
    timeout 300 ncu --metrics $M --clock-control none -k regex:advec_u -c 4 --csv --log-file $OUT/ncu_$i.csv \
      python tools/variant_probe.py --variant "$v" --config "$cfg" --rounds 1 --reps 1 --no-check > $OUT/probe_$i.json 2> $OUT/probe_$i.err
    echo "$i|$cfg|$v" >> $OUT/index.txt
    i=$((i+1))
  done
done
