# config 2: launch/carveout overheads (floor probe) and ncu durations + DRAM bytes of the floor kernels
OUT=gpurun_out/r04d; mkdir -p $OUT
timeout 300 python tools/floor_probe.py > $OUT/floor_probe.json 2> $OUT/floor_probe.err; echo floor rc $?
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  --clock-control none --csv --log-file $OUT/ncu_floor.csv python tools/floor_probe.py --reps 2 > /dev/null 2> $OUT/ncu.err
echo ncu rc $?
