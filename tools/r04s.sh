# config 2: the stencil's z-march traversal without its ring (march4) vs the linear elementwise sweep (stream4)
OUT=gpurun_out/r04s; mkdir -p $OUT
timeout 300 python tools/floor_probe.py > $OUT/floor_probe.json 2> $OUT/floor_probe.err; echo rc $?
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"march4|stream4|advec" \
  --csv --log-file $OUT/ncu.csv python tools/floor_probe.py --reps 2 > /dev/null 2> $OUT/ncu.err; echo ncu rc $?
