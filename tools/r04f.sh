# HBM row pitch: 128-byte vs 16-byte aligned rows for the benchmarked kernels (times, bit-identity, DRAM bytes)
OUT=gpurun_out/r04f; mkdir -p $OUT
timeout 1500 python tools/layout_probe.py --json-out $OUT/layout.jsonl > /dev/null 2> $OUT/layout.err
echo layout rc $?
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"advec_u|diff_uvw" --csv --log-file $OUT/ncu_layout.csv \
  python tools/layout_probe.py --work advec_u:fp32:256 --work diff_uvw:fp32:512 --rounds 1 --reps 1 > /dev/null 2> $OUT/ncu.err
echo ncu rc $?
