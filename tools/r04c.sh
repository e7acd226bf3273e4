# config 2 (advec_u fp32 256^3): L2 eviction-priority variants and skeleton levels — times + DRAM bytes
OUT=gpurun_out/r04c; mkdir -p $OUT
timeout 300 python tools/floor_probe.py > $OUT/floor_probe.json 2> $OUT/floor_probe.err; echo floor rc $?

V="--variant KL_L2HINT=0 --variant KL_L2HINT=1 --variant KL_L2HINT=3 --variant KL_L2HINT=8 --variant KL_L2HINT=9 --variant KL_L2HINT=11 --variant KL_L2HINT=15 --variant KL_L2HINT=4"
timeout 600 python tools/variant_probe.py $V --rounds 5 --json-out $OUT/hints.jsonl > /dev/null 2> $OUT/hints.err
echo hints rc $?
S="--variant KL_SKEL=1 --variant KL_SKEL=2 --variant KL_SKEL=3 --variant KL_SKEL=1,KL_L2HINT=9"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:advec_u --csv --log-file $OUT/ncu_variants.csv \
  python tools/variant_probe.py $V $S --rounds 1 --reps 1 --no-check > /dev/null 2> $OUT/ncu.err
echo ncu rc $?
