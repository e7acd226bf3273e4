# bench A/B: 128-byte vs 16-byte row pitch for the headline workload (device value and e2e)
OUT=gpurun_out/r05j; mkdir -p $OUT
for i in 1 2 3; do
  for a in 128 16; do
    timeout 900 python bench.py --steps 20 --warmup 5 --no-suite --no-cpu-baseline --e2e-steps 3 --row-align $a \
      >> $OUT/bench_align$a.jsonl 2>> $OUT/err.txt
  done
done
echo done
