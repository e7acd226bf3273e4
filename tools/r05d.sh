# headline A/B under the bench's own timed loop: committed wisdom vs the sustained-load winner for 1024^3
OUT=gpurun_out/r05d; mkdir -p $OUT
for i in 1 2 3; do
  for w in wisdom profiles/r05c_wisdom_candidate; do
    tag=$(basename $w)
    timeout 600 python bench.py --steps 20 --warmup 5 --no-suite --no-cpu-baseline --e2e-steps 1 --wisdom $w \
      >> $OUT/bench_$tag.jsonl 2>> $OUT/err.txt
  done
done
echo done
