# headline record vs two runners-up under the bench loop on the 16-byte pitch; w_a / w_b were temporary
# copies of wisdom/ with the 1024^3 diff_uvw fp32 record replaced (64x2/2x4/zchunk 128, 32x4/4x2/zchunk 128)
OUT=gpurun_out/r05q; mkdir -p $OUT
for i in 1 2 3; do
  for w in wisdom w_a w_b; do
    timeout 600 python bench.py --steps 20 --warmup 5 --no-suite --no-cpu-baseline --e2e-steps 1 --wisdom $w >> $OUT/bench_$w.jsonl 2>> $OUT/err.txt
  done
done
echo done
