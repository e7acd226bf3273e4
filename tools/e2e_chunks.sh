# e2e (host-resident fields streamed over PCIe) vs the number of z-chunks per step.
OUT=${OUT:-gpurun_out/e2ec}
mkdir -p $OUT
for c in 8 16 32 64; do
  timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 3 --e2e-chunks $c --no-suite --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "import json; d=json.load(open('$OUT/bench_$c.json')); e=d['e2e']; print($c, e['value'], e['ms_per_step'], e.get('h2d_d2h_gbs'))"
done
