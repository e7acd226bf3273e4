set -x
OUT=gpurun_out/tune4
mkdir -p $OUT
for g in 1024,1024,1024 1024,1024,512 1024,1024,256 1024,1024,128; do
  timeout 1200 python -m paper_2303_12374_b200.autotune --kernel diff_uvw --precision fp32 --grid $g --strategy surrogate \
      --budget-evals 120 --budget-seconds 600 --family TMA --wisdom $OUT/wisdom --sessions $OUT/sessions \
      --json-out $OUT/summary.jsonl --seed 7 2>&1 | tail -1 | cut -c1-300
done
timeout 1200 python -m paper_2303_12374_b200.autotune --kernel diff_uvw --precision fp64 --grid 512,512,512 --strategy surrogate \
      --budget-evals 80 --budget-seconds 600 --family TMA --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl --seed 7 2>&1 | tail -1 | cut -c1-300
timeout 3000 python -m paper_2303_12374_b200.portability --out gpurun_out/portability.json --evals 40 2>&1 | tail -30
