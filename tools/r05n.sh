# config 2: long surrogate + random sessions over the WHOLE TMA family at 256^3 fp32 (outside the focused sub-space), then rebase
OUT=gpurun_out/r05n; mkdir -p $OUT
cp -r wisdom $OUT/wisdom
for st in surrogate random; do
  timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl \
    --kernel advec_u --precision fp32 --grid 256,256,256 --family TMA --strategy $st --budget-evals 100000 --budget-seconds 600 --seed 11 \
    > /dev/null 2>> $OUT/err.txt
  echo $st rc $?
done
timeout 900 python tools/rebase_wisdom.py --kernel advec_u --precision fp32 --grid 256,256,256 --wisdom $OUT/wisdom \
  --sessions $OUT/sessions/advec_u_fp32_256x256x256*.klsession --top 8 --rounds 5 --json-out $OUT/rebase.jsonl 2>&1 | tail -2
