# whole-TMA-family surrogate sessions for the weaker 512^3 rows (evisc_smag fp32/fp64, advec_u fp64), then rebase
OUT=gpurun_out/r05o; mkdir -p $OUT
cp -r wisdom $OUT/wisdom
for kp in evisc_smag:fp32 evisc_smag:fp64 advec_u:fp64; do
  k=${kp%:*}; p=${kp#*:}
  timeout 900 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl \
    --kernel $k --precision $p --grid 512,512,512 --family TMA --strategy surrogate --budget-evals 100000 --budget-seconds 480 --seed 13 \
    > /dev/null 2>> $OUT/err.txt
  timeout 900 python tools/rebase_wisdom.py --kernel $k --precision $p --grid 512,512,512 --wisdom $OUT/wisdom \
    --sessions $OUT/sessions/${k}_${p}_512x512x512*.klsession --top 6 --rounds 5 --json-out $OUT/rebase.jsonl 2>&1 | tail -1
done
