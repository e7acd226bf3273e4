# re-tune the headline (diff_uvw fp32 1024^3) and north-star advec_u fp32 512^3 records on one box:
# exhaustive FOCUSED_TMA sessions, then head-to-head rebase against the committed records
OUT=gpurun_out/r04q; mkdir -p $OUT
cp -r wisdom $OUT/wisdom
for kpg in diff_uvw:fp32:1024 advec_u:fp32:512; do
  IFS=: read k p n <<< "$kpg"
  timeout 1800 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl \
    --kernel $k --precision $p --grid $n,$n,$n --family TMA --focused --strategy exhaustive --budget-evals 3000 --budget-seconds 1500 \
    2>&1 | tail -1 | cut -c1-300
  timeout 900 python tools/rebase_wisdom.py --kernel $k --precision $p --grid $n,$n,$n --wisdom $OUT/wisdom \
    --sessions $OUT/sessions/${k}_${p}_${n}x${n}x${n}*.klsession --top 8 --rounds 5 --json-out $OUT/rebase.jsonl 2>&1 | tail -2
done
