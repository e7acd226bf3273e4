# tuning convergence on B200: random vs surrogate (the reference's Bayesian-style strategy) over the TMA family,
# 75 s per session, the paper's eight scenarios
OUT=gpurun_out/r05i; mkdir -p $OUT
for k in advec_u diff_uvw; do for n in 256 512; do for p in fp32 fp64; do for st in random surrogate; do
  timeout 300 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl \
    --kernel $k --precision $p --grid $n,$n,$n --family TMA --strategy $st --budget-evals 100000 --budget-seconds 75 --seed 7 \
    > /dev/null 2>> $OUT/err.txt
done; done; done; done
python tools/convergence.py $OUT/sessions/*.klsession > $OUT/convergence.json
echo rc $?
