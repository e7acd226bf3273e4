set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
python tools/dbg_advec2.py 256 2>&1 | tail -8
OUT=gpurun_out/tune3
mkdir -p $OUT
tune() {
  for fam in DIRECT:$4 ZMARCH:$5 TMA:$6; do
    f=${fam%%:*}; n=${fam##*:}
    [ "$n" = "0" ] && continue
    timeout 900 python -m paper_2303_12374_b200.autotune --kernel $1 --precision $2 --grid $3 --strategy random \
      --budget-evals $n --budget-seconds 300 --family $f --wisdom $OUT/wisdom --sessions $OUT/sessions \
      --json-out $OUT/summary.jsonl 2>&1 | tail -1 | cut -c1-300
  done
}
tune advec_u fp32 256,256,256 40 20 100
tune advec_u fp64 512,512,512 30 20 80
tune advec_u fp32 512,512,512 20 10 60
