# Tune every problem size the benchmark and the BASELINE configs use; writes wisdom + sessions.
set -x
OUT=${OUT:-gpurun_out/tune}
mkdir -p $OUT
tune() {  # kernel precision grid evals_direct evals_zmarch evals_tma
  for fam in DIRECT:$4 ZMARCH:$5 TMA:$6; do
    f=${fam%%:*}; n=${fam##*:}
    [ "$n" = "0" ] && continue
    timeout 900 python -m paper_2303_12374_b200.autotune --kernel $1 --precision $2 --grid $3 --strategy random \
      --budget-evals $n --budget-seconds 300 --family $f --wisdom $OUT/wisdom --sessions $OUT/sessions \
      --json-out $OUT/summary.jsonl 2>&1 | tail -1 | cut -c1-400
  done
}
tune diff_uvw fp32 1024,1024,1024 30 20 80
tune diff_uvw fp32 1024,1024,512 20 10 60
tune diff_uvw fp32 1024,1024,256 20 10 60
tune diff_uvw fp32 1024,1024,128 20 10 60
tune diff_uvw fp32 1024,1024,1 40 0 30
tune advec_u fp32 256,256,256 40 20 80
tune advec_u fp64 512,512,512 30 20 60
tune diff_uvw fp64 512,512,512 30 20 60
tune diff_uvw fp64 64,64,64 40 20 60
tune advec_u fp32 512,512,512 20 10 40
tune diff_uvw fp32 512,512,512 20 10 40
