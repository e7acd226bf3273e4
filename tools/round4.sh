# GPU tests (incl. the §8f family and the fused RK3 kernel), tune the new kernels into a copy of wisdom/,
# bench (suite + family + fusion), B200 report matrices over the committed sessions.
set -x
OUT=${OUT:-gpurun_out/r8}
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest.txt 2>&1; rc=$?; echo "pytest rc=$rc"; tail -15 $OUT/pytest.txt
[ $rc = 0 ] || exit $rc
cp -r wisdom $OUT/wisdom
at() { timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl "$@" 2>&1 | tail -1 | cut -c1-300; }
for p in fp32 fp64; do
  at --kernel diff_uvw_rk3 --precision $p --grid 512,512,512 --family TMA --focused --strategy exhaustive --budget-evals 2000 --budget-seconds 1500
  at --kernel rk3_uvw --precision $p --grid 512,512,512 --strategy random --budget-evals 60 --budget-seconds 300 --seed 3
  for k in advec_v advec_w advec_s diff_c evisc_smag; do
    at --kernel $k --precision $p --grid 512,512,512 --strategy random --budget-evals 60 --budget-seconds 300 --seed 3
  done
done
timeout 1200 python bench.py --wisdom $OUT/wisdom > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err; head -c 600 $OUT/bench.json
S=profiles/sessions_r01c
R="timeout 1200 python -m paper_2303_12374_b200.cli report"
$R matrix --backend cuda $S/diff_uvw_fp32_512x512x512.exhaustive.tma.restricted.seed0.klsession $S/diff_uvw_fp32_1024x1024x128.exhaustive.tma.restricted.seed0.klsession $S/diff_uvw_fp32_1024x1024x256.exhaustive.tma.restricted.seed0.klsession $S/diff_uvw_fp32_1024x1024x512.exhaustive.tma.restricted.seed0.klsession $S/diff_uvw_fp32_1024x1024x1024.exhaustive.tma.restricted.seed0.klsession --out $OUT/matrix_diff_uvw_fp32.csv
$R ppm --matrix $OUT/matrix_diff_uvw_fp32.csv --out $OUT/ppm_diff_uvw_fp32.csv
$R matrix --backend cuda $S/advec_u_fp32_256x256x256.exhaustive.tma.restricted.seed0.klsession $S/advec_u_fp32_512x512x512.exhaustive.tma.restricted.seed0.klsession --out $OUT/matrix_advec_u_fp32.csv
$R ppm --matrix $OUT/matrix_advec_u_fp32.csv --out $OUT/ppm_advec_u_fp32.csv
$R matrix --backend cuda $S/diff_uvw_fp64_64x64x64.exhaustive.tma.restricted.seed0.klsession $S/diff_uvw_fp64_512x512x512.exhaustive.tma.restricted.seed0.klsession --out $OUT/matrix_diff_uvw_fp64.csv
$R ppm --matrix $OUT/matrix_diff_uvw_fp64.csv --out $OUT/ppm_diff_uvw_fp64.csv
$R histogram --backend cuda $S/diff_uvw_fp32_1024x1024x1024.exhaustive.tma.restricted.seed0.klsession --out $OUT/hist_diff_uvw_fp32_1024.csv
$R histogram --backend cuda $S/advec_u_fp64_512x512x512.exhaustive.tma.restricted.seed0.klsession --out $OUT/hist_advec_u_fp64_512.csv
cat $OUT/matrix_*.csv $OUT/ppm_*.csv
