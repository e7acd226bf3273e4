# packed plane march: family GPU tests, retune diff_c / evisc_smag, bench, ncu of evisc_smag / diff_c.
set -x
OUT=${OUT:-gpurun_out/r11}
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_family.py tests/test_gpu_capture_tune.py -q -x > $OUT/pytest.txt 2>&1; rc=$?; echo "pytest rc=$rc"; tail -15 $OUT/pytest.txt
[ $rc = 0 ] || exit $rc
cp -r wisdom $OUT/wisdom
at() { timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl "$@" 2>&1 | tail -1 | cut -c1-300; }
for p in fp32 fp64; do
  for k in diff_c evisc_smag; do
    at --kernel $k --precision $p --grid 512,512,512 --family TMA --focused --strategy exhaustive --budget-evals 2000 --budget-seconds 1500
    at --kernel $k --precision $p --grid 512,512,512 --family DIRECT --strategy random --budget-evals 40 --budget-seconds 300 --seed 3
  done
done
timeout 1200 python bench.py --wisdom $OUT/wisdom > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err; head -c 400 $OUT/bench.json
P="python tools/profile_kernel.py --wisdom $OUT/wisdom --config wisdom --launches 2"
for k in diff_c evisc_smag; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $OUT/${k}_fp32_512 $P --kernel $k --precision fp32 --grid 512,512,512 2>&1 | tail -1
done
