# GPU tests, full re-tune (tools/tune_r01b.sh) into a fresh wisdom dir, bench, launch list, ncu of the top kernels.
set -x
OUT=${OUT:-gpurun_out/r7}
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest.txt 2>&1; rc=$?; echo "pytest rc=$rc"; tail -15 $OUT/pytest.txt
[ $rc = 0 ] || exit $rc
OUT=$OUT bash tools/tune_r01b.sh > $OUT/tune_log.txt 2>&1
grep -c best_config $OUT/tune_log.txt
timeout 900 python bench.py --wisdom $OUT/wisdom > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err; head -c 1200 $OUT/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --wisdom $OUT/wisdom --steps 3 --warmup 3 --e2e-steps 0 --no-suite --no-cpu-baseline > $OUT/bench_under_ncu.json 2>&1
P="python tools/profile_kernel.py --wisdom $OUT/wisdom --config wisdom --launches 2"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diff_uvw -s 1 -c 1 -o $OUT/diff_fp32_1024 $P --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advec_u -s 1 -c 1 -o $OUT/advec_fp32_512 $P --kernel advec_u --precision fp32 --grid 512,512,512 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advec_u -s 1 -c 1 -o $OUT/advec_fp64_512 $P --kernel advec_u --precision fp64 --grid 512,512,512 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diff_uvw -s 1 -c 1 -o $OUT/diff_fp64_512 $P --kernel diff_uvw --precision fp64 --grid 512,512,512 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advec_u -s 1 -c 1 -o $OUT/advec_fp32_256 $P --kernel advec_u --precision fp32 --grid 256,256,256 2>&1 | tail -1
