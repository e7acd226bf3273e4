# GPU validation of the committed state: gpu tests, smoke, bench, launch list, ncu of both tuned kernels.
set -x
OUT=${OUT:-gpurun_out/val}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest.txt
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err; head -c 3000 $OUT/bench.json
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-suite --no-cpu-baseline > $OUT/bench_under_ncu.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diff_uvw -s 1 -c 1 -o $OUT/diff_1024_tuned python tools/profile_kernel.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 --config wisdom --launches 2 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advec_u -s 1 -c 1 -o $OUT/advec_256_tuned python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 256,256,256 --config wisdom --launches 2 2>&1 | tail -3
fi
