# After the advec_u fp32 packed kernel: GPU tests, re-tune advec_u fp32, bench, launch list, ncu of the top kernels.
set -x
OUT=${OUT:-gpurun_out/r6}
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest.txt
cp -r wisdom $OUT/wisdom
R='unravel == "XYZ" && min_blocks == 1 && (zchunk == 32 || zchunk == 64 || zchunk == 128) && depth <= 2 && block_x * tile_x >= 32'
at() { timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl "$@" 2>&1 | tail -1 | cut -c1-300; }
for g in 256,256,256 512,512,512; do
  at --kernel advec_u --precision fp32 --grid $g --family TMA --strategy exhaustive --budget-evals 2000 --budget-seconds 1500 --restrict "$R"
  at --kernel advec_u --precision fp32 --grid $g --family TMA --strategy surrogate --budget-evals 60 --budget-seconds 600 --seed 1
  at --kernel advec_u --precision fp32 --grid $g --family DIRECT --strategy random --budget-evals 20 --budget-seconds 300
done
timeout 900 python bench.py --wisdom $OUT/wisdom > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err; head -c 1500 $OUT/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --wisdom $OUT/wisdom --steps 3 --warmup 3 --e2e-steps 0 --no-suite --no-cpu-baseline > $OUT/bench_under_ncu.json 2>&1
P="python tools/profile_kernel.py --wisdom $OUT/wisdom --config wisdom --launches 2"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diff_uvw -s 1 -c 1 -o $OUT/diff_fp32_1024 $P --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advec_u -s 1 -c 1 -o $OUT/advec_fp32_512 $P --kernel advec_u --precision fp32 --grid 512,512,512 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advec_u -s 1 -c 1 -o $OUT/advec_fp64_512 $P --kernel advec_u --precision fp64 --grid 512,512,512 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diff_uvw -s 1 -c 1 -o $OUT/diff_fp64_512 $P --kernel diff_uvw --precision fp64 --grid 512,512,512 2>&1 | tail -2
