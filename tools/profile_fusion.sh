# ncu of the fused RK3 kernel and its unfused pair (512^3 fp32, wisdom-selected); launch list of a short bench.
OUT=${OUT:-gpurun_out/pf}
mkdir -p $OUT
P="python tools/profile_kernel.py --config wisdom --launches 2 --precision fp32 --grid 512,512,512"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diff_uvw_rk3 -s 1 -c 1 -o $OUT/diff_uvw_rk3 $P --kernel diff_uvw_rk3 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rk3_uvw -s 1 -c 1 -o $OUT/rk3_uvw $P --kernel rk3_uvw 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diff_uvw_fp32 -s 1 -c 1 -o $OUT/diff_uvw $P --kernel diff_uvw 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-suite --no-cpu-baseline > $OUT/bench_under_ncu.json 2>&1
echo done
