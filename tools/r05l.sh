# final: ncu of the headline kernel as the bench runs it (16-byte row pitch), the bench launch list, then the evidence run
OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diff_uvw --launch-skip 2 -c 1 -f -o $OUT/r05l_diff1024_row16 \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-suite --no-cpu-baseline > $OUT/r05l_ncu.log 2>&1
echo ncu full rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/r05l_launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-suite --no-cpu-baseline > $OUT/r05l_launch_bench.log 2>&1
echo ncu list rc $?
bash tools/r04j.sh r05l
