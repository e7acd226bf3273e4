set -x
mkdir -p gpurun_out/bp
timeout 900 python bench.py > gpurun_out/bp/bench.json 2> gpurun_out/bp/bench.err; tail -3 gpurun_out/bp/bench.err; cat gpurun_out/bp/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bp/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-suite --no-cpu-baseline > gpurun_out/bp/bench_under_ncu.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:diff_uvw -s 1 -c 1 -o gpurun_out/bp/diff_1024_tuned python tools/profile_kernel.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 --config wisdom --launches 2 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:advec_u -s 1 -c 1 -o gpurun_out/bp/advec_256_tuned python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 256,256,256 --config wisdom --launches 2 2>&1 | tail -3
