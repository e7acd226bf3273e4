# r02j: ncu evidence for config 2 (ysplit kernel vs previous record), headline kernel, bench launch list; sanitizers
set -x
timeout 600 python -m pytest tests/test_gpu_stencils.py -q -p no:cacheprovider -k balanced > gpurun_out/r02j_balanced.txt 2>&1
OLD='{"block_x":32,"block_y":8,"tile_x":4,"tile_y":2,"zchunk":64,"depth":3,"staging":"TMA","contiguous_x":true,"unravel":"XYZ","min_blocks":1,"ysplit":0}'
ncu --set full --clock-control none --import-source on -k regex:advec_u -c 1 -f -o gpurun_out/r02j_advec256_ysplit \
  python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 256,256,256 --config wisdom --launches 2 > gpurun_out/r02j_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:advec_u -c 1 -f -o gpurun_out/r02j_advec256_prev \
  python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 256,256,256 --config "$OLD" --launches 2 > gpurun_out/r02j_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:diff_uvw -c 1 -f -o gpurun_out/r02j_diff1024 \
  python tools/profile_kernel.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 --config wisdom --launches 2 > gpurun_out/r02j_ncu3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02j_launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-suite --no-cpu-baseline > gpurun_out/r02j_launch_bench.log 2>&1
python tools/ncu_summary.py gpurun_out/r02j_advec256_ysplit.ncu-rep gpurun_out/r02j_advec256_prev.ncu-rep gpurun_out/r02j_diff1024.ncu-rep > gpurun_out/r02j_ncu_summary.txt 2>&1
compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_stencils.py -q -p no:cacheprovider -k "balanced and fp32" > gpurun_out/r02j_memcheck.txt 2>&1
compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest tests/test_gpu_stencils.py -q -p no:cacheprovider -k "balanced and fp32" > gpurun_out/r02j_racecheck.txt 2>&1
compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_graph.py -q -p no:cacheprovider -k pdl > gpurun_out/r02j_memcheck_pdl.txt 2>&1
compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_graph.py -q -p no:cacheprovider -k pdl > gpurun_out/r02j_synccheck_pdl.txt 2>&1
echo done
