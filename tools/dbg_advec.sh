timeout 600 python -m pytest tests/test_gpu_stencils.py -q -x -k "rejected or sampled" 2>&1 | tail -15
CFG='{"staging":"TMA","block_x":32,"block_y":1,"tile_x":1,"tile_y":1,"zchunk":8,"block_z":1,"tile_z":1,"depth":1,"min_blocks":2}'
timeout 300 compute-sanitizer --tool racecheck --print-limit 3 python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 64,32,24 --config "$CFG" --launches 1 2>&1 | tail -12
timeout 300 compute-sanitizer --tool synccheck --print-limit 3 python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 64,32,24 --config "$CFG" --launches 1 2>&1 | tail -6
