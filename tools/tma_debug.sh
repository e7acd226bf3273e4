CFG='{"staging":"TMA","block_x":32,"block_y":4,"tile_x":1,"tile_y":1,"zchunk":8,"block_z":1,"tile_z":1,"depth":1}'
timeout 120 compute-sanitizer --tool memcheck --print-limit 2 --show-backtrace device python tools/profile_kernel.py --kernel diff_uvw --precision fp32 --grid 64,32,16 --config "$CFG" --launches 1 2>&1 | head -20
timeout 120 compute-sanitizer --tool memcheck --print-limit 2 --show-backtrace device python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 64,32,16 --config "$CFG" --launches 1 2>&1 | head -20
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
