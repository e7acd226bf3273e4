set -x
mkdir -p gpurun_out/pz
python -m pytest tests -q -m gpu -x 2>&1 | tail -3
CFG='{"staging":"ZMARCH","block_x":32,"block_y":8,"tile_x":1,"tile_y":2,"zchunk":32,"block_z":1,"tile_z":1}'
python tools/profile_kernel.py --kernel diff_uvw --precision fp32 --grid 512,512,512 --config "$CFG" --launches 3
timeout 300 ncu --set full --clock-control none --import-source on -k regex:diff_uvw -s 1 -c 1 -o gpurun_out/pz/diff_zm python tools/profile_kernel.py --kernel diff_uvw --precision fp32 --grid 512,512,512 --config "$CFG" --launches 2 2>&1 | tail -2
CFGA='{"staging":"ZMARCH","block_x":32,"block_y":8,"tile_x":1,"tile_y":2,"zchunk":32,"block_z":1,"tile_z":1}'
python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 512,512,512 --config "$CFGA" --launches 3
timeout 300 ncu --set full --clock-control none --import-source on -k regex:advec_u -s 1 -c 1 -o gpurun_out/pz/advec_zm python tools/profile_kernel.py --kernel advec_u --precision fp32 --grid 512,512,512 --config "$CFGA" --launches 2 2>&1 | tail -2
