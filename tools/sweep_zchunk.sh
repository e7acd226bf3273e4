# Larger z-chunks than the space's 128 (fewer chunk-boundary halo planes, fewer blocks) around the tuned points.
OUT=${OUT:-gpurun_out/zc}
mkdir -p $OUT
timeout 900 python tools/sweep.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 --vary zchunk=64,128,256,512,1024 --vary depth=1,2 --json-out $OUT/diff.jsonl
timeout 900 python tools/sweep.py --kernel advec_u --precision fp32 --grid 512,512,512 --vary zchunk=64,128,256,512 --vary depth=1,2 --json-out $OUT/advec.jsonl
timeout 900 python tools/sweep.py --kernel diff_uvw --precision fp64 --grid 512,512,512 --vary zchunk=64,128,256,512 --vary depth=1,2 --json-out $OUT/diff64.jsonl
