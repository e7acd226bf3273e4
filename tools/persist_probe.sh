# EXPERIMENT (reverted): the `persist` knob measured here existed only in the build this
# script ran against; the results are profiles/sweeps_r01/advec_u_*_persist.jsonl.
# advec_u persistent schedule (persist = blocks per SM sharing the plane-tiles
# evenly): parity tests, then sweeps around the tuned points at the BASELINE
# shapes (config 2: 256^3 fp32; north star 512^3 fp32; config 3: 512^3 fp64).
OUT=${OUT:-gpurun_out/pp}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_stencils.py -x -q -k "advec" 2>&1 | tail -3 | tee $OUT/tests.log
sw() { timeout 900 python tools/sweep.py --kernel advec_u "$@" 2>&1 | tail -40; }
sw --precision fp32 --grid 256,256,256 --vary persist=0,1,2 --vary zchunk=16,32,64,128 --json-out $OUT/a32_256.jsonl
sw --precision fp32 --grid 256,256,256 --vary persist=1,2 --vary block_y=2,4,8 --vary depth=1,2,3 --json-out $OUT/a32_256b.jsonl
sw --precision fp32 --grid 512,512,512 --vary persist=0,1,2 --vary zchunk=64,128 --json-out $OUT/a32_512.jsonl
sw --precision fp64 --grid 512,512,512 --vary persist=0,1,2 --vary zchunk=64,128 --json-out $OUT/a64_512.jsonl
sw --precision fp32 --grid 128,128,128 --vary persist=0,1,2 --vary zchunk=16,32,64 --json-out $OUT/a32_128.jsonl
