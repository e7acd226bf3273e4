# BASELINE config 1 (diff_uvw fp64 64^3): exhaustive session over the short
# z-chunks (8/16 planes) the focused sub-space leaves out, XYZ and ZXY orders;
# rk3_uvw at the same shape as the elementwise floor of a cold 64^3 pass.
OUT=${OUT:-gpurun_out/ts}
mkdir -p $OUT
cp -r wisdom $OUT/wisdom
timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl \
  --kernel diff_uvw --precision fp64 --grid 64,64,64 --family TMA --strategy exhaustive --budget-evals 3000 --budget-seconds 1200 \
  --restrict '(zchunk == 8 || zchunk == 16) && depth <= 2 && (unravel == "XYZ" || unravel == "ZXY") && min_blocks <= 4' 2>&1 | tail -1 | cut -c1-400
timeout 600 python tools/sweep.py --kernel rk3_uvw --precision fp64 --grid 64,64,64 --vary block_x=64,128,256 --json-out $OUT/rk3_64.jsonl 2>&1 | tail -4
timeout 600 python tools/sweep.py --kernel diff_uvw --precision fp64 --grid 64,64,64 --wisdom $OUT/wisdom --vary depth=1,2 --json-out $OUT/diff_64.jsonl 2>&1 | tail -4
