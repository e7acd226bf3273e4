# Wider exhaustive sessions for the headline shapes (XYZ order; min_blocks 1-4, depth 1-3, zchunk 32-128),
# keep-best merged into a copy of wisdom/; then the default bench.
set -x
OUT=${OUT:-gpurun_out/r14}
mkdir -p $OUT
cp -r wisdom $OUT/wisdom
R='unravel == "XYZ" && min_blocks <= 4 && (zchunk == 32 || zchunk == 64 || zchunk == 128) && block_x * tile_x >= 32'
at() { timeout 3000 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl "$@" 2>&1 | tail -1 | cut -c1-300; }
at --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 --family TMA --strategy exhaustive --budget-evals 8000 --budget-seconds 2700 --restrict "$R"
at --kernel advec_u --precision fp32 --grid 512,512,512 --family TMA --strategy exhaustive --budget-evals 8000 --budget-seconds 1500 --restrict "$R"
at --kernel advec_u --precision fp32 --grid 256,256,256 --family TMA --strategy exhaustive --budget-evals 8000 --budget-seconds 1200 --restrict "$R"
timeout 1200 python bench.py --wisdom $OUT/wisdom > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -2 $OUT/bench.err; head -c 300 $OUT/bench.json
