# Wider exhaustive sessions for the §8f family TMA kernels at 512^3 (the wisdom
# was made with the focused sub-space): XYZ, depth 1-3, min_blocks 1-2,
# zchunk 16-128; keep-best merged into a copy of wisdom/.
OUT=${OUT:-gpurun_out/wf}
mkdir -p $OUT
cp -r wisdom $OUT/wisdom
R='unravel == "XYZ" && depth <= 3 && min_blocks <= 2 && (zchunk == 16 || zchunk == 32 || zchunk == 64 || zchunk == 128)'
for k in advec_v advec_w advec_s diff_c; do
  for p in fp32 fp64; do
    timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl \
      --kernel $k --precision $p --grid 512,512,512 --family TMA --strategy exhaustive --budget-evals 4000 --budget-seconds 1200 \
      --restrict "$R" 2>&1 | tail -1 | cut -c1-200
  done
done
