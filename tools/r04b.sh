# round-2 late session: rk3_uvw vector path (parity + tuning at 512^3) and the config-2 size-matched floors
OUT=gpurun_out/r04b
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_family.py -q -p no:cacheprovider -k rk3 > $OUT/pytest_rk3.txt 2>&1
echo pytest rc $?
timeout 300 python tools/floor_probe.py > $OUT/floor_probe.json 2> $OUT/floor_probe.err
echo floor rc $?
cp -r wisdom $OUT/wisdom
R='contiguous_x && tile_x >= 2 && unravel == "XYZ" && min_blocks <= 2'
for p in fp32 fp64; do
  timeout 900 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl \
    --kernel rk3_uvw --precision $p --grid 512,512,512 --strategy random --budget-evals 250 --budget-seconds 600 \
    --restrict "$R" 2>&1 | tail -1 | cut -c1-300
  timeout 600 python tools/rebase_wisdom.py --kernel rk3_uvw --precision $p --grid 512,512,512 --wisdom $OUT/wisdom \
    --sessions $OUT/sessions/*rk3_uvw_$p*.klsession --top 6 --rounds 5 --json-out $OUT/rebase.jsonl 2>&1 | tail -2
done
timeout 900 python tools/skeleton_sweep.py --session profiles/sessions_r02/advec_u_fp32_256x256x256.exhaustive.tma.restricted.seed0.klsession \
  --top 8 --levels 1,2,3 --json-out $OUT/skeleton_levels.jsonl > /dev/null 2> $OUT/skeleton_levels.err
echo skel rc $?
