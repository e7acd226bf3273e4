# evisc_smag TMA column tiles with row-span vector loads (march_rows): parity,
# sweep of column tiles at 512^3, focused re-tune, ncu of the re-tuned fp32 kernel.
OUT=${OUT:-gpurun_out/er}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_family.py -q -x -k "evisc or plane or misaligned or family" > $OUT/pytest.txt 2>&1; rc=$?; echo "pytest rc=$rc"; tail -3 $OUT/pytest.txt
[ $rc = 0 ] || { tail -40 $OUT/pytest.txt; exit $rc; }
B='{"block_x":32,"block_y":2,"depth":2,"staging":"TMA","tile_x":4,"tile_y":4,"contiguous_x":true,"unravel":"XYZ","zchunk":64}'
for p in fp32 fp64; do
  timeout 900 python tools/sweep.py --kernel evisc_smag --precision $p --grid 512,512,512 --base "$B" --vary tile_x=2,4 --vary tile_y=2,4 --vary block_x=16,32 --vary block_y=1,2,4 --vary depth=1,2 --json-out $OUT/sweep_$p.jsonl 2>&1 | sort -k5 -n | head -8
done
cp -r wisdom $OUT/wisdom
at() { timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl "$@" 2>&1 | tail -1 | cut -c1-300; }
for p in fp32 fp64; do
  at --kernel evisc_smag --precision $p --grid 512,512,512 --family TMA --focused --strategy exhaustive --budget-evals 2000 --budget-seconds 1500
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:evisc -s 1 -c 1 -o $OUT/evisc_smag_fp32_512 \
  python tools/profile_kernel.py --wisdom $OUT/wisdom --config wisdom --launches 2 --kernel evisc_smag --precision fp32 --grid 512,512,512 2>&1 | tail -1
