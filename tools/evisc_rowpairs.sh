# evisc_smag TMA fp32 tile 1 x even: rows in packed pairs (march_rowpairs):
# parity, sweep around the tuned tile, focused re-tune (fp32), ncu.
OUT=${OUT:-gpurun_out/rp}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_family.py tests/test_gpu_graph.py -q -x > $OUT/pytest.txt 2>&1; rc=$?; echo "pytest rc=$rc"; tail -3 $OUT/pytest.txt
[ $rc = 0 ] || { tail -40 $OUT/pytest.txt; exit $rc; }
timeout 600 python tools/sweep.py --kernel evisc_smag --precision fp32 --grid 512,512,512 --wisdom wisdom --vary block_x=64,128 --vary block_y=2,4 --vary tile_y=2,4 --json-out $OUT/sweep.jsonl 2>&1 | tail -9
cp -r wisdom $OUT/wisdom
timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl \
  --kernel evisc_smag --precision fp32 --grid 512,512,512 --family TMA --focused --strategy exhaustive --budget-evals 2000 --budget-seconds 1500 2>&1 | tail -1 | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:evisc -s 1 -c 1 -o $OUT/evisc_smag_fp32_512 \
  python tools/profile_kernel.py --wisdom $OUT/wisdom --config wisdom --launches 2 --kernel evisc_smag --precision fp32 --grid 512,512,512 2>&1 | tail -1
