# full GPU suite, retune evisc_smag (pair path), bench, ncu of evisc_smag.
OUT=${OUT:-gpurun_out/r13}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.txt 2>&1; rc=$?; echo "pytest rc=$rc"; tail -15 $OUT/pytest.txt
[ $rc = 0 ] || exit $rc
cp -r wisdom $OUT/wisdom
at() { timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl "$@" 2>&1 | tail -1 | cut -c1-300; }
for p in fp32 fp64; do
  at --kernel evisc_smag --precision $p --grid 512,512,512 --family TMA --focused --strategy exhaustive --budget-evals 2000 --budget-seconds 1500
  at --kernel evisc_smag --precision $p --grid 512,512,512 --family DIRECT --strategy random --budget-evals 40 --budget-seconds 300 --seed 3
done
timeout 900 $S --vary zchunk=8,16,32,64 --vary block_y=2,4,8 --vary depth=1,2
timeout 1200 python bench.py --wisdom $OUT/wisdom > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -3 $OUT/bench.err; head -c 400 $OUT/bench.json
P="python tools/profile_kernel.py --wisdom $OUT/wisdom --config wisdom --launches 2"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:evisc -s 1 -c 1 -o $OUT/evisc_smag_fp32_512 $P --kernel evisc_smag --precision fp32 --grid 512,512,512 2>&1 | tail -1
