# diff_uvw split tendency ring (KL_TSPLIT): deeper halo'd prefetch at the same occupancy — headline + 512^3 records
OUT=gpurun_out/r04x; mkdir -p $OUT
V='--variant "" --variant KL_TSPLIT=1,KL_TDEPTH=1'
timeout 900 python tools/variant_probe.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 --variant "" --variant KL_TSPLIT=1,KL_TDEPTH=1 \
  --config '{"depth": 1}' --config '{"depth": 2}' --rounds 4 --reps 5 --json-out $OUT/tsplit.jsonl > /dev/null 2> $OUT/err_1024.txt
echo 1024 rc $?
for pg in fp32:512 fp64:512; do
  p=${pg%:*}; g=${pg#*:}
  timeout 900 python tools/variant_probe.py --kernel diff_uvw --precision $p --grid $g,$g,$g --variant "" --variant KL_TSPLIT=1,KL_TDEPTH=1 \
    --config '{"depth": 1}' --config '{"depth": 2}' --rounds 4 --json-out $OUT/tsplit.jsonl > /dev/null 2> $OUT/err_$p.txt
  echo $pg rc $?
done
