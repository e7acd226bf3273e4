# advec_u z-head experiment (KL_ZHEAD: z-window head from global into registers, u ring DEPTH+1 slots)
OUT=gpurun_out/r04v; mkdir -p $OUT
for g in 256 512; do
  timeout 900 python tools/variant_probe.py --kernel advec_u --precision fp32 --grid $g,$g,$g \
    --variant "" --variant KL_ZHEAD=1 --variant KL_ZHEAD=2 \
    --config '{"depth": 2}' --config '{"depth": 3}' --config '{"depth": 1}' \
    --rounds 3 --json-out $OUT/zhead.jsonl > /dev/null 2> $OUT/zhead_$g.err
  echo $g rc $?
done
timeout 600 python tools/variant_probe.py --kernel advec_u --precision fp64 --grid 512,512,512 \
    --variant "" --variant KL_ZHEAD=2 --config '{"depth": 2}' --config '{"depth": 3}' \
    --rounds 3 --json-out $OUT/zhead.jsonl > /dev/null 2> $OUT/zhead_fp64.err
echo fp64 rc $?
