# r02o: config-2 data-movement floor — advec_u fp32 256^3 record vs its KL_SKEL=1 skeleton (same TMA rings,
# barriers and ut stores, stencil replaced by ut += 1), at depth 1..3; then the 512^3 pair for comparison
for g in 256,256,256 512,512,512; do
timeout 900 python tools/ysplit_probe.py --kernel advec_u --precision fp32 --grid $g --reps 21 \
  --case '{}' --case '{"defines": {"KL_SKEL": 1}}' \
  --case '{"depth": 1}' --case '{"depth": 1, "defines": {"KL_SKEL": 1}}' \
  --case '{"depth": 3}' --case '{"depth": 3, "defines": {"KL_SKEL": 1}}' \
  --json-out gpurun_out/r02o_skel.jsonl > gpurun_out/r02o_skel_$g.log 2>&1
echo probe $g rc $?
done
