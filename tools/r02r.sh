# r02r: evisc_smag data-movement floor — wisdom record vs its KL_SKEL=1 skeleton (TMA ring, barriers and
# evisc stores only), fp32 (xshare record and the previous xshare=0 record) and fp64, 512^3
timeout 900 python tools/ysplit_probe.py --kernel evisc_smag --precision fp32 --grid 512,512,512 --reps 21 \
  --case '{}' --case '{"defines": {"KL_SKEL": 1}}' \
  --case '{"block_x": 128, "block_y": 2, "zchunk": 64, "xshare": 0}' \
  --case '{"block_x": 128, "block_y": 2, "zchunk": 64, "xshare": 0, "defines": {"KL_SKEL": 1}}' \
  --json-out gpurun_out/r02r_skel.jsonl > gpurun_out/r02r_fp32.log 2>&1
echo fp32 rc $?
timeout 900 python tools/ysplit_probe.py --kernel evisc_smag --precision fp64 --grid 512,512,512 --reps 21 \
  --case '{}' --case '{"defines": {"KL_SKEL": 1}}' \
  --json-out gpurun_out/r02r_skel.jsonl > gpurun_out/r02r_fp64.log 2>&1
echo fp64 rc $?
