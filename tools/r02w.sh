# r02w: data-movement floor across the best configurations (full kernel vs KL_SKEL=1 skeleton): advec_u fp32 256^3
# (the round-2 exhaustive ysplit session and round 1's focused session) and evisc_smag fp32 512^3
timeout 1200 python tools/skeleton_sweep.py --top 40 --json-out gpurun_out/r02w_skel.jsonl \
  --session profiles/sessions_r02/advec_u_fp32_256x256x256.exhaustive.tma.restricted.seed0.klsession > gpurun_out/r02w_a.log 2>&1
echo a rc $?
S=profiles/sessions_r01c/advec_u_fp32_256x256x256.exhaustive.tma.restricted.seed0.klsession
[ -n "$S" ] && timeout 1200 python tools/skeleton_sweep.py --top 30 --json-out gpurun_out/r02w_skel.jsonl --session $S > gpurun_out/r02w_b.log 2>&1
echo b rc $?
timeout 1200 python tools/skeleton_sweep.py --top 20 --json-out gpurun_out/r02w_skel.jsonl \
  --session profiles/sessions_r02/evisc_smag_fp32_512x512x512.exhaustive.tma.restricted.seed0.klsession > gpurun_out/r02w_c.log 2>&1
echo c rc $?
