# r02m: evisc_smag xshare — GPU parity, exhaustive sessions over the xshare sub-space at 512^3, head-to-head rebase
timeout 900 python -m pytest tests/test_gpu_family.py -q -p no:cacheprovider -k "shared_x_edges or plane_march" > gpurun_out/r02m_pytest.txt 2>&1
echo pytest rc $?
FOC='unravel == "XYZ" && min_blocks == 1 && (zchunk == 32 || zchunk == 64 || zchunk == 128) && depth <= 2 && xshare == 1'
for p in fp32 fp64; do
  timeout 1500 python -m paper_2303_12374_b200.autotune --kernel evisc_smag --precision $p --grid 512,512,512 \
    --family TMA --strategy exhaustive --budget-evals 3000 --budget-seconds 1200 --restrict "$FOC" \
    --wisdom gpurun_out/r02m_scratch --sessions profiles/sessions_r02 --json-out gpurun_out/r02m_tune.jsonl > gpurun_out/r02m_tune_$p.log 2>&1
  echo tune $p rc $?
  python tools/rebase_wisdom.py --kernel evisc_smag --precision $p --grid 512,512,512 \
    --sessions profiles/sessions_r02/evisc_smag_${p}_512x512x512.exhaustive.tma.restricted.seed0.klsession --top 8 --rounds 5 \
    --json-out gpurun_out/r02m_rebase.jsonl > gpurun_out/r02m_rebase_$p.log 2>&1
  echo rebase $p rc $?
done
cp wisdom/evisc_smag_*.wisdom gpurun_out/
cp profiles/sessions_r02/evisc_smag_* gpurun_out/ 2>/dev/null
