set -x
mkdir -p gpurun_out/e5
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for spec in "diff_uvw fp32 512,512,512" "advec_u fp32 512,512,512" "diff_uvw fp64 512,512,512" "advec_u fp64 512,512,512"; do
  set -- $spec
  timeout 900 python -m paper_2303_12374_b200.autotune --kernel $1 --precision $2 --grid $3 --strategy random --budget-evals 80 --budget-seconds 400 --wisdom gpurun_out/e5/wisdom --sessions gpurun_out/e5/sessions --json-out gpurun_out/e5/summary.jsonl --family TMA 2>&1 | tail -1
done
