set -x
mkdir -p gpurun_out/e3
for spec in "diff_uvw fp32 512,512,512" "diff_uvw fp64 512,512,512" "advec_u fp32 512,512,512" "advec_u fp64 512,512,512"; do
  set -- $spec
  timeout 600 python -m paper_2303_12374_b200.autotune --kernel $1 --precision $2 --grid $3 --strategy random --budget-evals 60 --budget-seconds 300 --wisdom gpurun_out/e3/wisdom --sessions gpurun_out/e3/sessions --json-out gpurun_out/e3/summary.jsonl --family ZMARCH 2>&1 | tail -2
done
