set -x
mkdir -p gpurun_out/explore
for spec in "advec_u fp32 256,256,256" "diff_uvw fp32 256,256,256" "advec_u fp64 256,256,256" "diff_uvw fp64 256,256,256"; do
  set -- $spec
  timeout 600 python -m paper_2303_12374_b200.autotune --kernel $1 --precision $2 --grid $3 --strategy random --budget-evals 80 --budget-seconds 240 --wisdom gpurun_out/explore/wisdom --sessions gpurun_out/explore/sessions --json-out gpurun_out/explore/summary.jsonl 2>&1 | tail -12
done
