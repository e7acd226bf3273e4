set -x
mkdir -p gpurun_out/zm
for spec in "advec_u fp32 256,256,256" "diff_uvw fp32 256,256,256" "advec_u fp64 256,256,256" "diff_uvw fp64 256,256,256"; do
  set -- $spec
  timeout 600 python -m paper_2303_12374_b200.autotune --kernel $1 --precision $2 --grid $3 --strategy random --budget-evals 60 --budget-seconds 240 --wisdom gpurun_out/zm/wisdom --sessions gpurun_out/zm/sessions --json-out gpurun_out/zm/summary.jsonl --restrict 'staging == "ZMARCH"' 2>&1 | tail -3
done
for k in diff_uvw advec_u; do
  for c in default wisdom; do
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/zm/prof_${k}_fp32_$c python tools/profile_kernel.py --kernel $k --precision fp32 --grid 512,512,512 --config $c --launches 2 2>&1 | tail -3
  done
done
