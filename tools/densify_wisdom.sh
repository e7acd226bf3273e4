# More anchor shapes in wisdom/ for the hot-path kernels (the selection cascade picks the nearest record):
# focused TMA exhaustive session per shape, keep-best merged into a copy of wisdom/.
set -x
OUT=${OUT:-gpurun_out/dens}
mkdir -p $OUT
cp -r wisdom $OUT/wisdom
at() { timeout 1500 python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl "$@" 2>&1 | tail -1 | cut -c1-200; }
for spec in "advec_u fp32 128" "advec_u fp32 1024" "advec_u fp64 128" "advec_u fp64 256" "advec_u fp64 1024" \
            "diff_uvw fp32 128" "diff_uvw fp32 256" "diff_uvw fp64 128" "diff_uvw fp64 256" "diff_uvw fp64 1024"; do
  set -- $spec
  at --kernel $1 --precision $2 --grid $3,$3,$3 --family TMA --focused --strategy exhaustive --budget-evals 2000 --budget-seconds 1200
done
