# Re-tune every problem size the benchmark and BASELINE configs use, after the
# space change (precision-aware shared-memory restriction; diff_uvw TMA column
# tiles).  Per problem: an exhaustive session over the focused TMA sub-space
# (XYZ launch order, min_blocks 1, zchunk 32/64/128, depth 1/2: every block
# shape and thread tile), then a surrogate session over the whole TMA family
# and a random one over DIRECT; keep-best merges them into $OUT/wisdom.
set -x
OUT=${OUT:-gpurun_out/tune5}
mkdir -p $OUT
R='unravel == "XYZ" && min_blocks == 1 && (zchunk == 32 || zchunk == 64 || zchunk == 128) && depth <= 2 && block_x * tile_x >= 32'
at() { timeout ${T:-1500} python -m paper_2303_12374_b200.autotune --wisdom $OUT/wisdom --sessions $OUT/sessions --json-out $OUT/summary.jsonl "$@" 2>&1 | tail -1 | cut -c1-400; }
tune() {  # kernel precision grid surrogate_evals
  at --kernel $1 --precision $2 --grid $3 --family TMA --strategy exhaustive --budget-evals 2000 --budget-seconds 1500 --restrict "$R"
  at --kernel $1 --precision $2 --grid $3 --family TMA --strategy surrogate --budget-evals $4 --budget-seconds 600 --seed 1
  at --kernel $1 --precision $2 --grid $3 --family DIRECT --strategy random --budget-evals 20 --budget-seconds 300
}
tune diff_uvw fp32 1024,1024,1024 60
tune advec_u fp32 256,256,256 60
tune advec_u fp32 512,512,512 40
tune advec_u fp64 512,512,512 60
tune diff_uvw fp64 512,512,512 60
tune diff_uvw fp32 512,512,512 40
tune diff_uvw fp64 64,64,64 40
tune diff_uvw fp32 1024,1024,512 30
tune diff_uvw fp32 1024,1024,256 30
tune diff_uvw fp32 1024,1024,128 30
at --kernel diff_uvw --precision fp32 --grid 1024,1024,1 --family TMA --strategy surrogate --budget-evals 60 --budget-seconds 300
at --kernel diff_uvw --precision fp32 --grid 1024,1024,1 --family DIRECT --strategy random --budget-evals 40 --budget-seconds 300
# the §8f family (DIRECT kernels on the Table-2 space) at 512^3
for k in advec_v advec_w advec_s diff_c evisc_smag; do
  for p in fp32 fp64; do
    at --kernel $k --precision $p --grid 512,512,512 --strategy random --budget-evals 60 --budget-seconds 300 --seed 3
  done
done
# §8f row 1: the fused RK3 epilogue (same space as diff_uvw) and the separate RK3 pass it replaces
for p in fp32 fp64; do
  at --kernel diff_uvw_rk3 --precision $p --grid 512,512,512 --family TMA --strategy exhaustive --budget-evals 2000 --budget-seconds 1500 --restrict "$R"
  at --kernel rk3_uvw --precision $p --grid 512,512,512 --strategy random --budget-evals 60 --budget-seconds 300 --seed 3
done
