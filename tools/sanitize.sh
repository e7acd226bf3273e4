# compute-sanitizer memcheck + racecheck (shared memory) of one TMA configuration per kernel family,
# wisdom-selected, on small ragged grids.  Summaries in $OUT/*.txt.
OUT=${OUT:-gpurun_out/san}
mkdir -p $OUT
P="python tools/profile_kernel.py --launches 1 --config wisdom"
run() {  # tool kernel precision grid
  timeout 900 compute-sanitizer --tool $1 --print-limit 20 $P --kernel $2 --precision $3 --grid $4 > $OUT/$1_$2_$3.txt 2>&1
  echo "$1 $2 $3 $4 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/$1_$2_$3.txt | tr '\n' ' ')"
}
for tool in memcheck racecheck; do
  run $tool diff_uvw fp32 150,70,45
  run $tool diff_uvw_rk3 fp64 90,70,45
  run $tool advec_u fp32 150,70,45
  run $tool advec_u fp64 90,50,45
  run $tool advec_v fp32 150,70,45
  run $tool advec_w fp64 90,50,45
  run $tool advec_s fp32 150,70,45
  run $tool diff_c fp32 150,70,45
  run $tool evisc_smag fp32 150,70,45
done
