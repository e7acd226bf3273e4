# ncu --set full of the current hot-path kernels at the bench / BASELINE shapes (wisdom-selected).
OUT=${OUT:-gpurun_out/nh}
mkdir -p $OUT
P="python tools/profile_kernel.py --config wisdom --launches 2"
cap() {  # name kernel precision grid
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o $OUT/$1 $P --kernel $2 --precision $3 --grid $4 2>&1 | tail -1
}
cap diff_fp32_1024 diff_uvw fp32 1024,1024,1024
cap advec_fp32_512 advec_u fp32 512,512,512
cap advec_fp32_256 advec_u fp32 256,256,256
cap diff_fp64_512 diff_uvw fp64 512,512,512
cap advec_fp64_512 advec_u fp64 512,512,512
