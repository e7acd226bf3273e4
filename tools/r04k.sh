# L2 prefetch of the planes beyond the TMA rings (KL_L2PF): headline and config-2 records, head to head
OUT=gpurun_out/r04k; mkdir -p $OUT
V="--variant KL_L2PF=0 --variant KL_L2PF=1 --variant KL_L2PF=2 --variant KL_L2PF=4 --variant KL_L2PF=8"
timeout 900 python tools/variant_probe.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 $V --rounds 4 --reps 5 --json-out $OUT/pf.jsonl > /dev/null 2> $OUT/pf_1024.err
echo 1024 rc $?
for kp in diff_uvw:fp32:512 advec_u:fp32:256 advec_u:fp32:512 diff_uvw:fp64:512 advec_u:fp64:512; do
  IFS=: read k p n <<< "$kp"
  timeout 900 python tools/variant_probe.py --kernel $k --precision $p --grid $n,$n,$n $V --rounds 5 --json-out $OUT/pf.jsonl > /dev/null 2> $OUT/pf_${k}_${p}_${n}.err
  echo $kp rc $?
done
