# z-march loop unrolling (KL_KUNROLL: the advec_u 6-plane z window rotates through registers) on the advec_u records
OUT=gpurun_out/r04l; mkdir -p $OUT
V="--variant KL_KUNROLL=1 --variant KL_KUNROLL=2 --variant KL_KUNROLL=3 --variant KL_KUNROLL=6"
for kp in advec_u:fp32:256 advec_u:fp32:512 advec_u:fp64:512; do
  IFS=: read k p n <<< "$kp"
  timeout 900 python tools/variant_probe.py --kernel $k --precision $p --grid $n,$n,$n $V --rounds 5 --json-out $OUT/unroll.jsonl > /dev/null 2> $OUT/unroll_${k}_${p}_${n}.err
  echo $kp rc $?
done
timeout 600 ncu --metrics smsp__inst_executed.sum,smsp__sass_inst_executed_op_mov.sum,gpu__time_duration.sum --clock-control none -k regex:advec_u --csv \
  --log-file $OUT/ncu_unroll.csv python tools/variant_probe.py --kernel advec_u --precision fp32 --grid 256,256,256 $V --rounds 1 --reps 1 --no-check > /dev/null 2> $OUT/ncu.err
echo ncu rc $?
