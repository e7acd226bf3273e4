# north star: each tunable variant of the 512^3 records evidenced by achieved HBM GB/s (event time + ncu DRAM bytes)
OUT=gpurun_out/r04i; mkdir -p $OUT
for kp in diff_uvw:fp32 advec_u:fp32 diff_uvw:fp64 advec_u:fp64; do
  k=${kp%:*}; p=${kp#*:}
  timeout 900 python tools/knob_sweep.py --kernel $k --precision $p --grid 512,512,512 --mode time --out $OUT/${k}_${p}.jsonl > /dev/null 2> $OUT/${k}_${p}.err
  echo $kp time rc $?
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"^${k}_" --csv --log-file $OUT/${k}_${p}_ncu.csv \
    python tools/knob_sweep.py --kernel $k --precision $p --grid 512,512,512 --mode ncu > /dev/null 2> $OUT/${k}_${p}_ncu.err
  echo $kp ncu rc $?
done
