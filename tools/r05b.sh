# one-knob evidence for the §8f family TMA records at 512^3
OUT=gpurun_out/r05b_knobs; mkdir -p $OUT
for kp in advec_v:fp32 diff_c:fp32 evisc_smag:fp32 advec_s:fp64; do
  k=${kp%:*}; p=${kp#*:}
  timeout 900 python tools/knob_sweep.py --kernel $k --precision $p --grid 512,512,512 --mode time --out $OUT/${k}_${p}.jsonl > /dev/null 2> $OUT/${k}_${p}.err
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"^${k}_" --csv --log-file $OUT/${k}_${p}_ncu.csv \
    python tools/knob_sweep.py --kernel $k --precision $p --grid 512,512,512 --mode ncu > /dev/null 2> $OUT/${k}_${p}_ncu.err
  echo $kp rc $?
done
