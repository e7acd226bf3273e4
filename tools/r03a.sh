# r03a: sanitizers over the round-2 additions (fused halo kernels diff_uvw_peer / advec_u_peer, the RK3 time loop
# with klb_cyclic_xy, evisc xshare) and ncu of the fused-halo slab launch vs the exchange interior launch (N = 8)
O=gpurun_out/r03a; mkdir -p $O
K="tests/test_gpu_slab.py -q -p no:cacheprovider"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest $K -k "fused or rk3" > $O/memcheck_fused_rk3.txt 2>&1
echo memcheck rc $? $(grep -E "ERROR SUMMARY|passed|failed" $O/memcheck_fused_rk3.txt | tr '\n' ' ')
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest $K -k "fused and fp32" > $O/racecheck_fused.txt 2>&1
echo racecheck rc $? $(grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" $O/racecheck_fused.txt | tr '\n' ' ')
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest $K -k "rk3 and fp32" > $O/synccheck_rk3.txt 2>&1
echo synccheck rc $? $(grep -E "ERROR SUMMARY|passed|failed" $O/synccheck_rk3.txt | tr '\n' ' ')
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_family.py -q -p no:cacheprovider -k "shared_x_edges" > $O/memcheck_xshare.txt 2>&1
echo memcheck xshare rc $? $(grep -E "ERROR SUMMARY|passed|failed" $O/memcheck_xshare.txt | tr '\n' ' ')
# the fused slab launch of the middle rank at N = 8, and the exchange variant's interior launch (its first diff_uvw_fp32)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diff_uvw_peer -c 1 -f -o $O/fused_n8 \
  python tools/fused_halo_probe.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 --ranks 8 --reps 1 > $O/ncu.log 2>&1
echo ncu fused rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^diff_uvw_fp32 -c 1 -f -o $O/exchange_n8 \
  python tools/fused_halo_probe.py --kernel diff_uvw --precision fp32 --grid 1024,1024,1024 --ranks 8 --reps 1 > $O/ncu2.log 2>&1
echo ncu exchange rc $?
python tools/ncu_summary.py $O/fused_n8.ncu-rep $O/exchange_n8.ncu-rep > $O/ncu_summary.txt 2>&1
echo summary rc $?
