# r02z: RK3 time loop with the fused halo (diff_uvw_rk3_peer + klb_cyclic_xy): virtual ranks and IPC processes
timeout 1500 python -m pytest tests/test_gpu_slab.py tests/test_gpu_multiproc.py -q -p no:cacheprovider -rA -k "fused or rk3" \
  > gpurun_out/r02z_pytest.txt 2>&1
echo pytest rc $?
