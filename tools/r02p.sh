# r02p: can NCCL run two ranks on the one GPU gpurun provides?  (production NCCL halo path at N=2)
export NCCL_DEBUG=INFO
KL_DEVICE_ORDINAL=0 KL_HALO_TRANSPORT=nccl timeout 300 python bench.py --gpus 2 --steps 3 --warmup 3 --no-suite --e2e-steps 0 \
  > gpurun_out/r02p_nccl2.json 2> gpurun_out/r02p_nccl2.err
echo nccl2 rc $?
KL_HALO_TRANSPORT=nccl timeout 300 python tests/multiproc_slab_check.py --help > gpurun_out/r02p_help.txt 2>&1
echo help rc $?
nvidia-smi -q | grep -i -A3 "compute mode" > gpurun_out/r02p_smi.txt 2>&1
which nvidia-cuda-mps-control >> gpurun_out/r02p_smi.txt 2>&1
echo done
