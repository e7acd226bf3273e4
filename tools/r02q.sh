# r02q: GPU test of the session checkpoint/resume; the driver's torchrun launch of both bench arms at N=2
# (both ranks pinned to the one GPU with KL_DEVICE_ORDINAL=0: a plumbing check, not a scaling number)
timeout 900 python -m pytest tests/test_gpu_capture_tune.py -q -p no:cacheprovider -rA > gpurun_out/r02q_pytest.txt 2>&1
echo pytest rc $?
KL_DEVICE_ORDINAL=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --no-suite --e2e-steps 1 \
  > gpurun_out/r02q_torchrun2.json 2> gpurun_out/r02q_torchrun2.err
echo torchrun2 rc $?
KL_DEVICE_ORDINAL=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29518 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 \
  > gpurun_out/r02q_torchrun2_ref.json 2> gpurun_out/r02q_torchrun2_ref.err
echo torchrun2 ref rc $?
