# round-2 evidence run on one fresh box: GPU tests, smoke, default bench, reference arm, 2-rank bench (no launcher)
T=${1:-r02k}
export KL_PARITY_LOG=gpurun_out/${T}_parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/${T}_pytest.txt 2>&1
echo pytest rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
echo smoke rc $?
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo bench rc $?
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
echo reference rc $?
KL_DEVICE_ORDINAL=0 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-suite --e2e-steps 1 > gpurun_out/${T}_bench_2ranks_1gpu.json 2> gpurun_out/${T}_bench_2ranks_1gpu.err
echo bench2 rc $?
timeout 300 python tools/dispatch_overhead.py > gpurun_out/${T}_dispatch.json 2>&1
echo dispatch rc $?
