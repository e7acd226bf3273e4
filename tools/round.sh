# tests -> tuning -> bench in one box session
set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
OUT=gpurun_out/tune2 timeout 2400 bash tools/tune_all.sh > gpurun_out/tune2_log.txt 2>&1
tail -3 gpurun_out/tune2_log.txt
timeout 900 python bench.py --wisdom gpurun_out/tune2/wisdom > gpurun_out/bench2.json 2> gpurun_out/bench2.err
tail -2 gpurun_out/bench2.err; head -c 600 gpurun_out/bench2.json
