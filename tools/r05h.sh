# the paper's evaluation (capture table, Table-2 tuning distribution, cross-scenario matrix) on one B200
OUT=gpurun_out/r05h; mkdir -p $OUT
timeout 3000 python tools/paper_eval.py --random 150 --out $OUT/paper_eval.json 2> $OUT/paper_eval.err
echo rc $?
