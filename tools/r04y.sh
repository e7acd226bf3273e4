# diff_uvw split tendency ring at 1024^3: head-to-head, more rounds (record vs split depth 2 / tdepth 1 vs split depth 1 / tdepth 2)
OUT=gpurun_out/r04y; mkdir -p $OUT
timeout 1200 python - > /dev/null 2> $OUT/err.txt <<'PY'
import json, sys
sys.path.insert(0, "tools")
import variant_probe
argv = ["--kernel", "diff_uvw", "--precision", "fp32", "--grid", "1024,1024,1024", "--rounds", "8", "--reps", "5",
        "--variant", "", "--variant", "KL_TSPLIT=1,KL_TDEPTH=1", "--variant", "KL_TSPLIT=1,KL_TDEPTH=2",
        "--config", json.dumps({"depth": 1}), "--config", json.dumps({"depth": 2}),
        "--json-out", "gpurun_out/r04y/tsplit.jsonl"]
variant_probe.main(argv)
PY
echo rc $?
