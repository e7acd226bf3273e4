# config 2: balanced row runs at exactly 4 blocks per SM (ysplit 4 -> 592 blocks) for the best 256^3 tilings
OUT=gpurun_out/r04g; mkdir -p $OUT
timeout 1200 python - > /dev/null 2> $OUT/ysplit.err <<'PY'
import json, sys
sys.path.insert(0, "tools")
import variant_probe
tiles = [dict(block_x=16, block_y=4, tile_x=4, tile_y=2), dict(block_x=16, block_y=8, tile_x=4, tile_y=2),
         dict(block_x=32, block_y=4, tile_x=4, tile_y=2), dict(block_x=64, block_y=2, tile_x=2, tile_y=4),
         dict(block_x=32, block_y=8, tile_x=4, tile_y=1)]
argv = ["--rounds", "5", "--no-check", "--json-out", "gpurun_out/r04g/ysplit.jsonl"]
for t in tiles:
    for y in (2, 4, 8):
        argv += ["--config", json.dumps(dict(t, ysplit=y))]
variant_probe.main(argv)
PY
echo rc $?
