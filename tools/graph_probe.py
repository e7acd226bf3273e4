"""Eager bound launches vs one captured CUDA graph on the launch-bound small
problems (bench.py graph_measure, standalone).

    python tools/graph_probe.py [--wisdom wisdom] [--n 200]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--wisdom", default=str(ROOT / "wisdom"))
ap.add_argument("--n", type=int, default=200)
a = ap.parse_args()
ctx = open_device(0)
print(json.dumps(bench.graph_measure(ctx, NvrtcCompiler(ctx), a.wisdom, n=a.n), indent=1))
