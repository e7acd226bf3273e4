"""``bench.py --gpus N`` without a launcher spawns its own N ranks (CPU check).

The reference arm needs no GPU, so the spawner, the torch-free rendezvous
(ProcessGroup) and the rank-0-prints-one-line contract are exercised here:
rank 0 runs the CPU reference on a small grid, rank 1 exits, the parent
returns 0 and exactly one JSON line reaches stdout with ``n_gpus: 2``.
"""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not (ROOT / "oracle" / "_build" / "libstencil_ref.so").exists()
                    or not (ROOT / "paper_2303_12374_b200" / "libklb200.so").exists(),
                    reason="oracle / C-ABI libraries not built")
def test_bench_spawns_two_ranks_for_the_reference_arm():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                          "--warmup", "1", "--workload", "advec_u_fp32_256x256x96", "--reference-budget", "30"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["decomposition"] == "z-slab x2"
