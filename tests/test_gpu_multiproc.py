"""The N > 1 path as several processes on ONE GPU (gpurun gives one; NCCL
refuses two ranks on a device, so the halo planes are relayed through the
host over gloo by ``StagedExchanger``): the slab decomposition stepped by
two/three ranks matches the oracle, and ``bench.py --gpus 2`` under torchrun
prints one valid JSON line (rank 0) for both arms."""

import json
import os
import re
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(nproc, *args, timeout=900):
    env = dict(os.environ, KL_HALO_TRANSPORT="staged", KL_DEVICE_ORDINAL="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), *args]
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("kernel,precision,grid,nproc", [("diff_uvw", "fp32", "64,40,30", 2),
                                                         ("advec_u", "fp64", "48,32,40", 3)])
def test_ranks_match_oracle(kernel, precision, grid, nproc):
    out = _torchrun(nproc, "tests/multiproc_slab_check.py", kernel, precision, grid)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    # torchrun multiplexes the ranks' stdout (lines may run together)
    assert len(re.findall(r"rank \d+ ok ", out.stdout)) == nproc, out.stdout
    assert "FAIL" not in out.stdout


def test_bench_two_ranks_prints_one_line_per_arm():
    common = ["--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "diff_uvw_fp32_256"]
    out = _torchrun(2, "bench.py", *common, "--e2e-steps", "1", "--e2e-chunks", "4")
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["decomposition"] == "z-slab x2"
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    ref = _torchrun(2, "bench.py", *common, "--impl", "reference")
    assert ref.returncode == 0, ref.stdout[-2000:] + ref.stderr[-2000:]
    lines = [json.loads(x) for x in ref.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["value"] > 0
