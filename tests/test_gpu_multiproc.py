"""The N > 1 path as several processes on ONE GPU (gpurun gives one GPU).

Every rank is its own process and CUDA context on the same device; the halo
planes travel by the production transport, ``IpcExchanger`` (CUDA IPC: each
rank maps its neighbours' field allocations and pulls the planes with copy
engines, ordered by interprocess events) — the same code that moves planes
over NVLink between GPUs.  The ghost planes are poisoned before every step,
so only a correct exchange reproduces the oracle of the undecomposed grid.

* ranks launched by torchrun (the driver's N > 1 launch) and by a plain
  spawner (no torch anywhere: the rendezvous is ``ProcessGroup``);
* ``bench.py --gpus 2`` with no launcher spawns its own ranks and prints one
  JSON line (rank 0) with ``n_gpus: 2``; both arms.
"""

import json
import os
import re
import socket
import subprocess
import sys
import time
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(nproc, *args, timeout=900):
    env = dict(os.environ, KL_DEVICE_ORDINAL="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), *args]
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def _spawn(nproc, *args, timeout=900):
    """N plain processes (no torch): RANK/WORLD_SIZE + a shared group name."""
    group = f"/klb_test_{os.getpid()}_{time.time_ns()}"
    procs = []
    for r in range(nproc):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(nproc), LOCAL_RANK=str(r), KLB_GROUP=group,
                   KL_DEVICE_ORDINAL="0")
        procs.append(subprocess.Popen([sys.executable, *args], cwd=ROOT, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=timeout) for p in procs]
    return [p.returncode for p in procs], "".join(o for o, _ in outs), "".join(e for _, e in outs)


@pytest.mark.parametrize("kernel,precision,grid,nproc", [("diff_uvw", "fp32", "64,40,30", 2),
                                                         ("advec_u", "fp64", "48,32,40", 3)])
def test_ranks_under_torchrun_match_oracle(kernel, precision, grid, nproc):
    out = _torchrun(nproc, "tests/multiproc_slab_check.py", kernel, precision, grid)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    # torchrun multiplexes the ranks' stdout (lines may run together)
    assert len(re.findall(r"rank \d+ ok ", out.stdout)) == nproc, out.stdout
    assert "FAIL" not in out.stdout


@pytest.mark.parametrize("kernel,precision,grid,nproc", [("diff_uvw", "fp64", "40,24,36", 3),
                                                         ("advec_u", "fp32", "64,48,50", 4),
                                                         ("evisc_smag", "fp32", "32,32,24", 2)])
def test_spawned_ranks_without_torch_match_oracle(kernel, precision, grid, nproc):
    codes, out, err = _spawn(nproc, "tests/multiproc_slab_check.py", kernel, precision, grid)
    assert codes == [0] * nproc, out[-2000:] + err[-3000:]
    assert len(re.findall(r"rank \d+ ok ", out)) == nproc and "FAIL" not in out, out


@pytest.mark.parametrize("kernel,precision,grid,nproc,shared", [("diff_uvw", "fp32", "64,40,30", 3, False),
                                                                ("diff_uvw", "fp64", "40,24,36", 2, False),
                                                                ("diff_uvw", "fp32", "48,32,20", 2, True),
                                                                ("advec_u", "fp32", "64,48,40", 3, False),
                                                                ("advec_u", "fp64", "48,32,30", 2, True),
                                                                # the RK3 time loop, 4 substeps (multiproc_slab_check)
                                                                ("diff_uvw_rk3", "fp32", "48,40,31", 3, False),
                                                                ("diff_uvw_rk3", "fp64", "40,32,24", 2, False)])
def test_fused_peer_halo_ranks_match_oracle(kernel, precision, grid, nproc, shared):
    """diff_uvw / advec_u with the z-halo fused into the kernel: one launch per rank
    over its whole slab, the planes outside the slab read through CUDA-IPC
    mappings of the neighbours' fields (the local ghost planes are poisoned
    and never read).  ``shared``: an exchange-mode driver on the same
    exchanger is stepped and closed first — its close must leave the fused
    driver's peer mappings in place."""
    env = {"KL_HALO_TRANSPORT": "fused", **({"KL_CHECK_SHARED": "1"} if shared else {})}
    os.environ.update(env)
    try:
        codes, out, err = _spawn(nproc, "tests/multiproc_slab_check.py", kernel, precision, grid)
    finally:
        for k in env:
            del os.environ[k]
    assert codes == [0] * nproc, out[-2000:] + err[-3000:]
    assert len(re.findall(r"rank \d+ ok ", out)) == nproc and "FAIL" not in out, out


def test_ipc_probe_agrees_across_ranks():
    """IpcExchanger.probe: every rank maps its neighbours' memory, reads a
    marker value through the mapping and opens their interprocess events —
    the check bench.py runs (KL_HALO_TRANSPORT=auto) before choosing IPC."""
    codes, out, err = _spawn(3, "tests/multiproc_slab_check.py", "probe")
    assert codes == [0, 0, 0], out[-2000:] + err[-3000:]
    assert len(re.findall(r"rank \d ok probe", out)) == 3, out


def _lines(stdout):
    return [json.loads(x) for x in stdout.splitlines() if x.startswith("{")]


def test_bench_spawns_its_own_ranks():
    """``python bench.py --gpus 2`` (how the driver runs BENCH) starts two ranks
    itself; rank 0 prints the only line, for both arms."""
    env = dict(os.environ, KL_DEVICE_ORDINAL="0")
    common = ["--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "diff_uvw_fp32_256"]
    out = subprocess.run([sys.executable, "bench.py", *common, "--e2e-steps", "1", "--e2e-chunks", "4"], cwd=ROOT,
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    lines = _lines(out.stdout)
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["decomposition"] == "z-slab x2"
    assert line["halo_transport"] == "ipc" and "comm nranks=2" in out.stderr
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    ref = subprocess.run([sys.executable, "bench.py", *common, "--impl", "reference"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert ref.returncode == 0, ref.stdout[-2000:] + ref.stderr[-2000:]
    lines = _lines(ref.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["value"] > 0
    assert lines[0]["config"] == line["config"]  # the driver matches the arms by config


def test_bench_under_torchrun_prints_one_line():
    out = _torchrun(2, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload",
                    "advec_u_fp32_256x256x96", "--e2e-steps", "0")
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    lines = _lines(out.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0, out.stdout
