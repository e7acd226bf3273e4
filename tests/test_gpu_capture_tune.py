"""Capture -> replay -> wisdom -> runtime selection on the GPU.

1. An application launch through WisdomKernel with KERNEL_LAUNCHER_CAPTURE
   set writes a .klcap holding the PRE-launch device buffers.
2. ``kltune tune cap.klcap --backend cuda`` replays the captured buffers
   across configurations (verify + timed reps) and appends the best to the
   kernel's wisdom file.
3. A fresh WisdomKernel selects that record (match_kind "exact") and its
   launch reproduces the oracle.
"""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_capture_tune_select_round_trip(gpu_ctx, tmp_path, monkeypatch):
    from paper_2303_12374_b200 import cli
    from paper_2303_12374_b200.capture import CapturePolicy, read_capture
    from paper_2303_12374_b200.cuda import NvrtcCompiler
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem
    from paper_2303_12374_b200.wisdom import WisdomFile, wisdom_path
    from stencil_helpers import TOL, oracle_outputs, rel_error

    lay = GridLayout(40, 24, 12, "fp64")
    prob = StencilProblem("advec_u", lay, gpu_ctx)
    comp = NvrtcCompiler(gpu_ctx)
    policy = CapturePolicy(names=frozenset({"advec_u_fp64"}), directory=str(tmp_path))
    wk = WisdomKernel(prob.definition, comp, wisdom_dir=tmp_path, capture_policy=policy)
    wk.launch(gpu_ctx.ident, prob.args())
    gpu_ctx.synchronize()
    cap_path = tmp_path / "advec_u_fp64_40x24x12.klcap"
    cap = read_capture(cap_path)
    assert cap.problem == (40, 24, 12) and len(cap.buffers) == 7
    # the capture holds the pre-launch ut (the launch has since updated it)
    ut_cap = np.frombuffer(cap.buffers[0].data, dtype=np.float64)
    ut_now = prob.fields["ut"].download_array(np.float64)[lay.lead:]
    assert not np.array_equal(ut_cap[: ut_now.size], ut_now)

    (tmp_path / "klconfig.json").write_text(json.dumps({"backend": "cuda", "repetitions": 3, "warmup": 1}))
    monkeypatch.chdir(tmp_path)
    rc = cli.main(["tune", str(cap_path), "--strategy", "random", "--budget-evals", "6", "--seed", "3",
                   "--wisdom", str(tmp_path)])
    assert rc == 0
    wfile = WisdomFile.load(wisdom_path(tmp_path, prob.definition.kernel_key()))
    rec = wfile.records[0]
    assert rec.device.name == gpu_ctx.ident.name and rec.problem == (40, 24, 12)

    prob.regenerate()
    fresh = WisdomKernel(prob.definition, comp, wisdom_dir=tmp_path, capture_policy=CapturePolicy())
    report = fresh.launch(gpu_ctx.ident, prob.args())
    gpu_ctx.synchronize()
    assert report.match_kind == "exact" and report.configuration == rec.config
    ref, _ = oracle_outputs("advec_u", lay)
    assert rel_error(prob.download("ut"), ref["ut"], lay) <= TOL["fp64"]
    prob.close()


def test_device_crc32_matches_zlib(gpu_ctx):
    """klb_crc32_device (per-chunk GPU CRC registers chained on the host) equals
    zlib.crc32 for any length and alignment (chunk = 4096 B, 4-byte fast path)."""
    import zlib

    from paper_2303_12374_b200.cuda import DeviceArray
    from paper_2303_12374_b200.cuda.capture_device import device_crc32

    rng = np.random.default_rng(7)
    data = rng.integers(0, 256, size=(6 << 20) + 64, dtype=np.uint8).tobytes()
    arr = DeviceArray(len(data))
    arr.upload(data, stream=gpu_ctx.stream)
    gpu_ctx.synchronize()
    try:
        for n, off in ((0, 0), (1, 0), (7, 1), (8, 4), (4095, 3), (4096, 0), (4097, 4), (12288, 8), (100003, 2),
                       ((5 << 20) + 13, 0), ((6 << 20) + 1, 63)):
            assert device_crc32(arr.ptr + off, n) == zlib.crc32(data[off:off + n]) & 0xFFFFFFFF, (n, off)
    finally:
        arr.free()


def test_device_capture_is_byte_identical_to_host_capture(gpu_ctx, tmp_path):
    """write_capture_device (device CRCs, chunked pinned download) writes the
    same bytes as the reference-layout host writer, and read_capture's zlib
    check accepts them."""
    from paper_2303_12374_b200.capture import capture_from_args, read_capture, serialize_capture
    from paper_2303_12374_b200.cuda.capture_device import write_capture_device
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    lay = GridLayout(37, 21, 9, "fp32")
    prob = StencilProblem("diff_uvw", lay, gpu_ctx)
    try:
        args = prob.args()
        host = serialize_capture(capture_from_args(prob.definition, args, "app", "t0"))
        path = write_capture_device(prob.definition, args, tmp_path / "dev.klcap", application="app", timestamp="t0",
                                    chunk=4096)
        assert path.read_bytes() == host
        cap = read_capture(path)
        assert cap.problem == (37, 21, 9) and len(cap.buffers) == 11
    finally:
        prob.close()


def test_isolated_executor_survives_a_sticky_error(gpu_ctx, tmp_path):
    """A configuration that traps poisons a CUDA context; the isolated executor
    reports it launch_failed and measures the next configuration in a fresh
    worker (the reference tuner never aborts on a failing configuration)."""
    from paper_2303_12374_b200.backend import STATUS_LAUNCH_FAILED, STATUS_OK
    from paper_2303_12374_b200.capture import BufferArg, Capture, ScalarArg, write_capture
    from paper_2303_12374_b200.cuda.isolated import IsolatedReplayExecutor
    from paper_2303_12374_b200.kerneldef import KernelDefinition
    from paper_2303_12374_b200.space import ConfigSpace, TunableParam

    src = """extern "C" __global__ void trapk(float* x, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (TRAP) __trap();
  if (i < n) x[i] += 1.0f;
}
"""
    space = ConfigSpace([TunableParam("block", (32, 64), 32), TunableParam("trap", (0, 1), 0)])
    d = KernelDefinition("trapk", space, source_text=src, problem_size=("arg1",), block=("block", 1, 1),
                         grid=("ceil_div(problem_x, block)", 1, 1), defines=[("TRAP", "trap")])
    n = 4096
    cap = Capture(d, (n,), scalars=[ScalarArg(1, "i32", n)],
                  buffers=[BufferArg(0, "output", "f32", np.zeros(n, np.float32).tobytes())])
    path = tmp_path / "trapk.klcap"
    write_capture(cap, path)
    ex = IsolatedReplayExecutor({"capture": str(path)}, repetitions=3, warmup=1, timeout=120)
    try:
        assert ex.measure({"block": 64, "trap": 0}).status == STATUS_OK
        assert ex.measure({"block": 32, "trap": 1}).status == STATUS_LAUNCH_FAILED
        m = ex.measure({"block": 32, "trap": 0})
        assert m.status == STATUS_OK and ex.restarts == 1
        assert ex.describe()["isolated"] and ex.problem == (n,)
    finally:
        ex.close()


def test_capture_is_ordered_after_work_on_the_launch_stream(gpu_ctx, tmp_path):
    """Chained kernels on one non-blocking stream (evisc_smag producing evisc,
    then a captured diff_uvw reading it, no host sync in between): the device
    capture runs on the launch stream, so it holds evisc as evisc_smag wrote
    it, and its CRCs verify."""
    from paper_2303_12374_b200.capture import CapturePolicy, read_capture
    from paper_2303_12374_b200.cuda import NvrtcCompiler
    from paper_2303_12374_b200.dispatch import WisdomKernel
    from paper_2303_12374_b200.stencils.layout import GridLayout
    from paper_2303_12374_b200.stencils.problem import StencilProblem

    lay = GridLayout(256, 256, 256, "fp32")
    smag = StencilProblem("evisc_smag", lay, gpu_ctx)
    diff = StencilProblem("diff_uvw", lay, gpu_ctx)
    diff.share_fields(smag, ("evisc", "u", "v", "w"))
    comp = NvrtcCompiler(gpu_ctx)
    try:
        wk_smag = WisdomKernel(smag.definition, comp, wisdom_dir=tmp_path, capture_policy=CapturePolicy())
        wk_diff = WisdomKernel(diff.definition, comp, wisdom_dir=tmp_path,
                               capture_policy=CapturePolicy(names=frozenset({"diff_uvw_fp32"}),
                                                            directory=str(tmp_path)))
        # compile both first so the chained launches are back to back
        wk_smag.bind(gpu_ctx.ident, smag.args(), stream=gpu_ctx.stream)
        wk_diff.resolve(gpu_ctx.ident, diff.definition.derive_problem_size(diff.scalar_env()), diff.scalar_env())
        gpu_ctx.synchronize()
        smag.regenerate()
        wk_smag.launch(gpu_ctx.ident, smag.args(), stream=gpu_ctx.stream)
        wk_diff.launch(gpu_ctx.ident, diff.args(), stream=gpu_ctx.stream)
        gpu_ctx.synchronize()
        cap = read_capture(tmp_path / "diff_uvw_fp32_256x256x256.klcap")  # CRCs checked
        from paper_2303_12374_b200.stencils.definitions import ARG_LAYOUT

        pos = [n for n, _ in ARG_LAYOUT["diff_uvw"]["buffers"]].index("evisc")
        got = np.frombuffer(next(b for b in cap.buffers if b.position == pos).data, dtype=np.float32)
        want = smag.fields["evisc"].download_array(np.float32)[lay.lead:]
        assert np.array_equal(got, want[: got.size])
    finally:
        diff.close()
        smag.close()


_STREAM_CHILD = r"""
import json, resource, sys
sys.path.insert(0, sys.argv[1])
from pathlib import Path
from paper_2303_12374_b200 import cli
from paper_2303_12374_b200.capture import CapturePolicy, read_capture_info
from paper_2303_12374_b200.cuda import NvrtcCompiler, open_device
from paper_2303_12374_b200.cuda.executor import CudaReplayExecutor
from paper_2303_12374_b200.dispatch import WisdomKernel
from paper_2303_12374_b200.stencils.layout import GridLayout
from paper_2303_12374_b200.stencils.problem import StencilProblem

out = Path(sys.argv[2])
ctx = open_device(0)
lay = GridLayout(512, 512, 512, "fp32")
prob = StencilProblem("diff_uvw", lay, ctx)
ptr_mod = prob.field_ptr("ut") % 128
wk = WisdomKernel(prob.definition, NvrtcCompiler(ctx), wisdom_dir=out,
                  capture_policy=CapturePolicy(names=frozenset({"diff_uvw_fp32"}), directory=str(out)))
wk.launch(ctx.ident, prob.args(), stream=ctx.stream)
ctx.synchronize()
prob.close()
cap = out / "diff_uvw_fp32_512x512x512.klcap"
info = read_capture_info(cap)
def status(key):
    for line in open("/proc/self/status"):
        if line.startswith(key + ":"):
            return int(line.split()[1]) * 1024


# peak resident memory of the upload alone (NVRTC compiles elsewhere in the
# process use hundreds of MB): reset the high-water mark, stream, read it back
with open("/proc/self/clear_refs", "w") as fh:
    fh.write("5")
base = status("VmRSS")
ex = CudaReplayExecutor.from_file(cap, ctx, repetitions=2, warmup=1, chunk=32 << 20, verify=False)
upload_peak = status("VmHWM") - base
mods = [b.ptr % 128 for b in ex.args if hasattr(b, "ptr")]
staging = ex.host_staging_bytes
ex.close()
(out / "klconfig.json").write_text(json.dumps({"backend": "cuda", "repetitions": 2, "warmup": 1}))
import os
os.chdir(out)
rc = cli.main(["tune", str(cap), "--strategy", "random", "--budget-evals", "2", "--seed", "1", "--wisdom", str(out)])
print(json.dumps({"rc": rc, "capture_bytes": cap.stat().st_size, "upload_peak_rss": upload_peak,
                  "maxrss_kb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss,
                  "ptr_mod": ptr_mod, "replay_mods": mods, "address_mods": [b.get("address_mod128") for b in info["buffers"]],
                  "staging": staging}))
"""


def test_streaming_replay_of_a_multi_gb_capture(tmp_path):
    """A 4.1 GB capture (diff_uvw fp32 512^3, seven 584 MB fields) is written
    from HBM, replayed with ``CudaReplayExecutor.from_file`` and tuned with
    ``kltune tune --backend cuda``, with the process's peak host RSS far below
    the capture size and the upload's own peak at the two pinned staging
    chunks (payloads stream through them, CRCs checked on the way), and every replay buffer placed at the original
    pointer's alignment mod 128 (the application's row alignment)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    res = subprocess.run([sys.executable, "-c", _STREAM_CHILD, str(root), str(tmp_path)], capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    print(out)
    assert out["rc"] == 0
    assert out["capture_bytes"] > 4_000_000_000
    # the upload's resident-memory peak is the staging chunks, not the payloads
    assert out["upload_peak_rss"] < out["staging"] + (256 << 20), out
    assert out["maxrss_kb"] * 1024 < out["capture_bytes"], out  # whole process, NVRTC included
    # fields sit at lead*4 = 116 mod 128 (rows 128-byte aligned); profiles at 0
    assert out["address_mods"].count(out["ptr_mod"]) == 7 and out["ptr_mod"] == 116
    assert out["replay_mods"] == out["address_mods"]


def test_autotune_checkpoint_resume_on_gpu(gpu_ctx, tmp_path):
    """A B200 tuning session streamed to disk (checkpoint) and continued
    (resume): the continuation keeps the recorded measurements of the first
    run and measures only the new proposals (SURVEY §5 checkpoint/resume)."""
    from paper_2303_12374_b200.autotune import tune_problem
    from paper_2303_12374_b200.tuner import Budget, load_session

    kw = dict(strategy="random", seed=5, wisdom_dir=None, session_dir=tmp_path, repetitions=3, warmup=1,
              family="TMA", log=lambda *a: None)
    first, _ = tune_problem("advec_u", "fp32", (64, 48, 40), gpu_ctx, budget=Budget(3, None), checkpoint=True, **kw)
    (path,) = list(tmp_path.glob("*.klsession"))
    seen = []
    kw["log"] = seen.append
    second, _ = tune_problem("advec_u", "fp32", (64, 48, 40), gpu_ctx, budget=Budget(6, None), resume=True, **kw)
    assert any("resuming" in str(x) for x in seen)
    assert len(second.evaluations) == 6
    for a, b in zip(first.evaluations, second.evaluations[:3]):
        assert a.config == b.config and a.measurement.objective == b.measurement.objective
    assert len(load_session(path).evaluations) == 6
