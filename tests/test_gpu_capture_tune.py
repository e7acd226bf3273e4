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
