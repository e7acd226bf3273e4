"""``WisdomKernel.launch``'s memoised derivations (problem size, cache key,
geometry keyed on the scalar arguments) must give exactly what a fresh
derivation gives: different scalars -> different problem/geometry, the same
scalars -> a cache hit with the same geometry (reference dispatch.py:158-204
semantics: one LaunchReport per call, first launch per key compiles)."""

from paper_2303_12374_b200.backend import DeviceIdent, MockCompiler
from paper_2303_12374_b200.capture import CapturePolicy, ScalarArg
from paper_2303_12374_b200.dispatch import WisdomKernel
from paper_2303_12374_b200.stencils.definitions import ARG_LAYOUT, definition_for
from paper_2303_12374_b200.stencils.layout import GridLayout


def _args(lay, kend):
    from paper_2303_12374_b200.cuda.device import DeviceBuffer

    out, pos = [], 0
    for _, role in ARG_LAYOUT["diff_uvw"]["buffers"]:
        out.append(DeviceBuffer(pos, role, "f32", 4096, 100))
        pos += 1
    vals = dict(dxi=1.0, dyi=1.0, jj=lay.jj, kk=lay.kk, istart=3, jstart=3, kstart=3, iend=3 + lay.itot,
                jend=3 + lay.jtot, kend=kend)
    for n in ARG_LAYOUT["diff_uvw"]["scalars"]:
        out.append(ScalarArg(pos, "f32" if n in ("dxi", "dyi") else "i32", vals[n]))
        pos += 1
    return out


class _Recorder(MockCompiler):
    def __init__(self):
        super().__init__()
        self.geometries = []

    def compile(self, request, device):
        exe = super().compile(request, device)
        rec = self.geometries

        class _Exe(type(exe)):
            def launch(self, geometry, args, **kw):
                rec.append(geometry)
                return 1e-6

        exe.__class__ = _Exe
        return exe


def test_memoised_launch_derivations_match_fresh_ones(tmp_path):
    d = definition_for("diff_uvw", "fp32")
    lay = GridLayout(64, 48, 40, "fp32")
    comp = _Recorder()
    wk = WisdomKernel(d, comp, wisdom_dir=tmp_path, capture_policy=CapturePolicy())
    dev = DeviceIdent("NVIDIA B200", "Blackwell")
    a, b = _args(lay, 43), _args(lay, 23)
    reports = [wk.launch(dev, x) for x in (a, b, a, list(a), b)]
    assert [r.problem for r in reports] == [(64, 48, 40), (64, 48, 20), (64, 48, 40), (64, 48, 40), (64, 48, 20)]
    assert [r.cache_hit for r in reports] == [False, False, True, True, True]
    assert comp.invocations == 2
    g = comp.geometries
    assert g[0] == g[2] == g[3] and g[1] == g[4] and g[0] != g[1]
    env = {f"arg{x.position}": x.value for x in b if isinstance(x, ScalarArg) and x.dtype == "i32"}
    fresh = d.derive_geometry(reports[1].configuration, (64, 48, 20), env)
    assert g[1] == fresh
