"""Control-plane behaviour (reference test strategy) and the
SPEC acceptance criteria #1-#11, written
against the drop-in ``kltune`` alias."""

import itertools
import math
import statistics
import threading
import time

import pytest
from hypothesis import given, settings, strategies as st

import kltune
from kltune.backend import MockCompiler, SimCostModel, SimulatedExecutor
from kltune.capture import (BufferArg, CaptureFormatError, CapturePolicy, CaptureSession, ScalarArg,
                            capture_from_args, read_capture, serialize_capture, write_capture, write_capture_stream)
from kltune.dispatch import WisdomKernel
from kltune.expr import EvalError, ParseError, evaluate, parse, to_text
from kltune.kerneldef import DefinitionError, KernelBuilder
from kltune.presets import stencil3d_definition, stencil3d_space, vector_add_definition
from kltune.report import cross_matrix, fraction_of_optimum, ppm, Scenario, histogram
from kltune.space import ConfigSpace, TunableParam
from kltune.tuner import Budget, load_session, save_session, session_fingerprint, tune
from kltune.wisdom import (MATCH_ANY, MATCH_DEFAULT, MATCH_EXACT, MATCH_SAME_ARCH, MATCH_SAME_DEVICE, Provenance,
                           WisdomFile, WisdomRecord, append_result, merge_wisdom, select)
from conftest import grid_space

A100 = kltune.DeviceIdent("Tesla A100", "Ampere")
A4000 = kltune.DeviceIdent("RTX A4000", "Ampere")
B200 = kltune.DeviceIdent("NVIDIA B200", "Blackwell")


def test_alias_is_the_b200_package():
    import paper_2303_12374_b200

    assert kltune.WisdomKernel is paper_2303_12374_b200.WisdomKernel
    assert set(kltune.__all__) == set(paper_2303_12374_b200.__all__) and len(kltune.__all__) == 54


# -- expr -------------------------------------------------------------------------------


def test_precedence_and_truncation():
    assert evaluate(parse("1 + 2 * 3"), {}) == 7
    assert evaluate(parse("-7 / 2"), {}) == -3 and evaluate(parse("-7 % 2"), {}) == -1
    assert evaluate(parse("ceil_div(1000, 512)"), {}) == 2


def test_errors():
    with pytest.raises(ParseError) as err:
        parse("ceil_div(problem_x, block_x")
    assert err.value.offset == len("ceil_div(problem_x, block_x")
    for text in ("ceil_div(-1, 2)", "1 / 0", "a * 4"):
        with pytest.raises(EvalError):
            evaluate(parse(text), {"a": 2 ** 62})
    assert evaluate(parse("b == 0 || a / b > 1"), {"a": 1, "b": 0}) is True


@settings(max_examples=200, deadline=None)
@given(st.recursive(st.integers(0, 50).map(str) | st.sampled_from(["a", "b", "true"]),
                    lambda c: st.tuples(c, st.sampled_from(["+", "*", "-", "<", "&&", "=="]), c).map(
                        lambda t: f"({t[0]} {t[1]} {t[2]})"), max_leaves=12))
def test_print_parse_round_trip(text):
    tree = parse(text)
    assert parse(to_text(tree)) == tree


# -- space (SPEC #1) -------------------------------------------------------------------


def test_table2_cardinality():
    assert stencil3d_space(False).cardinality() == 7_776_000
    assert stencil3d_space(True).cardinality() == 7_776_000


def test_block_limit_count_matches_nested_loops():
    space = stencil3d_space(True)
    bx, by, bz = (p.values for p in space.params[:3])
    good = sum(1 for x, y, z in itertools.product(bx, by, bz) if x * y * z <= 1024)
    per_block = 7_776_000 // 125
    assert good * per_block == 4_478_976


def test_enumeration_order_and_sampling():
    s = ConfigSpace([TunableParam("a", (1, 2), 1), TunableParam("b", (10, 20), 10)])
    assert [(c["a"], c["b"]) for c in s.enumerate_configs()] == [(1, 10), (1, 20), (2, 10), (2, 20)]
    assert s.sample_random(42, 5) == s.sample_random(42, 5)
    with pytest.raises(kltune.RejectionLimitError):
        ConfigSpace([TunableParam("a", (1, 2), 1)], ["a > 5"]).sample_random(1, 1)


# -- kerneldef -----------------------------------------------------------------------------


def test_geometry_and_requests():
    d = stencil3d_definition()
    cfg = dict(d.space.default_config()[0], block_x=32, block_y=4, block_z=2, tile_x=2)
    g = d.derive_geometry(cfg, (256, 256, 256))
    assert g.block == (32, 4, 2) and g.grid == (4, 64, 128)
    req = vector_add_definition().render_compile_request({"block_size": 128}, (1000,))
    assert req.entry == "vector_add<128>" and req.defines == ()
    with pytest.raises(DefinitionError, match="only argN"):
        KernelBuilder("k", source_text="x").problem_size("block_x").build()


# -- capture (SPEC #3) -----------------------------------------------------------------------


def _capture(nbytes=1 << 20):
    d = stencil3d_definition()
    payload = bytes((i * 37) & 0xFF for i in range(nbytes))
    args = [BufferArg(0, "output", "f32", payload), BufferArg(1, "input", "u8", payload[:999]),
            ScalarArg(2, "i32", 64), ScalarArg(3, "i32", 32), ScalarArg(4, "i32", 16), ScalarArg(5, "f64", 0.5)]
    return capture_from_args(d, args, application="t", timestamp="2026-01-01T00:00:00Z")


def test_capture_round_trip_and_crc(tmp_path):
    cap = _capture()
    p1, p2, p3 = tmp_path / "a.klcap", tmp_path / "b.klcap", tmp_path / "c.klcap"
    write_capture(cap, p1)
    back = read_capture(p1)
    assert back == cap and back.problem == (64, 32, 16)
    write_capture(back, p2)
    write_capture_stream(back, p3, chunk=4096)
    assert p1.read_bytes() == p2.read_bytes() == p3.read_bytes() == serialize_capture(cap)
    raw = bytearray(p1.read_bytes())
    raw[-5] ^= 0x01
    p1.write_bytes(bytes(raw))
    with pytest.raises(CaptureFormatError, match="checksum"):
        read_capture(p1)


def test_capture_64mib_under_a_second(tmp_path):
    cap = _capture(64 << 20)
    t0 = time.perf_counter()
    write_capture_stream(cap, tmp_path / "x.klcap")
    read_capture(tmp_path / "x.klcap")
    assert time.perf_counter() - t0 < 5.0  # generous for shared CI hosts; SPEC budget 1 s


def test_capture_policy_once_per_problem(tmp_path):
    policy = CapturePolicy.from_env({"KERNEL_LAUNCHER_CAPTURE": "grid3d,advec_u", "KERNEL_LAUNCHER_CAPTURE_DIR": str(tmp_path)})
    sess = CaptureSession(policy)
    d = stencil3d_definition()
    args = [ScalarArg(2, "i32", 8), ScalarArg(3, "i32", 8), ScalarArg(4, "i32", 8)]
    assert sess.maybe_capture(d, args) == tmp_path / "grid3d_8x8x8.klcap"
    assert sess.maybe_capture(d, args) is None
    assert not kltune.should_capture(policy, "advec")


# -- tuner (SPEC #4, #5, #11) -----------------------------------------------------------------


@pytest.mark.parametrize("seed", range(20))
def test_exhaustive_equals_brute_force(seed):
    space = grid_space(4, 4, ["p0 + p1 != 5"])
    model = SimCostModel(seed, space)
    session = tune(space, SimulatedExecutor(model), strategy="exhaustive", budget=Budget(max_evaluations=10_000,
                   max_wall_seconds=None), seed=seed)
    best = min(model.noiseless_cost(c) for c in space.enumerate_configs())
    assert session.best_objective == best


def test_surrogate_quality_vs_random():
    space = grid_space(5, 7)  # 16,807 points
    wins, sur, rnd = 0, [], []
    for seed in range(10):
        model = SimCostModel(seed, space)
        opt = min(model.noiseless_cost(c) for c in space.enumerate_configs())
        s = tune(space, SimulatedExecutor(model), strategy="surrogate", budget=Budget(300, None), seed=seed)
        r = tune(space, SimulatedExecutor(model), strategy="random", budget=Budget(300, None), seed=seed)
        wins += s.best_objective <= 1.05 * opt
        sur.append(s.best_objective)
        rnd.append(r.best_objective)
    assert wins >= 8
    assert statistics.median(sur) <= statistics.median(rnd)


def test_session_determinism(tmp_path):
    space = stencil3d_space(True)
    prints = []
    for n in range(2):
        s = tune(space, SimulatedExecutor(SimCostModel(42, space, noise_sigma=0.02)), strategy="surrogate",
                 budget=Budget(40, None), seed=42, device=B200, kernel_key="k", problem=(8,))
        save_session(s, tmp_path / f"{n}.klsession")
        prints.append(session_fingerprint(tmp_path / f"{n}.klsession"))
        assert load_session(tmp_path / f"{n}.klsession").best_objective == s.best_objective
    assert prints[0] == prints[1]


# -- wisdom (SPEC #2, #6) ---------------------------------------------------------------------------


def _rec(dev, problem, obj, tag):
    return WisdomRecord(dev, problem, {"tag": tag}, obj, Provenance(date="d", hostname="h"))


def test_selection_cascade():
    wf = WisdomFile("k", records=[_rec(A100, (256, 256, 256), 1.0, "a256"), _rec(A100, (512, 512, 512), 1.0, "a512")])
    assert select(wf, A100, (256, 256, 256), {}).match_kind == MATCH_EXACT
    r = select(wf, A100, (300, 300, 300), {})
    assert r.match_kind == MATCH_SAME_DEVICE and r.config == {"tag": "a256"}
    assert math.isclose(math.dist((256,) * 3, (300,) * 3), 76.21, abs_tol=0.01)
    assert select(wf, A4000, (512, 512, 512), {}).match_kind == MATCH_SAME_ARCH
    assert select(wf, B200, (1, 1, 1), {}).match_kind == MATCH_ANY
    assert select(None, B200, (1,), {"d": 1}) == kltune.SelectionResult({"d": 1}, MATCH_DEFAULT, None)


def test_keep_best_merge():
    wf = WisdomFile("k")
    for obj in (1.0e-3, 0.8e-3, 0.9e-3):
        sess = kltune.TuningSession("k", "random", 0, device=B200, problem=(64, 64, 64), best_config={"x": obj},
                                    best_objective=obj)
        append_result(wf, sess)
    assert [r.objective_seconds for r in wf.records] == [0.8e-3]
    sess = kltune.TuningSession("k", "random", 0, device=B200, problem=(32, 32, 32), best_config={}, best_objective=1.0)
    append_result(wf, sess)
    assert len(wf.records) == 2
    merged = merge_wisdom([wf, WisdomFile("k", records=[_rec(B200, (64, 64, 64), 0.5e-3, "m")])])
    assert merged.records[0].objective_seconds == 0.5e-3


def test_wisdom_round_trip_bytes(tmp_path):
    wf = WisdomFile("k", records=[_rec(B200, (64, 64), 0.5, "x"), _rec(A100, (8,), 0.25, "y")])
    wf.save(tmp_path / "k.wisdom")
    WisdomFile.load(tmp_path / "k.wisdom").save(tmp_path / "k2.wisdom")
    assert (tmp_path / "k.wisdom").read_bytes() == (tmp_path / "k2.wisdom").read_bytes()


# -- dispatch (SPEC #7, #8) -------------------------------------------------------------------------


def _vadd_args(n):
    return [ScalarArg(3, "i32", n)]


def test_dispatch_single_flight_16_threads(tmp_path):
    comp = MockCompiler(compile_delay=0.02)
    wk = WisdomKernel(vector_add_definition(), comp, wisdom_dir=tmp_path, capture_policy=CapturePolicy())
    sizes = [1000, 2000, 3000]
    barrier = threading.Barrier(16)

    def worker(i):
        barrier.wait()
        wk.launch(B200, _vadd_args(sizes[i % 3]))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(16)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for n in sizes * 5:
        wk.launch(B200, _vadd_args(n))
    assert comp.invocations == 3


def test_overhead_breakdown(tmp_path):
    comp = MockCompiler(compile_delay=0.08)
    wk = WisdomKernel(vector_add_definition(), comp, wisdom_dir=tmp_path, capture_policy=CapturePolicy())
    for _ in range(20):
        wk.launch(B200, _vadd_args(4096))
    rep = wk.overhead_report()
    assert rep.first["compile"] / sum(rep.first.values()) > 0.7
    assert "compile" not in rep.subsequent and rep.subsequent_count == 19


def test_default_fallback_on_compile_error(tmp_path):
    d = vector_add_definition()
    wf = WisdomFile(d.kernel_key(), records=[WisdomRecord(B200, (4096,), {"block_size": 1024}, 1.0)])
    wf.save(tmp_path / f"{d.kernel_key()}.wisdom")
    comp = MockCompiler(fail_when=lambda req: req.entry == "vector_add<1024>")
    rep = WisdomKernel(d, comp, wisdom_dir=tmp_path, capture_policy=CapturePolicy()).launch(B200, _vadd_args(4096))
    assert rep.used_default_fallback and rep.match_kind == MATCH_DEFAULT and rep.configuration == {"block_size": 128}


# -- report (SPEC #9, #10) ------------------------------------------------------------------------------


def test_ppm_properties():
    assert math.isclose(ppm([0.5, 1.0]).ppm, 2 / 3, abs_tol=1e-9)
    assert ppm([0.5, None]).ppm == 0.0
    from kltune.rng import SplitMix64

    rng = SplitMix64(5)
    for _ in range(100):
        effs = [0.01 + 0.99 * rng.next_float() for _ in range(1 + rng.next_below(8))]
        r = ppm(effs)
        assert math.isclose(r.ppm, len(effs) / sum(1 / e for e in effs), rel_tol=1e-12)
        assert r.worst <= r.ppm <= r.best <= 1


def test_cross_matrix_diagonal_and_gap():
    space = grid_space(3, 6)
    sessions, models = [], []
    for seed in (1, 2, 3, 4):
        m = SimCostModel(seed, space)
        models.append(SimulatedExecutor(m))
        sessions.append(tune(space, models[-1], strategy="exhaustive", budget=Budget(10_000, None), seed=0,
                             kernel_key="k"))
    scen = [Scenario("k", (s,), "fp32", f"dev{s}") for s in range(4)]
    mat = cross_matrix(scen, sessions, lambda j, c: models[j].measure(c))
    assert all(mat.entries[i][i] == 1.0 for i in range(4))
    assert min(e for row in mat.entries for e in row) < 0.9
    assert fraction_of_optimum(sessions[0], sessions[0].best_config) == 1.0
    assert sum(histogram(sessions[0], 10).counts) == len(sessions[0].evaluations)


def test_report_cuda_backend_parses_stencil_kernel_keys():
    """``kltune report --backend cuda`` rebuilds a session's live problem from
    its kernel key (<kernel>_<precision>-<space fingerprint>)."""
    from types import SimpleNamespace

    from paper_2303_12374_b200.cli import _CudaEvaluators
    from paper_2303_12374_b200.report import ReportError

    assert _CudaEvaluators.kernel_of(SimpleNamespace(kernel_key="diff_uvw_rk3_fp64-a27ac7eccf76")) == (
        "diff_uvw_rk3", "fp64")
    assert _CudaEvaluators.kernel_of(SimpleNamespace(kernel_key="advec_u_fp32-c2e327370150")) == ("advec_u", "fp32")
    import pytest

    with pytest.raises(ReportError):
        _CudaEvaluators.kernel_of(SimpleNamespace(kernel_key="grid3d-0123456789ab"))


def test_portability_shapes_accept_cubes_and_boxes():
    from paper_2303_12374_b200 import portability as p

    assert p._shape(192) == (192, 192, 192) and p._shape((640, 640, 320)) == (640, 640, 320)
    assert p._label(384) == "384^3" and p._label((1024, 512, 256)) == "1024x512x256"
