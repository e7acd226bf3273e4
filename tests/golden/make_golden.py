"""Generate golden fixtures for the control-plane parity tests FROM THE REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only under the alias ``kltune_ref``
(SURVEY.md §4 recipe), drives it with deterministic inputs and writes
``tests/golden/control_plane.json``.  tests/test_golden.py replays the same
inputs through paper_2303_12374_b200 and demands identical outputs — so the
fixtures pin our implementation to the reference's behaviour even on hosts
(the GPU box) where the reference is absent.
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg/src/kltune")
OUT = Path(__file__).resolve().parent / "control_plane.json"


def load_reference():
    spec = importlib.util.spec_from_file_location("kltune_ref", REF / "__init__.py",
                                                  submodule_search_locations=[str(REF)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["kltune_ref"] = mod
    spec.loader.exec_module(mod)
    for sub in ("presets", "util", "rng", "expr", "space", "kerneldef", "capture", "backend", "tuner", "wisdom",
                "report"):
        importlib.import_module(f"kltune_ref.{sub}")
    return mod


EXPRESSIONS = [
    ("1 + 2 * 3", {}), ("(1 + 2) * 3", {}), ("-7 / 2", {}), ("-7 % 2", {}), ("7 % -2", {}), ("ceil_div(1000, 512)", {}),
    ("block_x * block_y * block_z <= 1024", {"block_x": 256, "block_y": 4, "block_z": 2}),
    ('unravel == "XYZ" || tile_z > 1', {"unravel": "ZYX", "tile_z": 4}), ("min(a, b) - max(a, -b)", {"a": 3, "b": -9}),
    ("a / b", {"a": -(2 ** 63), "b": -1}), ("a + 1", {"a": 2 ** 63 - 1}), ("1 / 0", {}), ("1 % 0", {}),
    ("ceil_div(-1, 2)", {}), ("b == 0 || a / b > 1", {"a": 1, "b": 0}), ("!true && 1 / 0 == 1", {}),
    ("1 < 2 < 3", {}), ("tile_x", {}), ('"a" < "b"', {}), ("- - 5", {}), ("!(a > 1) || !(b < 2)", {"a": 2, "b": 1}),
    ("ceil_div(problem_x, block_x * tile_x) * ceil_div(problem_y, block_y * tile_y)",
     {"problem_x": 1000, "problem_y": 77, "block_x": 64, "tile_x": 4, "block_y": 2, "tile_y": 2}),
]
BAD_SYNTAX = ["ceil_div(problem_x, block_x", "1 +", "foo(1)", "min(1)", '"abc', "3 $ 4", "99999999999999999999",
              "(1))", ""]


def expr_cases(ref):
    xp = ref.expr
    out = []
    for text, env in EXPRESSIONS:
        tree = xp.parse(text)
        try:
            res = {"value": xp.evaluate(tree, env)}
        except xp.EvalError as e:
            res = {"error": "EvalError", "message": str(e)}
        out.append({"text": text, "env": env, "printed": xp.to_text(tree), **res})
    bad = []
    for text in BAD_SYNTAX:
        try:
            xp.parse(text)
            bad.append({"text": text, "ok": True})
        except xp.ParseError as e:
            bad.append({"text": text, "offset": e.offset, "message": str(e)})
    return {"evaluate": out, "parse_errors": bad}


def space_cases(ref):
    presets, space_mod = ref.presets, ref.space
    s_lim, s_raw = presets.stencil3d_space(True), presets.stencil3d_space(False)
    small = space_mod.ConfigSpace([space_mod.TunableParam("a", (1, 2, 3), 2), space_mod.TunableParam("b", (10, 20), 10),
                                   space_mod.TunableParam("c", (True, False), False)], ["a * b > 15 || c"])
    enum = list(small.enumerate_configs())
    return {
        "fingerprint_limited": s_lim.fingerprint(), "fingerprint_raw": s_raw.fingerprint(),
        "cardinality": s_raw.cardinality(),
        "default": s_lim.default_config()[0],
        "samples_seed42": s_lim.sample_random(42, 25),
        "samples_seed7_raw": s_raw.sample_random(7, 10),
        "encoding": [s_lim.normalized_encoding(c) for c in s_lim.sample_random(3, 5)],
        "small_enumeration": enum, "small_valid": small.valid_cardinality(),
        "small_fingerprint": small.fingerprint(),
        "first_enumerated": [c for _, c in zip(range(40), s_lim.enumerate_configs())],
        "space_json": s_lim.to_json_obj(),
    }


def kerneldef_cases(ref):
    presets = ref.presets
    d = presets.stencil3d_definition(True)
    v = presets.vector_add_definition()
    geoms = []
    for cfg in d.space.sample_random(11, 30):
        for problem in ((256, 256, 256), (1000, 77, 5), (33, 1024, 512)):
            g = d.derive_geometry(cfg, problem, {})
            req = d.render_compile_request(cfg, problem, {})
            geoms.append({"config": cfg, "problem": list(problem), "block": list(g.block), "grid": list(g.grid),
                          "smem": g.shared_mem_bytes, "entry": req.entry, "defines": list(req.defines)})
    vreq = v.render_compile_request({"block_size": 128}, (1000,), {})
    return {
        "stencil_kernel_key": d.kernel_key(), "vector_kernel_key": v.kernel_key(),
        "stencil_json": ref.util.canonical_dumps(d.to_json_obj()),
        "vector_json": ref.util.canonical_dumps(v.to_json_obj()),
        "geometries": geoms,
        "vector_request": {"entry": vreq.entry, "defines": list(vreq.defines), "flags": list(vreq.flags)},
        "vector_geometry": list(v.derive_geometry({"block_size": 128}, (1000,)).grid),
    }


def _records(ref, seed):
    rng = ref.rng.SplitMix64(seed)
    devices = [ref.backend.DeviceIdent("NVIDIA B200", "Blackwell"), ref.backend.DeviceIdent("Tesla A100", "Ampere"),
               ref.backend.DeviceIdent("RTX A4000", "Ampere"), ref.backend.DeviceIdent("H100", "Hopper")]
    recs = []
    for n in range(rng.next_below(7) + 1):
        dev = devices[rng.next_below(4)]
        dims = rng.next_below(3) + 1
        problem = tuple(16 * (1 + rng.next_below(64)) for _ in range(dims))
        prov = ref.wisdom.Provenance(date="2026-01-01T00:00:00Z", hostname="h", versions={"python": "3"})
        recs.append(ref.wisdom.WisdomRecord(dev, problem, {"block_x": 16 << rng.next_below(5), "n": n},
                                            0.5 + rng.next_below(4) * 0.25, prov))
    return recs


def wisdom_cases(ref):
    cases = []
    for seed in range(60):
        wf = ref.wisdom.WisdomFile("k-abc", records=_records(ref, seed))
        rng = ref.rng.SplitMix64(1000 + seed)
        for q in range(4):
            dev = [("NVIDIA B200", "Blackwell"), ("Tesla A100", "Ampere"), ("GH200", "Hopper"), ("MI300", "CDNA3")][
                rng.next_below(4)]
            dims = rng.next_below(3) + 1
            problem = tuple(16 * (1 + rng.next_below(64)) for _ in range(dims))
            res = ref.wisdom.select(wf, ref.backend.DeviceIdent(*dev), problem, {"default": True})
            idx = None if res.record is None else next(i for i, r in enumerate(wf.records) if r is res.record)
            cases.append({"seed": seed, "device": list(dev), "problem": list(problem), "match_kind": res.match_kind,
                          "record_index": idx, "config": res.config})
    # selection goldens of SPEC.md:449-452
    a100 = ref.backend.DeviceIdent("Tesla A100", "Ampere")
    wf = ref.wisdom.WisdomFile("k", records=[ref.wisdom.WisdomRecord(a100, (256, 256, 256), {"c": 1}, 1.0),
                                             ref.wisdom.WisdomRecord(a100, (512, 512, 512), {"c": 2}, 1.0)])
    with tempfile.TemporaryDirectory() as tmp:
        path = Path(tmp) / "x.wisdom"
        big = ref.wisdom.WisdomFile("k-abc", records=_records(ref, 5))
        big.save(path)
        blob = path.read_bytes()
    merged = ref.wisdom.merge_wisdom([ref.wisdom.WisdomFile("k-abc", records=_records(ref, s)) for s in range(8)])
    return {
        "cases": cases,
        "spec_query_300": ref.wisdom.select(wf, a100, (300, 300, 300), {}).config,
        "file_sha256": hashlib.sha256(blob).hexdigest(), "file_text": blob.decode(),
        "merged": [r.to_json_obj() for r in merged.records],
    }


def capture_cases(ref):
    presets, cap = ref.presets, ref.capture
    d = presets.stencil3d_definition(True)
    args = [cap.BufferArg(0, "output", "f32", bytes(range(256)) * 16), cap.BufferArg(1, "input", "f64", b"\x01" * 200),
            cap.ScalarArg(2, "i32", 40), cap.ScalarArg(3, "i32", 30), cap.ScalarArg(4, "i32", 20),
            cap.ScalarArg(5, "f32", 0.25)]
    c = cap.capture_from_args(d, args, application="golden", timestamp="2026-01-01T00:00:00Z")
    blob = cap.serialize_capture(c)
    return {"sha256": hashlib.sha256(blob).hexdigest(), "length": len(blob), "problem": list(c.problem),
            "head_hex": blob[:96].hex()}


def tuner_cases(ref):
    out = []
    space = ref.space.ConfigSpace([ref.space.TunableParam(f"p{i}", tuple(range(v)), 0)
                                   for i, v in enumerate((4, 5, 3, 6))], ["p0 + p1 != 7"])
    for strategy, seed, evals in (("random", 1, 30), ("surrogate", 2, 45), ("exhaustive", 0, 60), ("surrogate", 9, 60)):
        model = ref.backend.SimCostModel(seed, space, noise_sigma=0.05 if seed == 9 else 0.0,
                                         failure_restriction="p3 == 5")
        ex = ref.backend.SimulatedExecutor(model, repetitions=5)
        s = ref.tuner.tune(space, ex, strategy=strategy, budget=ref.tuner.Budget(max_evaluations=evals,
                                                                                max_wall_seconds=None), seed=seed,
                           device=ref.backend.DeviceIdent("sim", "sim"), kernel_key="golden-k", problem=(64, 64))
        with tempfile.TemporaryDirectory() as tmp:
            p = Path(tmp) / "s.klsession"
            ref.tuner.save_session(s, p)
            fp = ref.tuner.session_fingerprint(p)
        out.append({"strategy": strategy, "seed": seed, "evals": evals, "fingerprint": fp,
                    "best": s.best_objective, "mu": model.mu, "a_diag": [model.a[i][i] for i in range(4)]})
    return out


def report_cases(ref):
    rng = ref.rng.SplitMix64(77)
    vecs = []
    for _ in range(20):
        v = [0.05 + 0.95 * rng.next_float() for _ in range(1 + rng.next_below(6))]
        r = ref.report.ppm(v)
        vecs.append({"effs": v, "best": r.best, "worst": r.worst, "ppm": r.ppm})
    return vecs


def main():
    ref = load_reference()
    data = {
        "generated_from": "/root/reference/pkg/src/kltune (kltune 0.1.0)",
        "expr": expr_cases(ref), "space": space_cases(ref), "kerneldef": kerneldef_cases(ref),
        "wisdom": wisdom_cases(ref), "capture": capture_cases(ref), "tuner": tuner_cases(ref),
        "report": report_cases(ref),
    }
    OUT.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
