"""Checkpoint / resume of tuning sessions (SURVEY.md §5 "Checkpoint / resume":
the reference's tune() always starts fresh, tuner.py:200-213; the build
streams session lines as they are measured and continues an interrupted
session).  CPU only: the simulated executor stands in for the B200."""

import json

import pytest

from kltune.backend import SimCostModel, SimulatedExecutor
from kltune.presets import stencil3d_space
from kltune.tuner import (STATUS_RUNNING, Budget, load_checkpoint, load_session, save_session,
                          session_fingerprint, tune)

from conftest import grid_space


class Crash(Exception):
    pass


class CountingExecutor(SimulatedExecutor):
    """Simulated executor that counts real measurements and can die after n."""

    def __init__(self, model, die_after=None):
        super().__init__(model)
        self.measured = 0
        self.die_after = die_after
        self.prefetched = []

    def measure(self, config):
        if self.die_after is not None and self.measured >= self.die_after:
            raise Crash()
        self.measured += 1
        return super().measure(config)

    def prefetch(self, configs):
        self.prefetched.extend(configs)


def _space(strategy):
    return grid_space(4, 6, ["p0 + p1 != 5"]) if strategy == "exhaustive" else stencil3d_space(True)


@pytest.mark.parametrize("strategy", ["exhaustive", "random", "surrogate"])
def test_resume_equals_uninterrupted(tmp_path, strategy):
    space = _space(strategy)
    total, cut = 45, 17  # the cut lies inside the surrogate bootstrap's successor phase too (> 20 after resume)
    kw = dict(strategy=strategy, seed=7, kernel_key="k", problem=(64, 64, 64))
    full = tune(space, CountingExecutor(SimCostModel(3, space)), budget=Budget(total, None), **kw)
    save_session(full, tmp_path / "full.klsession")

    # first run dies after `cut` measurements; its checkpoint holds them
    ck = tmp_path / "ck.klsession"
    with pytest.raises(Crash):
        tune(space, CountingExecutor(SimCostModel(3, space), die_after=cut), budget=Budget(total, None),
             checkpoint=ck, **kw)
    head = json.loads(ck.read_text().splitlines()[0])
    assert head["status"] == STATUS_RUNNING
    prefix = load_checkpoint(ck)
    assert len(prefix.evaluations) == cut
    assert [e.config for e in prefix.evaluations] == [e.config for e in full.evaluations[:cut]]

    ex = CountingExecutor(SimCostModel(3, space))
    tune(space, ex, budget=Budget(total, None), resume=prefix, checkpoint=ck, **kw)
    assert ex.measured == total - cut  # the prefix is not measured again
    # nothing replayed is compiled again: the prefetched proposals are exactly the ones past the prefix
    # (the surrogate prefetches only its bootstrap draws)
    ahead = full.evaluations[cut:total if strategy != "surrogate" else 20]
    assert ex.prefetched == [e.config for e in ahead]
    assert session_fingerprint(ck) == session_fingerprint(tmp_path / "full.klsession")
    assert load_session(ck).best_objective == full.best_objective


def test_checkpoint_file_equals_end_of_session_write(tmp_path):
    space = stencil3d_space(True)
    kw = dict(strategy="surrogate", seed=11, kernel_key="k", problem=(8,))
    a = tune(space, SimulatedExecutor(SimCostModel(5, space)), budget=Budget(30, None),
             checkpoint=tmp_path / "a.klsession", **kw)
    save_session(a, tmp_path / "b.klsession")
    assert (tmp_path / "a.klsession").read_bytes() == (tmp_path / "b.klsession").read_bytes()


def test_torn_last_line_is_dropped(tmp_path):
    space = stencil3d_space(True)
    ck = tmp_path / "ck.klsession"
    with pytest.raises(Crash):
        tune(space, CountingExecutor(SimCostModel(1, space), die_after=9), strategy="random", seed=2,
             budget=Budget(40, None), checkpoint=ck, kernel_key="k")
    text = ck.read_text()
    ck.write_text(text + '{"config": {"block_x": 3')  # a write cut short by the crash
    prefix = load_checkpoint(ck)
    assert len(prefix.evaluations) == 9
    assert prefix.best_objective == min(e.measurement.objective for e in prefix.evaluations)
    # a finished session file loads unchanged through load_checkpoint
    done = tune(space, SimulatedExecutor(SimCostModel(1, space)), strategy="random", seed=2,
                budget=Budget(12, None), kernel_key="k")
    save_session(done, tmp_path / "done.klsession")
    assert load_checkpoint(tmp_path / "done.klsession").best_objective == done.best_objective


def test_resume_rejects_a_different_session():
    space = stencil3d_space(True)
    prefix = tune(space, SimulatedExecutor(SimCostModel(1, space)), strategy="random", seed=2,
                  budget=Budget(6, None), kernel_key="k")
    with pytest.raises(ValueError, match="cannot resume"):
        tune(space, SimulatedExecutor(SimCostModel(1, space)), strategy="random", seed=3,
             budget=Budget(10, None), kernel_key="k", resume=prefix)
    with pytest.raises(ValueError, match="cannot resume"):
        tune(space, SimulatedExecutor(SimCostModel(1, space)), strategy="surrogate", seed=2,
             budget=Budget(10, None), kernel_key="k", resume=prefix)
    # same strategy and seed over another space: the replay diverges and says where
    other = stencil3d_space(False)
    with pytest.raises(ValueError, match="diverges at evaluation"):
        tune(other, SimulatedExecutor(SimCostModel(1, other)), strategy="random", seed=2,
             budget=Budget(10, None), kernel_key="k", resume=prefix)


def test_resume_keeps_wall_budget_spent():
    space = stencil3d_space(True)
    prefix = tune(space, SimulatedExecutor(SimCostModel(1, space)), strategy="random", seed=2,
                  budget=Budget(5, None), kernel_key="k")
    prefix.evaluations[-1].wall_offset = 1e6  # the prefix already used the whole wall budget
    s = tune(space, SimulatedExecutor(SimCostModel(1, space)), strategy="random", seed=2,
             budget=Budget(None, 900.0), kernel_key="k", resume=prefix)
    assert len(s.evaluations) == 5


def test_cli_checkpoint_and_resume(tmp_path, monkeypatch):
    """`kltune tune --checkpoint` then `--resume` over a capture (sim backend)."""
    from kltune import cli
    from kltune.capture import BufferArg, ScalarArg, capture_from_args, write_capture
    from kltune.presets import stencil3d_definition

    monkeypatch.chdir(tmp_path)
    d = stencil3d_definition()
    args = [BufferArg(0, "output", "f32", bytes(64)), ScalarArg(2, "i32", 64), ScalarArg(3, "i32", 32),
            ScalarArg(4, "i32", 16), ScalarArg(5, "f64", 0.5)]
    write_capture(capture_from_args(d, args, application="t", timestamp="2026-01-01T00:00:00Z"), "c.klcap")
    common = ["tune", "c.klcap", "--backend", "sim", "--strategy", "surrogate", "--seed", "4", "--no-wisdom"]
    assert cli.main(common + ["--budget-evals", "30", "--session-out", "full.klsession"]) == 0
    assert cli.main(common + ["--budget-evals", "12", "--checkpoint", "--session-out", "part.klsession"]) == 0
    assert len(load_checkpoint("part.klsession").evaluations) == 12
    assert cli.main(common + ["--budget-evals", "30", "--resume", "part.klsession"]) == 0
    assert session_fingerprint("part.klsession") == session_fingerprint("full.klsession")


def test_resuming_into_the_same_file_never_truncates_it(tmp_path):
    """A resumed run that dies before its first new measurement leaves the
    checkpoint it resumed from intact (the prefix is rewritten to a temporary
    file and renamed over it)."""
    space = stencil3d_space(True)
    ck = tmp_path / "ck.klsession"
    kw = dict(strategy="random", seed=9, kernel_key="k", budget=Budget(30, None), checkpoint=ck)
    with pytest.raises(Crash):
        tune(space, CountingExecutor(SimCostModel(2, space), die_after=7), **kw)
    prefix = load_checkpoint(ck)
    with pytest.raises(Crash):
        tune(space, CountingExecutor(SimCostModel(2, space), die_after=0), resume=prefix, **kw)
    again = load_checkpoint(ck)
    assert [e.config for e in again.evaluations] == [e.config for e in prefix.evaluations]
    assert not (tmp_path / "ck.klsession.part").exists()
