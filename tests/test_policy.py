"""Refresh schedule parity (host logic): must match the reference exactly."""

import itertools

import numpy as np
import pytest

from oracle import flashblock_oracle as orc
from paper_2602_05305_b200 import policy as P
from paper_2602_05305_b200.errors import ShapeError


def test_decide_full_matrix_matches_oracle():
    # reference tests/test_policy.py:37-44
    for mode, tau, cv, fv, upd, gate in itertools.product(
            P.MODES, (1, 2, 4), (True, False), (True, False), (0, 1, 2, 3, 9), (True, False)):
        got = P.decide(P.ReuseConfig(tau=tau, mode=mode), cv, fv, upd, gate)
        assert got.value == orc.decide(mode, tau, cv, fv, upd, gate)


def test_config_validation_and_immutability():
    for bad in (dict(tau=0), dict(gamma=1.0 + 1e-9), dict(gamma=-0.1), dict(mode="sometimes")):
        with pytest.raises(ValueError):
            P.ReuseConfig(**bad)
    P.ReuseConfig(tau=1, gamma=0.0)
    with pytest.raises(AttributeError):
        P.ReuseConfig().tau = 5


def test_count_updated_tokens():
    a = np.array([0, 0, 5, 7])
    assert P.count_updated_tokens(a, a.copy()) == 0
    assert P.count_updated_tokens(a, np.array([1, 2, 3, 4])) == 4
    assert P.count_updated_tokens(np.array([], dtype=int), np.array([], dtype=int)) == 0
    with pytest.raises(ShapeError):
        P.count_updated_tokens(np.array([1, 2]), np.array([1, 2, 3]))


@pytest.mark.parametrize("bs,steps,per", [(32, 32, 1), (32, 16, 2), (8, 8, 3), (16, 10, 2),
                                          (32, 32, 0), (5, 9, 2), (100, 7, 3), (1, 1, 1)])
def test_unmask_schedule_matches_oracle(bs, steps, per):
    got = P.unmask_schedule(bs, steps, per)
    assert got == orc.unmask_schedule(bs, steps, per)
    assert sum(got) == bs


def test_refresh_schedule_matches_reference_simulator(golden_meta):
    # decisions captured from the reference's own run_sequence (tests/golden/make_golden.py)
    for case in golden_meta["schedules"]:
        got = P.refresh_schedule(P.ReuseConfig(tau=case["tau"]), case["block_size"],
                                 case["steps"], case["per_step"])
        want = ["Recompute" if d in ("FirstVisit", "Recompute") else "Reuse"
                for d in case["decisions"]]
        assert [d.value for d in got] == want, case


def test_headline_schedule_refreshes_once_per_block():
    # C2 headline: S=32 steps, 1 unmask/step, tau=2 -> 1 refresh in 32 steps
    sched = P.refresh_schedule(P.ReuseConfig(tau=2), 32, 32, 1)
    assert [d.value for d in sched].count("Recompute") == 1
    # 2 unmask/step with tau=2 refreshes every step
    sched = P.refresh_schedule(P.ReuseConfig(tau=2), 32, 16, 2)
    assert all(d.value == "Recompute" for d in sched)
