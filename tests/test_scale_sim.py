"""Multi-GPU placement (R26, §9): a length-only replay of the
lockstep, sequence-partitioned decode loop at the bench's weak-scaling sizes
(8192 GPT-J requests and 367,446 arena rows per GPU) must keep the
bytes-weighted lockstep efficiency >= 0.9 at G = 2/4/8 under worst-fit
placement, and the replay's planner must be the library's
(s3_plan_ffd_multibin, bit-exact on sampled steps)."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import scale_sim  # noqa: E402
from paper_2306_06000_b200 import build as s3build  # noqa: E402
from paper_2306_06000_b200 import s3 as abi  # noqa: E402


@pytest.mark.parametrize("policy", ["oracle", "bucket"])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_worst_fit_lockstep_efficiency(policy, G):
    s3build.build()
    checked = []

    def check(step, free, slots, snap, plan):
        if free is None:                       # "snapshot this step?"
            return step in (-1, 3, 40, 200)
        caps, reqs = snap
        fr, sl = free.copy(), slots.copy()
        rank = np.zeros(caps.shape[0], np.int32)
        abi.s3_plan_ffd_multibin(caps, reqs, fr, sl, rank)
        want = {int(q): r for r, _, q in plan}
        got = {int(q): int(r) for q, r in zip(reqs, rank) if r >= 0}
        assert got == want, f"step {step}: library plan differs from the replay"
        checked.append(step)
        return True

    r = scale_sim.simulate(8192 * G, G, "worst", policy=policy, check_plan=check)
    assert len(checked) == 4
    assert r["eff_run"] >= 0.9, r
    assert r["eff_window"] >= 0.9, r


def test_first_fit_was_unbalanced():
    # the round-1 rule (first rank with room) at G = 8: ~0.57 over the run
    r = scale_sim.simulate(8192 * 8, 8, "first", policy="oracle")
    assert r["eff_run"] < 0.7
