"""paper_2605_28760_b200.verify against hand-computed cases and the reference's own
golden trajectories (a trajectory strictly matches itself; an injected fault is
located).  Host-only."""
import copy
import os

import numpy as np
import pytest

from paper_2605_28760_b200.errors import InputError
from paper_2605_28760_b200.verify import rank_check, record_deltas, sign_match, strict_compare
from paper_2605_28760_b200.zo_engine import read_trajectory


def test_sign_match_bins_and_high_signal():
    rep = sign_match([0.0, 5e-5, -2e-3, 0.5, 0.02], [0.0, -1e-6, -1e-3, 0.1, -0.01], tau=0.005)
    assert rep.total == 5 and rep.matches == 3
    assert (rep.high_signal_pairs, rep.high_signal_matches) == (2, 1)
    bins = {b["label"]: (b["pairs"], b["matches"]) for b in rep.bins}
    assert bins["zero"] == (1, 1) and bins["(0,1e-4)"] == (1, 0) and bins["[1e-1,inf)"] == (1, 1)
    assert sign_match([1e-4], [1e-4], tau=1.0).high_signal_fraction == 1.0  # vacuous
    with pytest.raises(InputError):
        sign_match([1.0], [1.0, 2.0])


def test_strict_compare_self_and_fault(golden_dir):
    t = read_trajectory(os.path.join(golden_dir, "traj_micro_lozo.jsonl"))
    rep = strict_compare(t, t)
    assert rep.accepted == rep.steps and rep.max_dloss_plus == 0.0
    h, recs, fin = copy.deepcopy(t)
    recs[3].loss_plus += 1e-3
    recs[5].u_digest = "0" * 16
    rep = strict_compare(t, (h, recs, fin), loss_tol=1e-6)
    assert rep.loss_mismatch_steps == [3] and rep.digest_mismatch_steps == [5] and rep.rejected == 2
    assert len(record_deltas(recs)) == len(recs)


def test_strict_compare_skips_unaudited_digests(golden_dir):
    """run_serving_path(digest_every=k) leaves the records between audits with empty digests:
    strict_compare compares the audited ones only, counts them, and still checks losses."""
    t = read_trajectory(os.path.join(golden_dir, "traj_micro_lozo.jsonl"))
    h, recs, fin = copy.deepcopy(t)
    for i, r in enumerate(recs):
        if i % 4:
            r.u_digest = r.v_digest = ""
    rep = strict_compare(t, (h, recs, fin))
    assert rep.accepted == rep.steps and rep.digests_audited == len(range(0, len(recs), 4))
    recs[4].u_digest = "0" * 16  # a wrong audited digest is still caught
    recs[1].loss_minus += 1e-3   # and an unaudited step's loss is still compared
    rep = strict_compare(t, (h, recs, fin), loss_tol=1e-6)
    assert rep.digest_mismatch_steps == [recs[4].step] and rep.loss_mismatch_steps == [recs[1].step]


def test_rank_check():
    g = np.random.default_rng(0)
    low = g.standard_normal((20, 2)) @ g.standard_normal((2, 30))
    assert rank_check(low, 2) < 1e-12 and rank_check(np.zeros((4, 4)), 1) == 0.0
    assert rank_check(g.standard_normal((8, 8)), 1) > 0.1
