"""Trajectory verification -- the ``zoserve.verify`` surface (verify.py:21-31) that
judges a device run against a reference run: sign agreement of L+ - L- (criterion 3),
strict step-by-step equivalence (seeds, U/V digests, paired losses within a
tolerance) and the low-rank audit of a weight delta.  Pure functions of finished
trajectories (``zo_engine.read_trajectory`` triples / ``ZoStepRecord`` lists);
nothing here touches a device.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import InputError

__all__ = ["SignMatchReport", "sign_match", "record_deltas", "StrictCompareReport", "strict_compare",
           "rank_check"]

# |delta| bins of the report, keyed by the reference run (verify.py:38-58)
_BINS = (("zero", 0.0, 0.0), ("(0,1e-4)", 0.0, 1e-4), ("[1e-4,1e-3)", 1e-4, 1e-3), ("[1e-3,1e-2)", 1e-3, 1e-2),
         ("[1e-2,1e-1)", 1e-2, 1e-1), ("[1e-1,inf)", 1e-1, float("inf")))


def _sign(x: float) -> int:
    return (x > 0) - (x < 0)


def _bin(delta: float) -> str:
    a = abs(delta)
    if a == 0.0:
        return "zero"
    for label, lo, hi in _BINS[1:]:
        if lo <= a < hi or (lo == 0.0 and a < hi):
            return label
    return _BINS[-1][0]


@dataclass
class SignMatchReport:
    """verify.py:61-113: zero is its own sign; high-signal = |delta_ref| >= tau (an
    empty high-signal set reports 1.0)."""
    total: int
    matches: int
    tau: float
    high_signal_pairs: int
    high_signal_matches: int
    bins: list = field(default_factory=list)

    @property
    def overall_fraction(self) -> float:
        return self.matches / self.total if self.total else 1.0

    @property
    def high_signal_fraction(self) -> float:
        return self.high_signal_matches / self.high_signal_pairs if self.high_signal_pairs else 1.0

    def to_dict(self) -> dict:
        return {"total": self.total, "matches": self.matches, "overall_fraction": self.overall_fraction,
                "tau": self.tau, "high_signal_pairs": self.high_signal_pairs,
                "high_signal_matches": self.high_signal_matches,
                "high_signal_fraction": self.high_signal_fraction, "bins": self.bins}


def record_deltas(records) -> list[float]:
    """L+ - L- per step, in step order (verify.py:116-118)."""
    return [r.loss_plus - r.loss_minus for r in records]


def sign_match(deltas_a, deltas_b, tau: float = 0.005) -> SignMatchReport:
    """verify.py:121-162; list A is the reference run."""
    a, b = list(deltas_a), list(deltas_b)
    if len(a) != len(b):
        raise InputError(f"sign_match needs aligned runs: {len(a)} vs {len(b)} steps")
    counts = {label: [0, 0] for label, _, _ in _BINS}
    matches = hs = hs_m = 0
    for da, db in zip(a, b):
        hit = _sign(da) == _sign(db)
        matches += hit
        c = counts[_bin(da)]
        c[0] += 1
        c[1] += hit
        if abs(da) >= tau:
            hs += 1
            hs_m += hit
    bins = [{"label": k, "pairs": p, "matches": m, "fraction": (m / p) if p else None} for k, (p, m) in counts.items()]
    return SignMatchReport(len(a), matches, tau, hs, hs_m, bins)


@dataclass
class StrictCompareReport:
    """verify.py:171-235: a step is accepted iff seed, both digests and both losses
    (within loss_tol) agree."""
    steps: int
    accepted: int
    seed_mismatches: int
    digest_mismatches: int
    max_dloss_plus: float
    max_dloss_minus: float
    loss_tol: float
    final_loss_difference: float | None
    seed_mismatch_steps: list = field(default_factory=list)
    digest_mismatch_steps: list = field(default_factory=list)
    loss_mismatch_steps: list = field(default_factory=list)
    digests_audited: int = -1  # steps whose U/V digests were compared (-1: not counted)

    @property
    def rejected(self) -> int:
        return self.steps - self.accepted

    def to_dict(self) -> dict:
        d = dict(self.__dict__)
        d["rejected"] = self.rejected
        return d


def strict_compare(traj_a, traj_b, loss_tol: float = 1e-12) -> StrictCompareReport:
    """verify.py:238-301 over (header, records, final) triples."""
    ha, ra, fa = traj_a
    hb, rb, fb = traj_b
    if ha.get("schema") != hb.get("schema"):
        raise InputError(f"trajectory schema mismatch: {ha.get('schema')} vs {hb.get('schema')}")
    if len(ra) != len(rb):
        raise InputError(f"step count mismatch: {len(ra)} vs {len(rb)}")
    seed_bad, dig_bad, loss_bad = [], [], []
    n_audited = 0
    accepted, max_dp, max_dm = 0, 0.0, 0.0
    for x, y in zip(ra, rb):
        if x.step != y.step:
            raise InputError(f"step misalignment: {x.step} vs {y.step}")
        ok = True
        if x.seed != y.seed:
            seed_bad.append(x.step)
            ok = False
        # an empty digest is an unaudited step (runtime.run_serving_path digest_every > 1)
        audited = all((x.u_digest, y.u_digest, x.v_digest, y.v_digest))
        n_audited += audited
        if audited and (x.u_digest != y.u_digest or x.v_digest != y.v_digest):
            dig_bad.append(x.step)
            ok = False
        dp, dm = abs(x.loss_plus - y.loss_plus), abs(x.loss_minus - y.loss_minus)
        max_dp, max_dm = max(max_dp, dp), max(max_dm, dm)
        if dp > loss_tol or dm > loss_tol:
            loss_bad.append(x.step)
            ok = False
        accepted += ok
    final = None
    if fa is not None and fb is not None and "eval_loss" in fa and "eval_loss" in fb:
        final = abs(fa["eval_loss"] - fb["eval_loss"])
    return StrictCompareReport(len(ra), accepted, len(seed_bad), len(dig_bad), max_dp, max_dm, loss_tol, final,
                               seed_bad, dig_bad, loss_bad, n_audited)


def rank_check(delta_w, r: int) -> float:
    """sigma_{r+1} / sigma_1 of a weight delta (verify.py:304-324); 0 for a zero matrix
    or r past the spectrum."""
    d = np.asarray(delta_w, dtype=np.float64)
    if d.ndim != 2:
        raise InputError(f"rank_check needs a matrix, got ndim={d.ndim}")
    if not np.any(d):
        return 0.0
    s = np.linalg.svd(d, compute_uv=False)
    if r >= s.size or s[0] == 0.0:
        return 0.0
    return float(s[r] / s[0])
