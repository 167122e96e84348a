"""Level-A seam on the host (no GPU): the patched ``zoserve.runtime.forward_score``
must accept exactly the call the reference's ``_MeteredScorer`` makes
(runtime.py:174: ``forward_score(params, mcfg, batch, view=view,
precision=self.precision)``) and hand view-less calls back to the original with
the caller's precision."""
from types import SimpleNamespace

from paper_2605_28760_b200.plugin import install_into_zoserve


def _fake_zoserve():
    seen = []

    def forward_score(params, cfg, batch, view=None, precision="real64"):  # model.py:223-229
        seen.append((view, precision))
        return 1.25

    rt = SimpleNamespace(forward_score=forward_score, _fold_all=lambda state, params, meter: None)
    return SimpleNamespace(runtime=rt), seen


def test_patched_forward_score_takes_reference_keywords():
    zs, seen = _fake_zoserve()
    un = install_into_zoserve(zs)
    try:
        # the exact keyword form of runtime.py:174
        assert zs.runtime.forward_score({}, None, None, view=None, precision="real32") == 1.25
        assert zs.runtime.forward_score({}, None, None) == 1.25
        assert seen == [(None, "real32"), (None, "real64")]
    finally:
        un()
