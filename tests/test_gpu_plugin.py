"""Level-A drop-in (plugin.ReferenceScorer) through the C ABI on duck-typed
reference objects (the interface adapter.py:53-197 / model.py:406-427 define:
entries[lid].window_slot / perturb_slot with A, B, scale; perturb_sign; epsilon;
batch.prompts / golds / option_array() / batch_id).  The reference package is not
on the GPU box, so the objects are built here and the expected losses come from the
float64 oracle.  Covers lora_only and scope="full" (VectorProbe mutating the 1-D
params in place between the +1 and -1 calls)."""
from types import SimpleNamespace

import numpy as np
import pytest

import zo_tolerances as _T
from oracle import reference as R

pytestmark = pytest.mark.gpu
TOL = _T.LOSS["fp16"]


def _objects(full: bool):
    cfg = R.ModelCfg(vocab=64, dim=32, n_layers=2, n_heads=2, prompt_len=16, init_seed=7, init_scale=0.08)
    z = R.ZoCfg(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=2, nu=5, batch_size=8,
                scope="full" if full else "lora_only")
    params = R.init_params(cfg)
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=64, prompt_len=16, train_size=64, dev_size=8, val_size=8))
    p, gl, idx = R.sample_minibatch(splits, "train", z.seed, 3, z.batch_size)
    opts = np.array([[cfg.vocab - 2], [cfg.vocab - 1]])
    batch = SimpleNamespace(prompts=p, golds=gl, option_array=lambda: opts, batch_id=R.batch_id(idx))
    shapes = {k: v.shape for k, v in params.items() if v.ndim == 2}
    vshapes = {k: v.shape for k, v in params.items() if v.ndim == 1}
    dirs, _, _ = R.step_dirs(shapes, z, 3, vshapes)
    vecs = R.step_dirs.vectors
    Slot = lambda A, B: SimpleNamespace(A=A, B=B, scale=1.0, rank=A.shape[1])
    g = np.random.default_rng(5)
    entries = {lid: SimpleNamespace(update_slots=[], window_slot=Slot(1e-2 * g.standard_normal(u.shape), v),
                                    perturb_slot=Slot(u, v)) for lid, (u, v) in dirs.items()}
    state = SimpleNamespace(epsilon=z.epsilon, perturb_sign=0, entries=entries)
    tokens = np.concatenate([p, opts[gl]], axis=1)
    return cfg, z, params, batch, state, dirs, vecs, tokens, opts[gl]


def _oracle_loss(cfg, z, params, state, dirs, vecs, sign, tokens, gold):
    eff = dict(params)
    for lid, (u, v) in dirs.items():
        eff[lid] = R.compose(params[lid], state.entries[lid].window_slot.A, v, u, sign, z.epsilon)
    for vid, zz in vecs.items():
        eff[vid] = R.vector_probe_values(params[vid], zz, z.epsilon)[0 if sign == 1 else 1]
    return R.canonical_mean(R.forward_nll(eff, cfg, tokens, gold))


@pytest.mark.parametrize("full", [False, True])
def test_reference_scorer_pair(full):
    from paper_2605_28760_b200.plugin import ReferenceScorer
    cfg, z, params, batch, state, dirs, vecs, tokens, gold = _objects(full)
    base = {k: v.copy() for k, v in params.items()}
    ref = {s: _oracle_loss(cfg, z, base, state, dirs, vecs, s, tokens, gold) for s in (1, -1)}
    scorer = ReferenceScorer(params, cfg, state, rank=2, batch_size=8)
    # the reference's estimate_coefficient + VectorProbe order (zo_engine.py:269-332)
    state.perturb_sign = 1
    for vid, zz in vecs.items():
        params[vid] = params[vid] + (1.0 * z.epsilon) * zz
    lp = scorer(batch)
    state.perturb_sign = -1
    for vid, zz in vecs.items():
        params[vid] = params[vid] + (-2.0 * z.epsilon) * zz
    lm = scorer(batch)
    assert abs(lp - ref[1]) <= TOL and abs(lm - ref[-1]) <= TOL, (lp, lm, ref)
    # the probe difference, which the estimator consumes
    assert abs((lp - lm) - (ref[1] - ref[-1])) <= max(_T.DL_REL["fp16"] * abs(ref[1] - ref[-1]), 2e-4)
    # pure: the reference's params/state were not written by the scorer
    for k in base:
        if base[k].ndim == 2:
            np.testing.assert_array_equal(params[k], base[k])


def test_install_into_zoserve_patches_and_restores():
    from paper_2605_28760_b200.plugin import install_into_zoserve
    calls = []
    rt = SimpleNamespace(forward_score=lambda *a, **k: calls.append("orig") or 1.0,
                         _fold_all=lambda *a, **k: calls.append("fold"))
    zs = SimpleNamespace(runtime=rt)
    orig = (rt.forward_score, rt._fold_all)
    un = install_into_zoserve(zs)
    assert (rt.forward_score, rt._fold_all) != orig
    assert rt.forward_score(None, None, None, None) == 1.0 and calls == ["orig"]  # view=None -> reference path
    un()
    assert (rt.forward_score, rt._fold_all) == orig
