"""Device abort path: a non-finite paired loss must leave every device slot and
weight untouched and surface as ScoringAbort (runtime.py:147, 312-317 -- the
reference's transactional step; here the trigger is a NaN/inf loss detected on
the device by k_coefficient, zo_kernels.cu, instead of an injected exception).

The fault is injected into the weights themselves (an inf embedding row for one
prompt token), so it travels through the real kernels: embed -> LN -> GEMMs ->
k_loss -> k_coefficient (abort flag) -> k_update / fold skipped.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

VOCAB, DIM, LAYERS, HEADS, PROMPT = 512, 128, 2, 2, 63


def _batch(t, seed=42, B=16):
    from oracle import reference as R
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=VOCAB, prompt_len=PROMPT, train_size=64, dev_size=4,
                                       val_size=4))
    p, gl, _ = R.sample_minibatch(splits, "train", seed, t, B)
    gold = np.array([[VOCAB - 2], [VOCAB - 1]])[gl]
    return np.concatenate([p, gold], axis=1).astype(np.int32), gold.astype(np.int32)


def _engine(rank=2, estimator="lozo_lazy"):
    from paper_2605_28760_b200.engine import ZoEngine
    eng = ZoEngine(VOCAB, DIM, LAYERS, HEADS, PROMPT, max_batch=16, rank=rank, estimator=estimator)
    eng.init_params(7, 0.02)
    return eng


def _poison(eng, token):
    E = eng.download("embed")
    E[token, :] = np.inf
    eng.upload({"embed": E})


@pytest.mark.parametrize("path", ["eager", "graph"])
def test_nonfinite_loss_skips_lozo_update(path):
    import torch

    from paper_2605_28760_b200.engine import A, U
    from paper_2605_28760_b200.errors import ScoringAbort
    eng = _engine()
    tok0, gold0 = _batch(0)
    out = eng.step(42, 0, 4, 1e-3, 1e-3, False, tok0, gold0)
    assert np.isfinite(out[:2]).all()
    a_before = eng.get_slot(A).copy()
    assert np.any(a_before != 0.0)
    tok1, gold1 = _batch(1)
    _poison(eng, int(tok1[0, 5]))
    w_before = eng.download("blk0.ff_up")
    if path == "eager":
        with pytest.raises(ScoringAbort):
            eng.step(42, 1, 4, 1e-3, 1e-3, False, tok1, gold1)
    else:
        d_tok = torch.from_numpy(tok1).cuda()
        d_gold = torch.from_numpy(np.stack([gold1, gold1])).cuda()
        eng.step_graph(42, 1, 4, 1e-3, 1e-3, False, d_tok.data_ptr(), d_gold.data_ptr(), tok1.shape[0])
        eng.synchronize()
        o4 = eng.read_out4()
        assert not np.isfinite(o4[0]) and o4[3] == 0.0, o4
    a_after = eng.get_slot(A)
    assert np.array_equal(a_after, a_before), "the update ran on a non-finite coefficient"
    assert np.array_equal(eng.download("blk0.ff_up"), w_before)
    # the U stream of the aborted step was still sampled (directions are counter-keyed)
    assert np.any(eng.get_slot(U) != 0.0)
    eng.close()


def test_nonfinite_loss_skips_factorized_dense_update():
    from paper_2605_28760_b200.errors import ScoringAbort
    eng = _engine(rank=2, estimator="factorized_sqrt_r")
    tok, gold = _batch(0)
    _poison(eng, int(tok[3, 7]))
    before = {lid: eng.download(lid) for lid in ("blk0.qkv", "blk1.ff_down", "embed")}
    with pytest.raises(ScoringAbort):
        eng.step(42, 0, 1, 1e-3, 1e-3, False, tok, gold)
    for lid, w in before.items():
        after = eng.download(lid)
        same = (after == w) | (np.isinf(after) & np.isinf(w))
        assert same.all(), f"{lid} changed on an aborted factorized step"
    eng.close()


def test_run_serving_path_marks_device_abort():
    """A poisoned weight makes step 0's losses non-finite: run_serving_path stops,
    marks the run aborted and records no step (runtime.py:312-317)."""
    from oracle import reference as R
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.runtime import run_serving_path
    from paper_2605_28760_b200.zo_engine import ZoConfig
    mcfg = M.ModelConfig(vocab=VOCAB, dim=DIM, n_layers=LAYERS, n_heads=HEADS, prompt_len=PROMPT, init_seed=7,
                         init_scale=0.02)
    task = M.generate_task(M.TaskConfig(seed=11, vocab=VOCAB, prompt_len=PROMPT, train_size=64, dev_size=4,
                                        val_size=4))
    zcfg = ZoConfig(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=2, nu=4, batch_size=16)
    host = R.init_params(R.ModelCfg(vocab=VOCAB, dim=DIM, n_layers=LAYERS, n_heads=HEADS, prompt_len=PROMPT,
                                    init_seed=7, init_scale=0.02))
    host["embed"] = host["embed"].copy()
    host["embed"][:, :] = np.inf
    run = run_serving_path(mcfg, task, zcfg, 4, eval_every=10 ** 9, params=host, compute_param_digests=False)
    assert run.aborted and run.steps_completed == 0 and run.trajectory == []
