"""The multi-GPU step halves as captured CUDA graphs (zob200.h zo_step_score_graph /
zo_step_apply_graph / zo_qdir_score_graph / zo_qdir_apply_graph) against their eager
_async forms, with the ranks emulated on one GPU as in tests/test_gpu_qdir.py:
every result -- gathered coefficients, the window A, folded weights, factorized
dense updates -- must be bitwise identical, and each half must replay as one graph."""
import numpy as np
import pytest

from oracle import reference as R

pytestmark = pytest.mark.gpu


def _setup(estimator="lozo_lazy", rank=2, steps=12):
    import torch
    from paper_2605_28760_b200.engine import ZoEngine
    cfg = R.ModelCfg(vocab=512, dim=128, n_layers=2, n_heads=2, prompt_len=63, init_seed=7, init_scale=0.02)
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=512, prompt_len=63, train_size=64, dev_size=4, val_size=4))
    toks, golds = [], []
    for s in range(steps):
        p, gl, _ = R.sample_minibatch(splits, "train", 42, s, 16)
        g = np.array([[510], [511]])[gl]
        toks.append(np.concatenate([p, g], axis=1))
        golds.append(g)
    d_tok = torch.from_numpy(np.stack(toks).astype(np.int32)).cuda()
    d_gold = torch.from_numpy(np.stack(golds).astype(np.int32)).cuda()
    eng = ZoEngine(cfg.vocab, cfg.dim, cfg.n_layers, cfg.n_heads, cfg.prompt_len, max_batch=16, rank=rank,
                   estimator=estimator)
    eng.init_params(cfg.init_seed, cfg.init_scale)
    return eng, d_tok, d_gold


@pytest.mark.parametrize("estimator", ["lozo_lazy", "factorized_sqrt_r"])
def test_exact_mode_split_graph_equals_async(estimator):
    """Exact-trajectory mode at world 2: each rank scores 8 of the 16 examples, the NLLs are
    gathered into canonical order, every rank applies the same update."""
    import torch
    world, B, nu = 2, 16, 3
    bl = B // world
    results = {}
    for graph in (False, True):
        eng, d_tok, d_gold = _setup(estimator)
        eng.set_schedule("row_invariant")
        score = eng.step_score_graph if graph else eng.step_score_async
        apply = eng.step_apply_graph if graph else eng.step_apply_async
        nll = torch.zeros(world, 2, bl, dtype=torch.float64, device="cuda")
        full = torch.zeros(2, B, dtype=torch.float64, device="cuda")
        outs = []
        for t in range(7):
            for g in range(world):
                score(42, t, nu, 1e-3, d_tok[t, g * bl:].data_ptr(), d_gold[t, g * bl:].data_ptr(), bl)
                eng.nll_io(nll[g].data_ptr(), 2 * bl, False)
            full.view(2, world, bl).copy_(nll.transpose(0, 1))
            eng.nll_io(full.data_ptr(), 2 * B, True)
            apply(1e-3, 1e-3, False, B)
            outs.append(eng.read_out4())
            if estimator == "lozo_lazy" and (t + 1) % nu == 0:
                eng.fold_async()
        outs.append(eng.get_slot(2))
        outs.append(eng.download("blk1.ff_up"))
        if graph:
            k = eng.split_graph_kernels()
            assert k[0] > 10 and k[1] >= 2, k
        results[graph] = outs
        eng.close()
    for a, b in zip(results[False], results[True]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("estimator", ["lozo_lazy", "factorized_sqrt_r"])
def test_qdir_split_graph_equals_async(estimator):
    import torch
    G, nu = 2, 4
    results = {}
    for graph in (False, True):
        eng, d_tok, d_gold = _setup(estimator)
        score = eng.qdir_score_graph if graph else eng.qdir_score_async
        apply = eng.qdir_apply_graph if graph else eng.qdir_apply_async
        gathered = torch.zeros(G, 4, dtype=torch.float64, device="cuda")
        outs = []
        for t in range(5):
            for g in range(G):
                s = t * G + g
                score(42, t, G, g, nu, 1e-3, 1e-3, False, d_tok[s].data_ptr(), d_gold[s].data_ptr(), 16)
                eng.out4_io(gathered[g].data_ptr(), False)
            apply(42, t, G, 1e-3, gathered.data_ptr())
            outs.append(gathered.cpu().numpy().copy())
            if estimator == "lozo_lazy" and ((t + 1) * G) % nu == 0:
                eng.fold_async()
        outs.append(eng.get_slot(2))
        outs.append(eng.download("blk0.qkv"))
        if graph:
            k = eng.split_graph_kernels()
            assert k[2] > 10 and k[3] >= 2, k
        results[graph] = outs
        eng.close()
    for a, b in zip(results[False], results[True]):
        np.testing.assert_array_equal(a, b)
