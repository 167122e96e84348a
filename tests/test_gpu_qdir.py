"""q-direction mode (SURVEY.md §8(e) mode 2) through the C ABI, on one GPU.

The G ranks of a macro-step are emulated on one ctx: the scoring of direction g
leaves the parameter state untouched, so scoring g = 0..G-1 back to back and then
applying the gathered [G, 4] coefficients is exactly what G replicas do.
Checks: G = 1 is bit-identical to zo_step_async; for G > 1 the U/V streams are the
reference's, the losses match the float64 oracle (oracle.reference.qdir_macro_step)
within the fp16 tolerance, and the applied update is bit-exact given the device's
own coefficients (A += beta_g U_g in g order; factorized: the dense W64 update).
"""
import numpy as np
import pytest

from oracle import reference as R

pytestmark = pytest.mark.gpu

import zo_tolerances as _T

LOSS_TOL = _T.LOSS["fp16"]


def _setup(estimator="lozo_lazy", rank=2, steps=8):
    import torch
    from paper_2605_28760_b200.engine import ZoEngine
    cfg = R.ModelCfg(vocab=512, dim=128, n_layers=2, n_heads=2, prompt_len=63, init_seed=7, init_scale=0.02)
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=512, prompt_len=63, train_size=64, dev_size=4, val_size=4))
    batches, toks, golds = [], [], []
    for s in range(steps):
        p, gl, idx = R.sample_minibatch(splits, "train", 42, s, 16)
        g = np.array([[510], [511]])[gl]
        tok = np.concatenate([p, g], axis=1)
        batches.append((tok, g, idx))
        toks.append(tok)
        golds.append(g)
    d_tok = torch.from_numpy(np.stack(toks).astype(np.int32)).cuda()
    d_gold = torch.from_numpy(np.stack(golds).astype(np.int32)).cuda()
    eng = ZoEngine(cfg.vocab, cfg.dim, cfg.n_layers, cfg.n_heads, cfg.prompt_len, max_batch=16, rank=rank,
                   estimator=estimator)
    eng.init_params(cfg.init_seed, cfg.init_scale)
    return cfg, eng, batches, d_tok, d_gold


def _macro(eng, t, G, nu, lr, d_tok, d_gold):
    """Score the G directions of macro-step t, gather, apply; returns the [G, 4] gather."""
    import torch
    gathered = torch.zeros(G, 4, dtype=torch.float64, device="cuda")
    for g in range(G):
        s = t * G + g
        eng.qdir_score_async(42, t, G, g, nu, 1e-3, lr, False, d_tok[s].data_ptr(), d_gold[s].data_ptr(), 16)
        eng.out4_io(gathered[g].data_ptr(), False)
    eng.qdir_apply_async(42, t, G, lr, gathered.data_ptr())
    torch.cuda.synchronize()
    return gathered.cpu().numpy()


def test_qdir_G1_bitwise_equals_step_async():
    import torch
    outs = []
    for mode in ("step", "qdir"):
        cfg, eng, _, d_tok, d_gold = _setup()
        res = []
        for t in range(6):
            if mode == "step":
                eng.step_async(42, t, 3, 1e-3, 1e-3, False, d_tok[t].data_ptr(), d_gold[t].data_ptr(), 16)
            else:
                eng.qdir_score_async(42, t, 1, 0, 3, 1e-3, 1e-3, False, d_tok[t].data_ptr(), d_gold[t].data_ptr(),
                                     16)
                buf = torch.zeros(4, dtype=torch.float64, device="cuda")
                eng.out4_io(buf.data_ptr(), False)
                eng.qdir_apply_async(42, t, 1, 1e-3, buf.data_ptr())
            res.append(eng.read_out4())
            if (t + 1) % 3 == 0:
                eng.fold_async()
        res.append(eng.get_slot(2))
        res.append(eng.download("blk1.ff_up"))
        outs.append(res)
        eng.close()
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("G,nu", [(2, 4), (4, 4)])
def test_qdir_lozo_vs_oracle(G, nu):
    from paper_2605_28760_b200.engine import U as SU, V as SV
    from paper_2605_28760_b200.numerics import digest_hex
    lr = 1e-3
    cfg, eng, batches, d_tok, d_gold = _setup(steps=2 * G)
    params = R.init_params(cfg)
    st = R.LozoState()
    z = R.ZoCfg(seed=42, epsilon=1e-3, learning_rate=lr, rank=2, nu=nu, batch_size=16)
    for t in range(2):
        A_before = eng.get_slot(2)
        g4 = _macro(eng, t, G, nu, lr, d_tok, d_gold)
        recs = R.qdir_macro_step(params, cfg, st, z, t, G, batches[t * G:(t + 1) * G])
        for g, rec in enumerate(recs):
            assert abs(g4[g, 0] - rec.loss_plus) <= LOSS_TOL and abs(g4[g, 1] - rec.loss_minus) <= LOSS_TOL, (g4, rec)
        # the last direction's U and the shared window V are the reference's streams
        assert digest_hex(eng.digest(SU)) == recs[-1].u_digest
        assert digest_hex(eng.digest(SV)) == recs[-1].v_digest
        # update bit-exact given the device's coefficients: A += beta_g * U_g in g order
        A = eng.split(2, A_before)
        for g in range(G):
            for lid in eng.lids:
                u = R.gaussian(42, t * G + g, lid, R.ROLE_U, eng.shapes[lid][0], 2)
                A[lid] = A[lid] + g4[g, 3] * u
        got = eng.split(2, eng.get_slot(2))
        for lid in eng.lids:
            np.testing.assert_array_equal(got[lid], A[lid])
        # keep the oracle on the device's trajectory (coefficients differ within tolerance)
        st.A = {k: v.copy() for k, v in got.items()}
        if ((t + 1) * G) % nu == 0:  # run_serving_path's fold after the window's last step
            eng.fold()
            R.fold_all(params, st)
    assert eng.sampler_flags()[0] == 0
    eng.close()


def test_qdir_factorized_dense_update_bit_exact():
    import math
    G, r, lr = 2, 4, 1e-3
    cfg, eng, batches, d_tok, d_gold = _setup("factorized_sqrt_r", rank=r, steps=G)
    W0 = {lid: eng.download(lid) for lid in ("blk0.qkv", "embed")}
    g4 = _macro(eng, 0, G, 1, lr, d_tok, d_gold)
    params = R.init_params(cfg)
    z = R.ZoCfg(seed=42, epsilon=1e-3, learning_rate=lr, rank=r, nu=1, batch_size=16,
                estimator="factorized_sqrt_r")
    recs = R.qdir_macro_step(params, cfg, R.LozoState(), z, 0, G, batches[:G])
    for g, rec in enumerate(recs):
        assert abs(g4[g, 0] - rec.loss_plus) <= LOSS_TOL and abs(g4[g, 1] - rec.loss_minus) <= LOSS_TOL
    for lid, w in W0.items():
        m, n = w.shape
        for g in range(G):
            u = R.gaussian(42, g, lid, R.ROLE_U, m, r)
            v = R.gaussian(42, g, lid, R.ROLE_V, n, r)
            R.axpy_outer_raw(w, -(lr * g4[g, 2]) * (1.0 / math.sqrt(r)), u, v)
        np.testing.assert_array_equal(eng.download(lid), w)
    eng.close()


def test_qdir_rejects_G_not_dividing_nu():
    from paper_2605_28760_b200.errors import ConfigError
    cfg, eng, _, d_tok, d_gold = _setup(steps=1)
    with pytest.raises(ConfigError):
        eng.qdir_score_async(42, 0, 3, 0, 4, 1e-3, 1e-3, False, d_tok[0].data_ptr(), d_gold[0].data_ptr(), 16)
    eng.close()
