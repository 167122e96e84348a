"""Scorer / step parity on the GPU against the reference's golden fixtures.

Tolerances: tests/tolerances.py (fp16 / bf16 tensor-core operands, fp32 accumulate;
~3x the observed error); U/V digests and the float64 init are bit-exact.
"""
import json
import os

import numpy as np
import pytest

from oracle import reference as R

pytestmark = pytest.mark.gpu

import zo_tolerances as TOL

NLL_TOL = TOL.NLL
LOSS_TOL = TOL.LOSS
DL_REL = TOL.DL_REL  # |d(L+ - L-)| relative


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _engine(g, precision="fp16", rank=None, estimator="lozo_lazy", max_batch=None, scope="lora_only"):
    from paper_2605_28760_b200.engine import ZoEngine
    m = g["model"]
    return ZoEngine(m["vocab"], m["dim"], m["n_layers"], m["n_heads"], m["prompt_len"], opt_len=1,
                    max_batch=max_batch or 16, rank=rank or g.get("rank", 2), estimator=estimator,
                    precision=precision, scope=scope)


def _params_digest(eng, cfg):
    params = {lid: eng.download(lid) for lid in eng.lids}
    for i in range(cfg.n_layers):
        for ln in ("ln1", "ln2"):
            params[f"blk{i}.{ln}.scale"] = np.ones(cfg.dim)
            params[f"blk{i}.{ln}.shift"] = np.zeros(cfg.dim)
    params["ln_f.scale"] = np.ones(cfg.dim)
    params["ln_f.shift"] = np.zeros(cfg.dim)
    return R.params_digest(params)


@pytest.mark.parametrize("name", ["micro", "small"])
def test_init_params_bit_exact(golden_dir, name):
    g = _load(golden_dir, f"forward_{name}.json")
    cfg = R.ModelCfg(**g["model"])
    eng = _engine(g)
    eng.init_params(cfg.init_seed, cfg.init_scale)
    assert _params_digest(eng, cfg) == g["params_digest"]


@pytest.mark.parametrize("precision", ["fp16", "bf16"])
@pytest.mark.parametrize("name", ["micro", "small"])
def test_forward_nll_vs_reference(golden_dir, name, precision):
    g = _load(golden_dir, f"forward_{name}.json")
    cfg = R.ModelCfg(**g["model"])
    eng = _engine(g, precision)
    eng.init_params(cfg.init_seed, cfg.init_scale)
    step, r = g["step"], g["rank"]
    eng.sample_v(g["zseed"], step, 50)
    eng.sample_u(g["zseed"], step)
    A = {lid: g["a_scale"] * R.gaussian(g["a_seed"], step, lid, R.ROLE_U, eng.shapes[lid][0], r) for lid in eng.lids}
    eng.set_slot(2, eng.join(2, A))
    # the device U/V must be the reference's streams
    U = eng.split(0, eng.get_slot(0))
    for lid in eng.lids[:3]:
        np.testing.assert_array_equal(U[lid], R.gaussian(g["zseed"], step, lid, R.ROLE_U, eng.shapes[lid][0], r))
    tokens = np.asarray(g["tokens"])
    gold = tokens[:, cfg.prompt_len:]
    eng.prepare_probe(g["epsilon"], 0)
    nll = eng.score(tokens, np.stack([gold, gold]), nsign=2)
    eng.prepare_probe(g["epsilon"], 1)
    nll0 = eng.score(tokens, gold, nsign=1)[0]
    ref_p, ref_m, ref_0 = (np.array(g["nll"][f"real64:{s}"]) for s in (1, -1, 0))
    tol = NLL_TOL[precision]
    d_ref = R.canonical_mean(ref_p) - R.canonical_mean(ref_m)
    d_got = R.canonical_mean(nll[0]) - R.canonical_mean(nll[1])
    _report(f"forward_{name}_{precision}", {
        "max_abs_nll_plus": float(np.max(np.abs(nll[0] - ref_p))),
        "max_abs_nll_minus": float(np.max(np.abs(nll[1] - ref_m))),
        "max_abs_nll_sign0": float(np.max(np.abs(nll0 - ref_0))),
        "dL_ref": d_ref, "dL_got": d_got, "rel_err_dL": abs(d_got - d_ref) / max(abs(d_ref), 1e-30)})
    np.testing.assert_allclose(nll[0], ref_p, atol=tol, rtol=0)
    np.testing.assert_allclose(nll[1], ref_m, atol=tol, rtol=0)
    np.testing.assert_allclose(nll0, ref_0, atol=tol, rtol=0)
    # the probe difference is what the estimator consumes: compare L+ - L-
    assert abs(d_got - d_ref) <= max(DL_REL[precision] * abs(d_ref), 2e-4), (d_got, d_ref)


def _report(name, data):
    """Parity numbers for the record (gpurun_out/ is brought back from the GPU box)."""
    os.makedirs("gpurun_out/parity", exist_ok=True)
    with open(os.path.join("gpurun_out/parity", name + ".json"), "w") as f:
        json.dump(data, f, indent=1)


def _traj(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        lines = [json.loads(l) for l in f if l.strip()]
    return lines[0], [l for l in lines if l["record"] == "step"], lines[-1]


@pytest.mark.parametrize("name", ["micro_lozo", "small_lozo", "micro_full"])
def test_device_step_trajectory(golden_dir, name):
    """zo_step (fused device lozo_step) vs the reference's run_serving_path trajectory."""
    from paper_2605_28760_b200.engine import U as SU, V as SV
    from paper_2605_28760_b200.numerics import digest_hex
    h, recs, fin = _traj(golden_dir, f"traj_{name}.jsonl")
    cfg = R.ModelCfg(**h["model"])
    z = R.ZoCfg(**h["zo"])
    splits = R.generate_task(R.TaskCfg(**h["task"]))
    eng = _engine({"model": h["model"], "rank": z.rank}, max_batch=z.batch_size, scope=z.scope)
    eng.init_params(cfg.init_seed, cfg.init_scale)
    rows = []
    for t, rec in enumerate(recs):
        p, gl, idx = R.sample_minibatch(splits, "train", z.seed, t, z.batch_size)
        gold = np.array([[cfg.vocab - 2], [cfg.vocab - 1]])[gl]
        tokens = np.concatenate([p, gold], axis=1)
        out = eng.step(z.seed, t, z.nu, z.epsilon, z.learning_rate, z.divide_by_r, tokens, gold)
        rows.append({"step": t, "u_ok": digest_hex(eng.digest(SU)) == rec["u_digest"],
                     "v_ok": digest_hex(eng.digest(SV)) == rec["v_digest"],
                     "dLp": float(out[0] - rec["loss_plus"]), "dLm": float(out[1] - rec["loss_minus"]),
                     "c_ref": rec["coefficient"], "c": float(out[2]),
                     "sign_ok": bool(np.sign(out[0] - out[1]) == np.sign(rec["loss_plus"] - rec["loss_minus"]))})
        if (t + 1) % z.nu == 0:
            eng.fold()
    _report(f"traj_{name}", {"rows": rows, "max_dL": max(max(abs(r["dLp"]), abs(r["dLm"])) for r in rows)})
    assert all(r["u_ok"] and r["v_ok"] for r in rows)
    assert max(max(abs(r["dLp"]), abs(r["dLm"])) for r in rows) <= LOSS_TOL["fp16"], rows
    for r in rows:  # the coefficient the update consumes, on high-signal steps
        if abs(r["c_ref"]) * 2e-3 >= TOL.HIGH_SIGNAL:
            assert abs(r["c"] - r["c_ref"]) <= TOL.C_REL * abs(r["c_ref"]), r
    assert sum(r["sign_ok"] for r in rows) >= 0.9 * len(rows)
    assert eng.sampler_flags()[0] == 0


@pytest.mark.parametrize("precision", ["fp16"])
def test_forward_vs_oracle_streamk_shapes(precision):
    """A config large enough that every layer GEMM runs stream-K and the fused extension
    partials span many tiles (d=1024, dh=128, M=2048), against the float64 oracle."""
    from paper_2605_28760_b200.engine import ZoEngine
    cfg = R.ModelCfg(vocab=4096, dim=1024, n_layers=2, n_heads=8, prompt_len=63, init_seed=7, init_scale=0.02)
    eng = ZoEngine(cfg.vocab, cfg.dim, cfg.n_layers, cfg.n_heads, cfg.prompt_len, max_batch=16, rank=2,
                   precision=precision)
    eng.init_params(cfg.init_seed, cfg.init_scale)
    params = R.init_params(cfg)
    eng.sample_v(42, 0, 50)
    eng.sample_u(42, 3)
    A = {lid: 1e-3 * R.gaussian(43, 3, lid, R.ROLE_U, eng.shapes[lid][0], 2) for lid in eng.lids}
    eng.set_slot(2, eng.join(2, A))
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=cfg.vocab, prompt_len=63, train_size=64, dev_size=4,
                                       val_size=4))
    p, gl, idx = R.sample_minibatch(splits, "train", 42, 3, 16)
    gold = np.array([[cfg.vocab - 2], [cfg.vocab - 1]])[gl]
    tokens = np.concatenate([p, gold], axis=1)
    eng.prepare_probe(1e-3, 0)
    nll = eng.score(tokens, np.stack([gold, gold]), nsign=2)
    ref = {}
    for sign in (1, -1):
        eff = dict(params)
        for lid in eng.lids:
            m, n = eng.shapes[lid]
            u = R.gaussian(42, 3, lid, R.ROLE_U, m, 2)
            v = R.gaussian(42, 0, lid, R.ROLE_V, n, 2)
            eff[lid] = R.compose(params[lid], A[lid], v, u, sign, 1e-3)
        ref[sign] = R.forward_nll(eff, cfg, tokens, gold)
    d_ref = R.canonical_mean(ref[1]) - R.canonical_mean(ref[-1])
    d_got = R.canonical_mean(nll[0]) - R.canonical_mean(nll[1])
    _report(f"forward_oracle_d1024_{precision}", {
        "max_abs_nll_plus": float(np.max(np.abs(nll[0] - ref[1]))),
        "max_abs_nll_minus": float(np.max(np.abs(nll[1] - ref[-1]))), "dL_ref": d_ref, "dL_got": d_got})
    np.testing.assert_allclose(nll[0], ref[1], atol=NLL_TOL[precision], rtol=0)
    np.testing.assert_allclose(nll[1], ref[-1], atol=NLL_TOL[precision], rtol=0)
    assert abs(d_got - d_ref) <= max(DL_REL[precision] * abs(d_ref), 2e-4), (d_got, d_ref)


def test_graph_step_bitwise_equals_eager():
    """The CUDA-graph replay of the step body is bit-identical to eager launches
    (losses, coefficient and the window A arena), across a window boundary."""
    import torch
    from paper_2605_28760_b200.engine import ZoEngine
    cfg = R.ModelCfg(vocab=512, dim=128, n_layers=2, n_heads=2, prompt_len=63, init_seed=7, init_scale=0.02)
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=512, prompt_len=63, train_size=64, dev_size=4, val_size=4))
    toks, golds = [], []
    for t in range(7):
        p, gl, _ = R.sample_minibatch(splits, "train", 42, t, 16)
        g = np.array([[510], [511]])[gl]
        toks.append(np.concatenate([p, g], axis=1))
        golds.append(g)
    d_tok = torch.from_numpy(np.stack(toks).astype(np.int32)).cuda()
    d_gold = torch.from_numpy(np.stack(golds).astype(np.int32)).cuda()
    outs = []
    for graph in (False, True):
        eng = ZoEngine(cfg.vocab, cfg.dim, cfg.n_layers, cfg.n_heads, cfg.prompt_len, max_batch=16, rank=2)
        eng.init_params(cfg.init_seed, cfg.init_scale)
        res = []
        for t in range(7):
            fn = eng.step_graph if graph else eng.step_async
            fn(42, t, 3, 1e-3, 1e-3, False, d_tok[t].data_ptr(), d_gold[t].data_ptr(), 16)
            res.append(eng.read_out4())
            if (t + 1) % 3 == 0:
                eng.fold_async()
        res.append(eng.get_slot(2))
        res.append(eng.download("blk0.qkv"))
        outs.append(res)
        eng.close()
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("rank", [16, 128])
def test_factorized_high_rank_step_vs_oracle(rank):
    """MeZO-style factorized step at high rank (BASELINE config 5 shape family): the
    r > 8 paths (separate extension pass, 1-term 16-bit extension columns, embedding
    delta folded into the logits) against the float64 oracle's factorized_step, and the
    dense float64 update bit-exact given the device coefficient."""
    import math
    from paper_2605_28760_b200.engine import ZoEngine
    cfg = R.ModelCfg(vocab=512, dim=128, n_layers=2, n_heads=2, prompt_len=63, init_seed=7, init_scale=0.02)
    z = R.ZoCfg(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=rank, nu=1, batch_size=16,
                estimator="factorized_sqrt_r")
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=512, prompt_len=63, train_size=64, dev_size=4, val_size=4))
    eng = ZoEngine(cfg.vocab, cfg.dim, cfg.n_layers, cfg.n_heads, cfg.prompt_len, max_batch=16, rank=rank,
                   estimator="factorized_sqrt_r")
    eng.init_params(cfg.init_seed, cfg.init_scale)
    params = R.init_params(cfg)
    for t in range(2):
        p, gl, idx = R.sample_minibatch(splits, "train", z.seed, t, z.batch_size)
        gold = np.array([[cfg.vocab - 2], [cfg.vocab - 1]])[gl]
        tokens = np.concatenate([p, gold], axis=1)
        w_before = eng.download("blk1.ff_down")
        out = eng.step(z.seed, t, 1, z.epsilon, z.learning_rate, False, tokens, gold)
        ref_params = {k: v.copy() for k, v in params.items()}
        rec = R.factorized_step(ref_params, cfg, z, t, tokens, gold, idx)
        assert abs(out[0] - rec.loss_plus) <= LOSS_TOL["fp16"] and abs(out[1] - rec.loss_minus) <= LOSS_TOL["fp16"]
        # dense update with the device's c: W += (-(lr c)/sqrt(r)) U V^T, k ascending
        m, n = w_before.shape
        u = R.gaussian(z.seed, t, "blk1.ff_down", R.ROLE_U, m, rank)
        v = R.gaussian(z.seed, t, "blk1.ff_down", R.ROLE_V, n, rank)
        R.axpy_outer_raw(w_before, -(z.learning_rate * float(out[2])) * (1.0 / math.sqrt(rank)), u, v)
        np.testing.assert_array_equal(eng.download("blk1.ff_down"), w_before)
        params = {lid: eng.download(lid) for lid in eng.lids} | {k: v for k, v in params.items() if v.ndim == 1}
    eng.close()


@pytest.mark.parametrize("opt_len", [2, 3])
def test_multi_token_options_vs_oracle(opt_len):
    """Options of L > 1 tokens (model.py:202-215 sums the NLL of rows prompt_len-1+j, j < L):
    the forward runs positions [0, T-1) only (the last token is never attended by a scored
    row), the L scored rows per sequence go through the pruned last layer, the LM head and
    the loss; paired probes against the float64 oracle."""
    from paper_2605_28760_b200.engine import ZoEngine
    cfg = R.ModelCfg(vocab=256, dim=64, n_layers=2, n_heads=2, prompt_len=20, init_seed=7, init_scale=0.05)
    B, r, step, eps = 8, 2, 3, 1e-3
    rng = np.random.default_rng(0)
    prompts = rng.integers(4, cfg.vocab, size=(B, cfg.prompt_len))
    gold = rng.integers(4, cfg.vocab, size=(B, opt_len))
    tokens = np.concatenate([prompts, gold], axis=1)
    eng = ZoEngine(cfg.vocab, cfg.dim, cfg.n_layers, cfg.n_heads, cfg.prompt_len, opt_len=opt_len, max_batch=B,
                   rank=r)
    eng.init_params(cfg.init_seed, cfg.init_scale)
    eng.sample_v(42, step, 50)
    eng.sample_u(42, step)
    params = R.init_params(cfg)
    A = {lid: 1e-3 * R.gaussian(43, step, lid, R.ROLE_U, eng.shapes[lid][0], r) for lid in eng.lids}
    eng.set_slot(2, eng.join(2, A))
    Uh, Vh = eng.split(0, eng.get_slot(0)), eng.split(1, eng.get_slot(1))
    eng.prepare_probe(eps, 0)
    nll = eng.score(tokens, np.stack([gold, gold]), nsign=2)
    for si, sign in enumerate((1, -1)):
        eff = dict(params)
        for lid in eng.lids:
            eff[lid] = R.compose(params[lid], A[lid], Vh[lid], Uh[lid], sign, eps)
        ref = R.forward_nll(eff, cfg, tokens, gold)
        np.testing.assert_allclose(nll[si], ref, atol=2e-2 * opt_len, rtol=0)
    eng.close()
