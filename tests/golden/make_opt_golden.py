"""Golden fixture for the OPT-architecture variant, from Hugging
Face transformers' own OPT implementation (transformers 5.5,
transformers/models/opt/modeling_opt.py) run in float64 on CPU in the build
container.  The GPU box does not need transformers: it reads the committed JSON.

    python tests/golden/make_opt_golden.py

forward_opt_micro.json: per-example option NLLs (row prompt_len-1, model.py:202-215
semantics) of OPTForCausalLM at composed weights W0 + A V^T + sign*eps*U V^T for
sign -1/0/+1 (every 2-D param incl. pos_embed, the zoserve matrix_ids rule), with
non-trivial biases / LN params; all params are regenerable from the recipe.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

MICRO_OPT = dict(vocab=64, dim=32, n_layers=2, n_heads=2, prompt_len=16, init_seed=7, init_scale=0.08,
                 arch="opt", max_positions=32)
MICRO_TASK = dict(seed=11, vocab=64, prompt_len=16, train_size=64, dev_size=8, val_size=8)


def opt_params(R, cfg, vec_seed=5, vec_scale=0.05):
    """init_params(opt) + biases / LN params from Role.INIT streams of `vec_seed`
    (1-D values: scale 1 + s*z, shift and bias s*z) so the bias and LN paths are exercised."""
    p = R.init_params(cfg)
    for k in sorted(p):
        if p[k].ndim == 1:
            z = R.gaussian(vec_seed, 0, k, R.ROLE_INIT, p[k].shape[0], 1).reshape(-1)
            p[k] = (1.0 + vec_scale * z) if k.endswith(".scale") else vec_scale * z
    return p


def compose_all(R, params, zseed, step, rank, a_scale, a_seed, sign, eps):
    eff = dict(params)
    for lid in sorted(k for k, v in params.items() if v.ndim == 2):
        m, n = params[lid].shape
        u = R.gaussian(zseed, step, lid, R.ROLE_U, m, rank)
        v = R.gaussian(zseed, (step // 50) * 50, lid, R.ROLE_V, n, rank)
        a = a_scale * R.gaussian(a_seed, step, lid, R.ROLE_U, m, rank)
        eff[lid] = R.compose(params[lid], a, v, u, sign, eps)
    return eff


def hf_nll(cfg, eff, tokens, gold):
    import torch
    from transformers import OPTConfig, OPTForCausalLM

    from paper_2605_28760_b200.opt_io import params_to_hf
    hc = OPTConfig(vocab_size=cfg.vocab, hidden_size=cfg.dim, num_hidden_layers=cfg.n_layers, ffn_dim=4 * cfg.dim,
                   num_attention_heads=cfg.n_heads, max_position_embeddings=cfg.max_positions,
                   word_embed_proj_dim=cfg.dim, do_layer_norm_before=True, enable_bias=True,
                   activation_function="relu", dropout=0.0, attention_dropout=0.0, pad_token_id=1,
                   tie_word_embeddings=True)
    model = OPTForCausalLM(hc).double().eval()
    sd = {k: torch.from_numpy(v) for k, v in params_to_hf(eff, cfg).items()}
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected and all("lm_head" in m for m in missing), (missing, unexpected)
    with torch.no_grad():
        logits = model(input_ids=torch.from_numpy(tokens)).logits.numpy()
    B = tokens.shape[0]
    nll = np.zeros(B)
    for j in range(gold.shape[1]):
        row = logits[:, cfg.prompt_len - 1 + j, :]
        m = row.max(axis=-1)
        lse = m + np.log(np.exp(row - m[:, None]).sum(axis=-1))
        nll += lse - row[np.arange(B), gold[:, j]]
    return nll


def main():
    from oracle import reference as R
    cfg = R.ModelCfg(**MICRO_OPT)
    splits = R.generate_task(R.TaskCfg(**MICRO_TASK))
    B, zseed, step, rank, a_scale, eps = 8, 42, 0, 2, 1e-3, 1e-3
    prompts, golds, idx = R.sample_minibatch(splits, "train", zseed, step, B)
    gold = np.array([[cfg.vocab - 2], [cfg.vocab - 1]], dtype=np.int64)[golds]
    tokens = np.concatenate([prompts, gold], axis=1)
    params = opt_params(R, cfg)
    res = {"model": MICRO_OPT, "task": MICRO_TASK, "batch": B, "zseed": zseed, "step": step, "rank": rank,
           "a_scale": a_scale, "a_seed": zseed + 1, "epsilon": eps, "vec_seed": 5, "vec_scale": 0.05,
           "params_digest": R.params_digest(params), "tokens": tokens.tolist(), "nll": {},
           "generator": "transformers OPTForCausalLM (float64, CPU)"}
    for sign in (-1, 0, 1):
        eff = compose_all(R, params, zseed, step, rank, a_scale, zseed + 1, sign, eps)
        res["nll"][str(sign)] = [float(v) for v in hf_nll(cfg, eff, tokens, gold)]
    with open(os.path.join(HERE, "forward_opt_micro.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
