"""OPT-architecture variant on CPU: the oracle's OPT forward is
pinned to Hugging Face transformers' OPTForCausalLM (tests/golden/forward_opt_micro.json,
written by make_opt_golden.py), the checkpoint mapping round-trips, and the
reference-architecture ModelConfig digest is unchanged by the new fields."""
import json
import os
import sys

import numpy as np
import pytest

from oracle import reference as R

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from make_opt_golden import compose_all, opt_params  # noqa: E402


def _load(golden_dir):
    with open(os.path.join(golden_dir, "forward_opt_micro.json")) as f:
        return json.load(f)


def test_oracle_opt_forward_matches_hf(golden_dir):
    g = _load(golden_dir)
    cfg = R.ModelCfg(**g["model"])
    params = opt_params(R, cfg, g["vec_seed"], g["vec_scale"])
    assert R.params_digest(params) == g["params_digest"]
    tokens = np.asarray(g["tokens"])
    gold = tokens[:, cfg.prompt_len:]
    for sign in (-1, 0, 1):
        eff = compose_all(R, params, g["zseed"], g["step"], g["rank"], g["a_scale"], g["a_seed"], sign,
                          g["epsilon"])
        nll = R.forward_nll(eff, cfg, tokens, gold)
        np.testing.assert_allclose(nll, g["nll"][str(sign)], rtol=0, atol=1e-11)


def test_hf_mapping_round_trip():
    from paper_2605_28760_b200.model import ModelConfig, matrix_shapes
    from paper_2605_28760_b200.opt_io import params_from_hf, params_to_hf
    cfg = ModelConfig(vocab=64, dim=32, n_layers=2, n_heads=2, prompt_len=16, arch="opt", max_positions=32)
    rc = R.ModelCfg(**{k: getattr(cfg, k) for k in R.ModelCfg.__dataclass_fields__})
    p = opt_params(R, rc)
    sd = params_to_hf(p, cfg)
    assert sd["model.decoder.layers.1.self_attn.k_proj.weight"].shape == (32, 32)
    assert "lm_head.weight" in sd
    back = params_from_hf(sd, cfg)
    assert set(back) == set(p)
    for k in p:
        np.testing.assert_array_equal(back[k], p[k])
    assert set(matrix_shapes(cfg)) == {k for k in p if p[k].ndim == 2}


def test_hf_config_mapping_and_rejections():
    from paper_2605_28760_b200.errors import ConfigError
    from paper_2605_28760_b200.opt_io import config_from_hf
    base = dict(vocab_size=50272, hidden_size=5120, num_hidden_layers=40, num_attention_heads=40, ffn_dim=20480,
                max_position_embeddings=2048, word_embed_proj_dim=5120, do_layer_norm_before=True,
                activation_function="relu", enable_bias=True)
    cfg = config_from_hf(base, prompt_len=63)
    assert (cfg.dim, cfg.n_layers, cfg.n_heads, cfg.max_positions, cfg.arch) == (5120, 40, 40, 2048, "opt")
    for bad in (dict(word_embed_proj_dim=512), dict(do_layer_norm_before=False), dict(activation_function="gelu")):
        with pytest.raises(ConfigError):
            config_from_hf({**base, **bad}, prompt_len=63)


def test_reference_arch_digest_unchanged(golden_dir):
    from paper_2605_28760_b200.model import ModelConfig
    with open(os.path.join(golden_dir, "traj_micro_lozo.jsonl")) as f:
        h = json.loads(f.readline())
    from paper_2605_28760_b200.zo_engine import ZoConfig  # noqa: F401
    mcfg = ModelConfig(**h["model"])
    # zoserve arch: the digest covers exactly the reference's ModelConfig fields
    ref = json.dumps(h["model"], sort_keys=True)
    from paper_2605_28760_b200.numerics import digest_hex, digest_text
    assert mcfg.digest() == digest_hex(digest_text(ref))
    assert ModelConfig(**h["model"], arch="opt").digest() != mcfg.digest()
