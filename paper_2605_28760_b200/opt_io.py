"""Real OPT checkpoints on the engine.

Maps a Hugging Face ``OPTForCausalLM`` / ``OPTModel`` state dict (names of
transformers/models/opt/modeling_opt.py) to this package's parameter ids in the
reference's (in, out) layout, and back:

===============================================  ==========================
HF name (``model.decoder.`` prefix)               here
===============================================  ==========================
embed_tokens.weight [V, d]                        embed [V, d] (tied head)
embed_positions.weight [max_pos + 2, d]           pos_embed
layers.i.self_attn.{q,k,v}_proj.weight [d, d]     blk{i}.qkv [d, 3d] = [Wq^T | Wk^T | Wv^T]
layers.i.self_attn.{q,k,v}_proj.bias              blk{i}.qkv.bias [3d]
layers.i.self_attn.out_proj.{weight,bias}         blk{i}.attn_out (^T), .bias
layers.i.self_attn_layer_norm.{weight,bias}       blk{i}.ln1.scale / .shift
layers.i.fc1.{weight,bias} / fc2                  blk{i}.ff_up (^T) / ff_down (^T), .bias
layers.i.final_layer_norm.{weight,bias}           blk{i}.ln2.scale / .shift
final_layer_norm.{weight,bias}                    ln_f.scale / .shift
===============================================  ==========================

The variants this decoder does not cover (OPT-350m's ``project_in/out`` and
post-LN) are rejected.  Tensors may be torch tensors or numpy arrays; the
returned host params are float64 and feed ``DeviceParams(cfg, host=...)``.
"""
from __future__ import annotations

import numpy as np

from .errors import ConfigError, InputError
from .engine import resolve_precision
from .model import ModelConfig

__all__ = ["config_from_hf", "params_from_hf", "params_to_hf", "load_hf_opt"]


def _np(t) -> np.ndarray:
    if hasattr(t, "detach"):
        t = t.detach().to("cpu")
        if str(t.dtype) in ("torch.bfloat16", "torch.float16"):
            t = t.float()
        t = t.numpy()
    return np.asarray(t, dtype=np.float64)


def config_from_hf(hf_config, prompt_len: int, init_seed: int = 7, init_scale: float = 0.02) -> ModelConfig:
    """ModelConfig(arch="opt") for an ``OPTConfig`` (or its dict)."""
    g = hf_config if isinstance(hf_config, dict) else hf_config.to_dict()
    d = int(g["hidden_size"])
    if int(g.get("word_embed_proj_dim", d)) != d:
        raise ConfigError("OPT variants with project_in/project_out (word_embed_proj_dim != hidden_size) "
                          "are not supported")
    if not g.get("do_layer_norm_before", True):
        raise ConfigError("post-LN OPT (do_layer_norm_before=False) is not supported")
    if g.get("activation_function", "relu") != "relu":
        raise ConfigError("only the ReLU FFN of OPT is supported")
    if int(g.get("ffn_dim", 4 * d)) != 4 * d:
        raise ConfigError("ffn_dim must be 4 * hidden_size")
    if not g.get("enable_bias", True):
        raise ConfigError("OPT without biases is not supported")
    return ModelConfig(vocab=int(g["vocab_size"]), dim=d, n_layers=int(g["num_hidden_layers"]),
                       n_heads=int(g["num_attention_heads"]), prompt_len=prompt_len, init_seed=init_seed,
                       init_scale=init_scale, arch="opt", max_positions=int(g["max_position_embeddings"]))


def _prefix(sd) -> str:
    for p in ("model.decoder.", "decoder.", ""):
        if p + "embed_tokens.weight" in sd:
            return p
    raise InputError("not an OPT state dict (no embed_tokens.weight)")


def params_from_hf(state_dict, cfg: ModelConfig) -> dict[str, np.ndarray]:
    """Host float64 params (reference layout) from an HF OPT state dict."""
    if cfg.arch != "opt":
        raise ConfigError("params_from_hf needs ModelConfig(arch='opt')")
    p = _prefix(state_dict)
    sd = {k[len(p):]: v for k, v in state_dict.items() if k.startswith(p)}
    out = {"embed": _np(sd["embed_tokens.weight"]), "pos_embed": _np(sd["embed_positions.weight"]),
           "ln_f.scale": _np(sd["final_layer_norm.weight"]), "ln_f.shift": _np(sd["final_layer_norm.bias"])}
    for i in range(cfg.n_layers):
        L, b = f"layers.{i}.", f"blk{i}."
        a = L + "self_attn."
        out[b + "qkv"] = np.concatenate([_np(sd[a + f"{x}_proj.weight"]).T for x in "qkv"], axis=1)
        out[b + "qkv.bias"] = np.concatenate([_np(sd[a + f"{x}_proj.bias"]) for x in "qkv"])
        out[b + "attn_out"] = _np(sd[a + "out_proj.weight"]).T
        out[b + "attn_out.bias"] = _np(sd[a + "out_proj.bias"])
        out[b + "ln1.scale"] = _np(sd[L + "self_attn_layer_norm.weight"])
        out[b + "ln1.shift"] = _np(sd[L + "self_attn_layer_norm.bias"])
        out[b + "ff_up"] = _np(sd[L + "fc1.weight"]).T
        out[b + "ff_up.bias"] = _np(sd[L + "fc1.bias"])
        out[b + "ff_down"] = _np(sd[L + "fc2.weight"]).T
        out[b + "ff_down.bias"] = _np(sd[L + "fc2.bias"])
        out[b + "ln2.scale"] = _np(sd[L + "final_layer_norm.weight"])
        out[b + "ln2.shift"] = _np(sd[L + "final_layer_norm.bias"])
    from .model import matrix_shapes
    for lid, shp in matrix_shapes(cfg).items():
        if out[lid].shape != shp:
            raise InputError(f"{lid}: checkpoint shape {out[lid].shape} != config shape {shp}")
    return {k: np.ascontiguousarray(v) for k, v in out.items()}


def params_to_hf(params, cfg: ModelConfig, prefix: str = "model.decoder.") -> dict[str, np.ndarray]:
    """Inverse of ``params_from_hf`` (float64 numpy; ``lm_head.weight`` tied)."""
    d = cfg.dim
    g = {k: np.asarray(params[k], dtype=np.float64) for k in params}
    sd = {prefix + "embed_tokens.weight": g["embed"], prefix + "embed_positions.weight": g["pos_embed"],
          prefix + "final_layer_norm.weight": g["ln_f.scale"], prefix + "final_layer_norm.bias": g["ln_f.shift"]}
    for i in range(cfg.n_layers):
        L, b = prefix + f"layers.{i}.", f"blk{i}."
        a = L + "self_attn."
        for j, x in enumerate("qkv"):
            sd[a + f"{x}_proj.weight"] = g[b + "qkv"][:, j * d:(j + 1) * d].T.copy()
            sd[a + f"{x}_proj.bias"] = g[b + "qkv.bias"][j * d:(j + 1) * d].copy()
        sd[a + "out_proj.weight"] = g[b + "attn_out"].T.copy()
        sd[a + "out_proj.bias"] = g[b + "attn_out.bias"]
        sd[L + "self_attn_layer_norm.weight"] = g[b + "ln1.scale"]
        sd[L + "self_attn_layer_norm.bias"] = g[b + "ln1.shift"]
        sd[L + "fc1.weight"] = g[b + "ff_up"].T.copy()
        sd[L + "fc1.bias"] = g[b + "ff_up.bias"]
        sd[L + "fc2.weight"] = g[b + "ff_down"].T.copy()
        sd[L + "fc2.bias"] = g[b + "ff_down.bias"]
        sd[L + "final_layer_norm.weight"] = g[b + "ln2.scale"]
        sd[L + "final_layer_norm.bias"] = g[b + "ln2.shift"]
    if prefix.startswith("model."):
        sd["lm_head.weight"] = g["embed"]
    return sd


def load_hf_opt(model_or_state_dict, prompt_len: int, precision: str = "fp16", max_batch: int = 16,
                device: int = 0, hf_config=None):
    """(ModelConfig, DeviceParams) for a transformers OPT model (or its state dict +
    ``hf_config``), ready for run_serving_path / lozo_step."""
    from .model import DeviceParams
    if hasattr(model_or_state_dict, "state_dict"):
        hf_config = model_or_state_dict.config if hf_config is None else hf_config
        sd = model_or_state_dict.state_dict()
    else:
        sd = model_or_state_dict
    if hf_config is None:
        raise ConfigError("hf_config is required with a bare state dict")
    cfg = config_from_hf(hf_config, prompt_len)
    host = params_from_hf(sd, cfg)
    return cfg, DeviceParams(cfg, host=host, precision=resolve_precision(precision),
                             max_batch=max_batch, device=device)
