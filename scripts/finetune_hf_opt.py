#!/usr/bin/env python
"""LoZO fine-tuning of a Hugging Face OPT checkpoint on the engine (the OPT decoder,
ModelConfig(arch="opt")).

    python scripts/finetune_hf_opt.py --model /path/to/opt-1.3b --steps 2000
    python scripts/finetune_hf_opt.py --random tiny --steps 200       # offline: random init

Loads the checkpoint through transformers, maps it with opt_io.load_hf_opt, runs the
reference-shaped run_serving_path (device-resident LoZO, folds every nu, dev evals) on the
synthetic marker task of the reference (model.py:312-403), prints the eval curve and the
throughput, and checks the loaded weights against transformers' own forward on one batch.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

RANDOM = {  # offline smoke configurations (random init)
    "tiny": dict(vocab_size=512, hidden_size=128, num_hidden_layers=2, ffn_dim=512, num_attention_heads=4,
                 max_position_embeddings=128),
    "opt-125m": dict(vocab_size=50272, hidden_size=768, num_hidden_layers=12, ffn_dim=3072, num_attention_heads=12,
                     max_position_embeddings=2048),
}


def main():
    ap = argparse.ArgumentParser()
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--model", help="transformers OPT checkpoint directory / id available locally")
    src.add_argument("--random", choices=sorted(RANDOM), help="random-init OPT config (no download)")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--prompt-len", type=int, default=63)
    ap.add_argument("--lr", type=float, default=1e-6)
    ap.add_argument("--eps", type=float, default=1e-3)
    ap.add_argument("--nu", type=int, default=50)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--eval-every", type=int, default=100)
    ap.add_argument("--precision", default="fp16", choices=["fp16", "bf16"])
    a = ap.parse_args()

    import torch
    import transformers as tr

    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.opt_io import load_hf_opt
    from paper_2605_28760_b200.runtime import run_serving_path
    from paper_2605_28760_b200.zo_engine import ZoConfig

    if a.model:
        hf = tr.OPTForCausalLM.from_pretrained(a.model, torch_dtype=torch.float32)
    else:
        torch.manual_seed(0)
        hf = tr.OPTForCausalLM(tr.OPTConfig(**RANDOM[a.random], word_embed_proj_dim=RANDOM[a.random]["hidden_size"],
                                            do_layer_norm_before=True, activation_function="relu"))
    hf.eval()
    t0 = time.perf_counter()
    mcfg, params = load_hf_opt(hf, prompt_len=a.prompt_len, precision=a.precision, max_batch=a.batch)
    t_load = time.perf_counter() - t0
    task = M.generate_task(M.TaskConfig(seed=11, vocab=mcfg.vocab, prompt_len=a.prompt_len, train_size=1000,
                                        dev_size=64, val_size=64))

    # the loaded weights score like transformers itself (sign 0, one batch)
    batch = M.sample_minibatch(task, "train", 42, 0, min(8, a.batch))
    tokens, gold = batch.sequences()
    got = M.forward_nll(params, mcfg, batch.prompts, gold)
    with torch.no_grad():
        logits = hf.double()(input_ids=torch.from_numpy(np.asarray(tokens))).logits.numpy()
    row = logits[:, a.prompt_len - 1, :]
    mx = row.max(axis=-1)
    ref = mx + np.log(np.exp(row - mx[:, None]).sum(axis=-1)) - row[np.arange(len(gold)), gold[:, 0]]
    hf.float()

    zcfg = ZoConfig(seed=42, epsilon=a.eps, learning_rate=a.lr, rank=2, nu=a.nu, batch_size=a.batch)
    run = run_serving_path(mcfg, task, zcfg, a.steps, eval_every=a.eval_every, params=params)
    out = {"model": a.model or f"random:{a.random}", "arch": mcfg.arch, "dim": mcfg.dim, "n_layers": mcfg.n_layers,
           "load_s": t_load, "max_abs_nll_vs_transformers": float(np.max(np.abs(got - ref))),
           "steps": run.steps_completed, "steps_per_s": run.steps_completed / run.train_wall_s,
           "eval_curve": [e.to_dict() for e in run.eval_curve]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
