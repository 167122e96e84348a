#!/usr/bin/env python
"""The paper's Phase 6 setting on one B200: OPT-1.3B, B=16, a
MeZO-style dense baseline vs high-rank factorized ZO (r = 128 / 256 / 512) -- per-step
device time of

* dense MeZO as the conventional training loop (baseline_loop.run_baseline, estimator
  "dense_mezo": a dense Role.DENSE_Z direction per weight regenerated every step, probe /
  restore / update written into the weights, one forward per sign), and
* the factorized estimator on the serving path (zo_step_async: rank-r directions, both
  probes in one fused forward, the dense update U V^T / sqrt(r) into the base) -- with
  the bit-exact float64 update ("exact") and the tensor-core update over fp32 masters
  ("tensor", zo_set_update_mode 1).

    python scripts/phase6.py [--model opt-1.3b] [--steps 10]
"""
import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def timed(fn, steps, warm=2):
    import torch
    for t in range(warm):
        fn(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(warm, warm + steps):
        fn(t)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    import torch
    from bench import MODELS
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.engine import ZoEngine
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-1.3b", choices=sorted(MODELS))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--ranks", default="128,256,512")
    ap.add_argument("--modes", default="exact,tensor", help="factorized dense update modes to time")
    a = ap.parse_args()
    mdl = MODELS[a.model]
    B, T = 16, 64
    task = M.generate_task(M.TaskConfig(seed=11, vocab=mdl["vocab"], prompt_len=T - 1, train_size=256,
                                        dev_size=2, val_size=2))
    toks, golds = [], []
    for t in range(a.steps + 2):
        seq, gold = M.sample_minibatch(task, "train", 42, t, B).sequences()
        toks.append(seq)
        golds.append(gold)
    d_tok = torch.from_numpy(np.stack(toks).astype(np.int32)).cuda()
    d_gold = torch.from_numpy(np.stack(golds).astype(np.int32)).cuda()
    out = {"model": a.model, "batch": B, "seq": T}

    eng = ZoEngine(mdl["vocab"], mdl["dim"], mdl["n_layers"], mdl["n_heads"], T - 1, max_batch=B, rank=2,
                   estimator="dense_mezo")
    eng.init_params(7, 0.02)
    out["dense_mezo_materialising_ms"] = timed(
        lambda t: eng.baseline_step_async(42, t, 1, 1e-3, 1e-7, False, False, d_tok[t].data_ptr(),
                                          d_gold[t].data_ptr(), B), a.steps)
    eng.close()
    for r in [int(x) for x in a.ranks.split(",")]:
        for mode in a.modes.split(","):
            eng = ZoEngine(mdl["vocab"], mdl["dim"], mdl["n_layers"], mdl["n_heads"], T - 1, max_batch=B, rank=r,
                           estimator="factorized_sqrt_r")
            eng.init_params(7, 0.02)
            eng.set_update_mode(mode)
            ms = timed(lambda t: eng.step_async(42, t, 1, 1e-3, 1e-7, False, d_tok[t].data_ptr(),
                                                d_gold[t].data_ptr(), B), a.steps)
            sfx = "" if mode == "exact" else "_tensor"
            out[f"factorized_r{r}{sfx}_serving_ms"] = ms
            out[f"speedup_r{r}{sfx}"] = out["dense_mezo_materialising_ms"] / ms
            eng.close()
            print(json.dumps(out), flush=True)
    os.makedirs(os.path.join(HERE, "gpurun_out"), exist_ok=True)
    with open(os.path.join(HERE, "gpurun_out", "phase6.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
