#!/usr/bin/env python
"""Run a few eager materialising-loop steps (baseline_loop.run_baseline's device
path, zo_baseline_step_async) at a BASELINE shape -- the target of the ncu launch
list / capture of the comparand's kernels (profiles/capture.sh).

    python scripts/materialise_steps.py [--model opt-13b] [--steps 2] [--recompute]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from bench import MODELS
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.engine import ZoEngine
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-13b", choices=sorted(MODELS))
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--recompute", action="store_true")
    a = ap.parse_args()
    mdl = MODELS[a.model]
    B, T = 16, 64
    eng = ZoEngine(mdl["vocab"], mdl["dim"], mdl["n_layers"], mdl["n_heads"], T - 1, max_batch=B, rank=2)
    eng.init_params(7, 0.02)
    task = M.generate_task(M.TaskConfig(seed=11, vocab=mdl["vocab"], prompt_len=T - 1, train_size=64, dev_size=2,
                                        val_size=2))
    for t in range(a.steps):
        seq, gold = M.sample_minibatch(task, "train", 42, t, B).sequences()
        tk = torch.from_numpy(np.ascontiguousarray(seq, dtype=np.int32)).cuda()
        gd = torch.from_numpy(np.ascontiguousarray(gold, dtype=np.int32)).cuda()
        t0 = time.perf_counter()
        eng.baseline_step_async(42, t, 50, 1e-3, 1e-7, False, a.recompute, tk.data_ptr(), gd.data_ptr(), B)
        eng.synchronize()
        print(f"step {t}: {1e3 * (time.perf_counter() - t0):.1f} ms  out4={eng.read_out4()}", flush=True)


if __name__ == "__main__":
    main()
