"""BASELINE config 4: an OPT-13B-shaped LoZO run through the public API
(run_serving_path: host minibatches, device step, folds every nu, async U/V digests,
dev evals), writing the trajectory in the reference's JSON-lines format.

    python scripts/long_run.py --model opt-13b --steps 20000 --eval-every 2000 --out gpurun_out/long
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

MODELS = {
    "opt-125m": dict(vocab=50272, dim=768, n_layers=12, n_heads=12),
    "opt-1.3b": dict(vocab=50272, dim=2048, n_layers=24, n_heads=32),
    "opt-6.7b": dict(vocab=50272, dim=4096, n_layers=32, n_heads=32),
    "opt-13b": dict(vocab=50272, dim=5120, n_layers=40, n_heads=40),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-13b", choices=sorted(MODELS))
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--eval-every", type=int, default=2000)
    ap.add_argument("--dev-size", type=int, default=64)
    ap.add_argument("--lr", type=float, default=1e-7)
    ap.add_argument("--out", default="gpurun_out/long")
    ap.add_argument("--estimator", default="lozo_lazy", choices=["lozo_lazy", "factorized_sqrt_r"],
                    help="factorized_sqrt_r with --rank 128 = BASELINE config 5 (1000 steps)")
    ap.add_argument("--rank", type=int, default=2)
    ap.add_argument("--digests", choices=["auto", "on", "off"], default="auto",
                    help="U/V digests on the host pool; auto = every step up to rank 8, an audit of every "
                         "--digest-every-th step above (r = 128 means 3.4 GB of directions per step, "
                         "SURVEY.md §0 fact 7)")
    ap.add_argument("--digest-every", type=int, default=50, help="audit period above rank 8 (--digests auto)")
    ap.add_argument("--dense-update", default="exact", choices=["exact", "tensor"],
                    help="factorized dense update: float64 bit-exact, or tcgen05 over fp32 masters (zob200.h)")
    a = ap.parse_args()
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.runtime import run_serving_path
    from paper_2605_28760_b200.zo_engine import ZoConfig, write_trajectory
    mdl = MODELS[a.model]
    mcfg = M.ModelConfig(prompt_len=63, init_seed=7, init_scale=0.02, **mdl)
    task = M.generate_task(M.TaskConfig(seed=11, vocab=mdl["vocab"], prompt_len=63, train_size=1000,
                                        dev_size=a.dev_size, val_size=8))
    zcfg = ZoConfig(seed=42, epsilon=1e-3, learning_rate=a.lr, rank=a.rank, nu=50, batch_size=16,
                    estimator=a.estimator)
    t0 = time.perf_counter()
    digests = a.digests != "off"
    every = a.digest_every if (a.digests == "auto" and a.rank > 8) else 1
    params = M.init_params(mcfg, precision="fp16", max_batch=16)
    eng = params.bind(zcfg.rank, zcfg.estimator, zcfg.batch_size, 1, zcfg.scope)
    if a.estimator == "factorized_sqrt_r":
        eng.set_update_mode(a.dense_update)
    run = run_serving_path(mcfg, task, zcfg, a.steps, precision="fp16", eval_every=a.eval_every,
                           compute_param_digests=False, digests=digests, digest_every=every, params=params)
    wall = time.perf_counter() - t0
    os.makedirs(a.out, exist_ok=True)
    tag = f"{a.model}_{a.steps}" + ("" if a.estimator == "lozo_lazy" else f"_fact_r{a.rank}")
    write_trajectory(os.path.join(a.out, f"traj_{tag}.jsonl"),
                     {"model": mdl, "steps": a.steps, "zo_digest": zcfg.digest()}, run.trajectory,
                     {"eval_loss": run.eval_curve[-1].loss, "eval_acc": run.eval_curve[-1].acc})
    summary = {"model": a.model, "estimator": a.estimator, "rank": a.rank, "dense_update": a.dense_update,
               "digest_every": every, "steps": run.steps_completed, "train_wall_s": run.train_wall_s,
               "steps_per_s_train": run.steps_completed / run.train_wall_s, "total_wall_s": wall,
               "meter": run.meter.to_dict(), "eval_curve": [p.to_dict() for p in run.eval_curve],
               "last_record": run.trajectory[-1].to_dict()}
    with open(os.path.join(a.out, f"summary_{tag}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: summary[k] for k in ("model", "steps", "train_wall_s", "steps_per_s_train")}))


if __name__ == "__main__":
    main()
