"""Generate the golden fixtures under tests/golden/ from the reference itself.

Run in the build container (the reference is importable read-only from
/root/reference/pkg/src; it does NOT exist on the GPU box, which only reads
the committed JSON/JSONL this script writes):

    python tests/golden/make_golden.py            # fast fixtures (~1 min)
    python tests/golden/make_golden.py --opt125m  # + OPT-125m-dims steps (~2 min)
    python tests/golden/make_golden.py --config1  # BASELINE config 1, 50 steps (~20 min)
    python tests/golden/make_golden.py --real32   # real32 trajectories (micro, small)

Fixtures
  streams.json      sample_gaussian digests / heads / u64 consumption for a key
                    grid incl. OPT-13B slot shapes (numerics.py:139-168)
  fnv.json          FNV-1a-64 vectors (numerics.py:60-124)
  forward_*.json    per-example option NLLs of _forward_logits/_option_nll
                    under composed probes (model.py:170-244, adapter.py:200-234)
  traj_*.jsonl      run_serving_path trajectories (runtime.py:253-359) with
                    header digests, per-step L+/L-/c/beta/u,v digests and the
                    final params digest, written by zoserve.write_trajectory
  traj_*baseline*   run_baseline trajectories (baseline_loop.py:122-239), the
                    materialising loop: cached and recompute products,
                    factorized and full scope
  adapter_rich.zoad ZOAD adapter file (+ .manifest.json) written by the
                    reference's save_adapter for a state with frozen, window
                    and probe slots (adapter.py:279-415)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import zoserve  # noqa: F401
    return zoserve


def streams():
    _ref()
    from zoserve.numerics import Role, StreamKey, digest_array, digest_hex, digest_text, sample_gaussian

    grid = [
        (42, 7, "blk0.qkv", Role.U, 768, 2),
        (42, 0, "blk0.qkv", Role.V, 2304, 2),
        (42, 0, "embed", Role.U, 50272, 2),
        (42, 50, "embed", Role.V, 768, 2),
        (42, 3, "blk39.ff_down", Role.U, 20480, 2),
        (42, 3, "blk39.ff_up", Role.V, 20480, 2),
        (42, 19999, "blk17.qkv", Role.U, 5120, 2),
        (42, 19950, "blk17.qkv", Role.V, 15360, 2),
        (42, 5, "blk0.ff_up", Role.U, 2048, 128),
        (7, 0, "blk0.ff_up", Role.INIT, 768, 3072),
        (7, 0, "embed", Role.INIT, 1000, 768),
        (0, 0, "", Role.U, 1, 1),
        (1, 123456789012, "x", Role.MINIBATCH, 3, 5),
        (2**40 + 3, 2**33, "blk3.attn_out", Role.DENSE_Z, 64, 64),
    ]
    out = []
    for seed, step, lid, role, r, c in grid:
        key = StreamKey(seed, step, lid, role)
        g = key.generator()
        kk = g.bit_generator.state["state"]["key"]
        x = g.standard_normal((r, c))
        st = g.bit_generator.state
        consumed = 4 * (int(st["state"]["counter"][0]) - 1) + int(st["buffer_pos"])
        assert np.array_equal(x, sample_gaussian(key, r, c))
        out.append({
            "seed": seed, "step": step, "layer_id": lid, "role": int(role), "rows": r, "cols": c,
            "lid_hash": f"{digest_text(lid):016x}",
            "key": [f"{int(kk[0]):016x}", f"{int(kk[1]):016x}"],
            "digest": digest_hex(digest_array(x)),
            "head": [float(v).hex() for v in x.reshape(-1)[:6]],
            "tail": [float(v).hex() for v in x.reshape(-1)[-3:]],
            "u64_consumed": consumed,
            "n_tail": int(np.sum(np.abs(x) > 3.6541528853610088)),
        })
    with open(os.path.join(OUT, "streams.json"), "w") as f:
        json.dump(out, f, indent=1)


def fnv():
    _ref()
    from zoserve.numerics import digest_array, digest_bytes, digest_hex, digest_text

    vec = {
        "empty": digest_hex(digest_bytes(b"")),
        "a": digest_hex(digest_bytes(b"a")),
        "foobar": digest_hex(digest_bytes(b"foobar")),
        "params": digest_hex(digest_text("params")),
        "arange8": digest_hex(digest_array(np.arange(8, dtype=np.float64))),
        "chain": digest_hex(digest_array(np.array([1.5, -2.25]), digest_text("blk0.qkv"))),
    }
    with open(os.path.join(OUT, "fnv.json"), "w") as f:
        json.dump(vec, f, indent=1)


def forward_fixture(name, mcfg_kw, tcfg_kw, B, zseed=42, step=0, rank=2, a_scale=1e-3):
    """Per-example NLLs at sign -1/0/+1 with a window slot A (random, small) + probe U."""
    _ref()
    from zoserve.adapter import AdapterState, LoraSlot
    from zoserve.model import ModelConfig, TaskConfig, _effective_weights, _forward_logits, _option_nll
    from zoserve.model import generate_task, init_params, matrix_ids, params_digest, sample_minibatch
    from zoserve.zo_engine import lozo_direction

    mcfg = ModelConfig(**mcfg_kw)
    task = generate_task(TaskConfig(**tcfg_kw))
    params = init_params(mcfg)
    batch = sample_minibatch(task, "train", zseed, step, B)
    state = AdapterState(epsilon=1e-3)
    for lid in matrix_ids(params):
        m, n = params[lid].shape
        u, v = lozo_direction(zseed, step, lid, m, n, rank, 50)
        a = a_scale * lozo_direction(zseed + 1, step, lid, m, n, rank, 50)[0]
        e = state.ensure_entry(lid, m, n)
        e.window_slot = LoraSlot(a, v.copy(), 1.0)
        state.set_probe(lid, u, v)
    gold = batch.option_array()[batch.golds]
    seq = np.concatenate([batch.prompts, gold], axis=1)
    res = {"model": mcfg_kw, "task": tcfg_kw, "batch": B, "zseed": zseed, "step": step,
           "rank": rank, "a_scale": a_scale, "a_seed": zseed + 1, "epsilon": 1e-3,
           "params_digest": params_digest(params), "indices": batch.indices.tolist(),
           "tokens": seq.tolist(), "nll": {}}
    for prec in ("real64", "real32"):
        dt = np.float64 if prec == "real64" else np.float32
        for sign in (-1, 0, 1):
            state.set_sign(sign)
            eff = _effective_weights(params, state.view(), np.dtype(dt))
            nll = _option_nll(_forward_logits(eff, mcfg, seq), gold, mcfg.prompt_len)
            res["nll"][f"{prec}:{sign}"] = [float(v) for v in nll.astype(np.float64)]
    state.set_sign(0)
    with open(os.path.join(OUT, f"forward_{name}.json"), "w") as f:
        json.dump(res, f, indent=1)


def trajectory(name, mcfg_kw, tcfg_kw, zcfg_kw, steps, precision="real64"):
    _ref()
    from zoserve.model import ModelConfig, TaskConfig, generate_task
    from zoserve.runtime import run_serving_path
    from zoserve.zo_engine import ZoConfig, write_trajectory

    mcfg = ModelConfig(**mcfg_kw)
    task = generate_task(TaskConfig(**tcfg_kw))
    zcfg = ZoConfig(**zcfg_kw)
    run = run_serving_path(mcfg, task, zcfg, steps, precision=precision, eval_every=10**9)
    header = {"model": mcfg_kw, "task": tcfg_kw, "zo": zcfg_kw, "steps": steps,
              "precision": precision, "model_digest": run.model_digest,
              "task_digest": run.task_digest, "zo_digest": zcfg.digest()}
    final = {"final_params_digest": run.final_params_digest,
             "pre_fold_params_digest": run.pre_fold_params_digest,
             "pre_fold_state_digest": run.pre_fold_digest,
             "eval_loss": run.eval_curve[-1].loss, "eval_acc": run.eval_curve[-1].acc}
    write_trajectory(os.path.join(OUT, f"traj_{name}.jsonl"), header, run.trajectory, final)


MICRO = dict(vocab=64, dim=32, n_layers=2, n_heads=2, prompt_len=16, init_seed=7, init_scale=0.08)
MICRO_TASK = dict(seed=11, vocab=64, prompt_len=16, train_size=64, dev_size=8, val_size=8)
SMALL = dict(vocab=512, dim=128, n_layers=2, n_heads=2, prompt_len=63, init_seed=7, init_scale=0.02)
SMALL_TASK = dict(seed=11, vocab=512, prompt_len=63, train_size=1000, dev_size=4, val_size=4)
OPT125 = dict(vocab=50272, dim=768, n_layers=12, n_heads=12, prompt_len=63, init_seed=7, init_scale=0.02)
OPT125_TASK = dict(seed=11, vocab=50272, prompt_len=63, train_size=1000, dev_size=2, val_size=2)
# BASELINE config 1 as SURVEY.md §8(c) anchors it (task_digest 7bd7555e57d086df): dev/val 64
OPT125_TASK64 = dict(seed=11, vocab=50272, prompt_len=63, train_size=1000, dev_size=64, val_size=64)


def baseline_trajectory(name, mcfg_kw, tcfg_kw, zcfg_kw, steps, recompute=False, precision="real64"):
    """run_baseline (baseline_loop.py:122-239): the materialising training loop."""
    _ref()
    from zoserve.baseline_loop import run_baseline
    from zoserve.model import ModelConfig, TaskConfig, generate_task
    from zoserve.zo_engine import ZoConfig, write_trajectory

    mcfg = ModelConfig(**mcfg_kw)
    task = generate_task(TaskConfig(**tcfg_kw))
    zcfg = ZoConfig(**zcfg_kw)
    run = run_baseline(mcfg, task, zcfg, steps, precision=precision, eval_every=10**9,
                       recompute_products=recompute)
    header = {"model": mcfg_kw, "task": tcfg_kw, "zo": zcfg_kw, "steps": steps, "precision": precision,
              "recompute_products": recompute, "model_digest": run.model_digest,
              "task_digest": run.task_digest, "zo_digest": zcfg.digest()}
    final = {"final_params_digest": run.final_params_digest, "weight_writes": run.weight_write_count,
             "eval_loss": run.eval_curve[-1].loss, "eval_acc": run.eval_curve[-1].acc}
    write_trajectory(os.path.join(OUT, f"traj_{name}.jsonl"), header, run.trajectory, final)


def baseline_trajectories():
    lozo = dict(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=2, nu=5, batch_size=8)
    baseline_trajectory("micro_baseline", MICRO, MICRO_TASK, lozo, 7)
    baseline_trajectory("micro_baseline_recompute", MICRO, MICRO_TASK, dict(lozo, divide_by_r=True), 7,
                        recompute=True)
    baseline_trajectory("micro_baseline_fact", MICRO, MICRO_TASK,
                        dict(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=8, estimator="factorized_sqrt_r",
                             batch_size=8), 4)
    baseline_trajectory("micro_baseline_full", MICRO, MICRO_TASK, dict(lozo, scope="full"), 4)
    dense = dict(seed=42, epsilon=1e-3, learning_rate=1e-3, estimator="dense_mezo", batch_size=8)
    baseline_trajectory("micro_baseline_dense", MICRO, MICRO_TASK, dense, 4)
    baseline_trajectory("micro_baseline_dense_recompute", MICRO, MICRO_TASK, dense, 4, recompute=True)


def adapter_fixture():
    _ref()
    from zoserve.adapter import AdapterState, LoraSlot, save_adapter

    def slot(m, n, k, scale, seed):
        g = np.random.default_rng(seed)
        return LoraSlot(g.standard_normal((m, k)), g.standard_normal((n, k)), scale)

    st = AdapterState(epsilon=2e-3, perturb_sign=0)
    st.ensure_entry("blk0.qkv", 8, 24)
    st.add_frozen_slot("blk0.qkv", slot(8, 24, 2, 0.5, 20))
    st.entries["blk0.qkv"].window_slot = slot(8, 24, 2, 1.0, 21)
    st.ensure_entry("blk1.ff_down", 32, 8)
    st.entries["blk1.ff_down"].window_slot = slot(32, 8, 2, 1.0, 23)
    st.entries["blk1.ff_down"].perturb_slot = slot(32, 8, 2, 1.0, 24)
    st.ensure_entry("embed", 16, 8)
    st.entries["embed"].perturb_slot = slot(16, 8, 1, 1.0, 22)
    save_adapter(st, os.path.join(OUT, "adapter_rich.zoad"))


def full_scope_trajectories():
    """scope="full": every 1-D param (LN scale/shift) probed and updated densely with
    Role.DENSE_Z directions (zo_engine.py:256-260, 269-295, 412-416, 439-452)."""
    trajectory("micro_full", MICRO, MICRO_TASK,
               dict(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=2, nu=5, batch_size=8, scope="full"), 8)
    trajectory("micro_fact_full", MICRO, MICRO_TASK,
               dict(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=4, estimator="factorized_sqrt_r",
                    batch_size=8, scope="full"), 4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--opt125m", action="store_true")
    ap.add_argument("--config1", action="store_true",
                    help="BASELINE config 1 in full: 50 run_serving_path steps at OPT-125m dims (~20 min)")
    ap.add_argument("--real32", action="store_true", help="real32 trajectories (micro, small)")
    ap.add_argument("--only", default=None, help="regenerate one fixture family (e.g. 'adapter')")
    a = ap.parse_args()
    if a.config1:
        trajectory("opt125m_lozo50", OPT125, OPT125_TASK64,
                   dict(seed=42, epsilon=1e-3, learning_rate=1e-7, rank=2, nu=50, batch_size=16), 50)
        return
    if a.real32:
        trajectory("micro_lozo_real32", MICRO, MICRO_TASK,
                   dict(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=2, nu=5, batch_size=8), 12,
                   precision="real32")
        trajectory("small_lozo_real32", SMALL, SMALL_TASK,
                   dict(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=2, nu=4, batch_size=16), 10,
                   precision="real32")
        return
    if a.only == "adapter":
        adapter_fixture()
        return
    if a.only == "full":
        full_scope_trajectories()
        return
    if a.only == "baseline":
        baseline_trajectories()
        return
    adapter_fixture()
    streams()
    fnv()
    forward_fixture("micro", MICRO, MICRO_TASK, B=8)
    forward_fixture("small", SMALL, SMALL_TASK, B=16)
    trajectory("micro_lozo", MICRO, MICRO_TASK,
               dict(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=2, nu=5, batch_size=8), 12)
    trajectory("micro_fact", MICRO, MICRO_TASK,
               dict(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=8,
                    estimator="factorized_sqrt_r", batch_size=8), 6)
    trajectory("small_lozo", SMALL, SMALL_TASK,
               dict(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=2, nu=4, batch_size=16), 10)
    full_scope_trajectories()
    baseline_trajectories()
    if a.opt125m:
        forward_fixture("opt125m", OPT125, OPT125_TASK, B=16)
        trajectory("opt125m_lozo", OPT125, OPT125_TASK,
                   dict(seed=42, epsilon=1e-3, learning_rate=1e-7, rank=2, nu=50, batch_size=16), 3)


if __name__ == "__main__":
    main()
