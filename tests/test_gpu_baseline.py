"""The materialising training-loop comparand (baseline_loop.py:122-239) on the GPU,
against the reference's own run_baseline trajectories (tests/golden/traj_*baseline*).

* With the reference's losses injected as the coefficient, the device probe /
  restore / update writes (cached dense product or recompute axpy_outer) must
  reproduce the reference's float64 parameters BIT-EXACTLY, and every step's
  U/V digests must match.
* run_baseline end to end: digests exact, losses within the fp16 tolerance.
* The fused device step (zo_baseline_step_async, the bench path) equals the
  host-driven loop bit for bit.
* All three estimators of run_baseline: lozo_lazy, factorized_sqrt_r and dense_mezo (a dense
  Role.DENSE_Z direction per weight, _DenseProbe).
"""
import json
import os

import numpy as np
import pytest

import zo_tolerances as _T

pytestmark = pytest.mark.gpu

NAMES = ["micro_baseline", "micro_baseline_recompute", "micro_baseline_fact", "micro_baseline_full",
         "micro_baseline_dense", "micro_baseline_dense_recompute"]


def _traj(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        lines = [json.loads(l) for l in f if l.strip()]
    return lines[0], [l for l in lines if l["record"] == "step"], lines[-1]


def _setup(h):
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.zo_engine import ZoConfig
    return M, M.ModelConfig(**h["model"]), M.generate_task(M.TaskConfig(**h["task"])), ZoConfig(**h["zo"])


def _bind(M, mcfg, task, zcfg):
    params = M.init_params(mcfg, max_batch=zcfg.batch_size)
    eng = params.bind(zcfg.rank, zcfg.estimator, zcfg.batch_size, len(task.config.options[0]), zcfg.scope)
    return params, eng


@pytest.mark.parametrize("name", NAMES)
def test_materialised_writes_bit_exact_with_reference_coefficients(golden_dir, name):
    from paper_2605_28760_b200.engine import U, V
    from paper_2605_28760_b200.numerics import digest_hex
    h, recs, fin = _traj(golden_dir, f"traj_{name}.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    params, eng = _bind(M, mcfg, task, zcfg)
    assert M.params_digest(params) == h["model_digest"]
    rc = bool(h["recompute_products"])
    for t, rec in enumerate(recs):
        batch = M.sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
        assert batch.batch_id == rec["minibatch_id"]
        tokens, gold = batch.sequences()
        eng.baseline_directions(zcfg.seed, t, zcfg.nu)
        assert digest_hex(eng.digest(U)) == rec["u_digest"]
        assert digest_hex(eng.digest(V)) == rec["v_digest"]
        lp_lm = []
        for p in (0, 1):
            eng.baseline_pass(p, zcfg.epsilon, rc)
            lp_lm.append(float(np.mean(eng.score(tokens, gold, nsign=1)[0])))
        eng.baseline_pass(2, zcfg.epsilon, rc)
        lp, lm = rec["loss_plus"], rec["loss_minus"]
        # the device losses of the materialised weights track the reference (fp16 scoring)
        assert abs(lp_lm[0] - lp) <= _T.LOSS_MATERIALISED and abs(lp_lm[1] - lm) <= _T.LOSS_MATERIALISED
        c = (lp - lm) / (2.0 * zcfg.epsilon)
        assert c == rec["coefficient"]
        eng.set_coefficient([lp, lm, c, rec["beta"]])
        eng.baseline_update(zcfg.learning_rate, rc)
    params.invalidate()
    assert M.params_digest(params) == fin["final_params_digest"]


@pytest.mark.parametrize("name", NAMES)
def test_run_baseline_vs_reference(golden_dir, name):
    from paper_2605_28760_b200.baseline_loop import compare_ready_export, run_baseline
    h, recs, fin = _traj(golden_dir, f"traj_{name}.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    run = run_baseline(mcfg, task, zcfg, h["steps"], eval_every=10**9,
                       recompute_products=bool(h["recompute_products"]),
                       params=M.init_params(mcfg, max_batch=zcfg.batch_size))
    assert run.model_digest == h["model_digest"] and run.task_digest == h["task_digest"]
    assert run.weight_write_count == fin["weight_writes"]
    signs = 0
    for a, b in zip(recs, run.trajectory):
        assert (a["u_digest"], a["v_digest"], a["minibatch_id"]) == (b.u_digest, b.v_digest, b.minibatch_id)
        assert abs(a["loss_plus"] - b.loss_plus) <= _T.LOSS_MATERIALISED
        assert abs(a["loss_minus"] - b.loss_minus) <= _T.LOSS_MATERIALISED
        signs += np.sign(a["coefficient"]) == np.sign(b.coefficient)
    assert signs >= 0.75 * len(recs)
    assert abs(run.eval_curve[-1].loss - fin["eval_loss"]) <= _T.LOSS_MATERIALISED
    out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", f"parity_{name}_b200.jsonl")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    compare_ready_export(run, out)


@pytest.mark.parametrize("recompute", [False, True])
def test_fused_device_step_equals_host_loop(golden_dir, recompute):
    import torch
    from paper_2605_28760_b200.baseline_loop import run_baseline
    h, recs, fin = _traj(golden_dir, "traj_micro_baseline.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    steps = 6  # crosses the nu = 5 window start
    run = run_baseline(mcfg, task, zcfg, steps, eval_every=10**9, recompute_products=recompute,
                       params=M.init_params(mcfg, max_batch=zcfg.batch_size))
    params, eng = _bind(M, mcfg, task, zcfg)
    for t in range(steps):
        batch = M.sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
        tokens, gold = batch.sequences()
        tk = torch.from_numpy(np.ascontiguousarray(tokens, dtype=np.int32)).cuda()
        gd = torch.from_numpy(np.ascontiguousarray(gold, dtype=np.int32)).cuda()
        eng.baseline_step_async(zcfg.seed, t, zcfg.nu, zcfg.epsilon, zcfg.learning_rate, zcfg.divide_by_r,
                                recompute, tk.data_ptr(), gd.data_ptr(), zcfg.batch_size)
        out4 = eng.read_out4()
        r = run.trajectory[t]
        assert out4[0] == r.loss_plus and out4[1] == r.loss_minus and out4[3] == r.beta
    params.invalidate()
    assert M.params_digest(params) == run.final_params_digest


def test_baseline_rejects_unfolded_window():
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.adapter import AdapterState
    from paper_2605_28760_b200.errors import ConfigError
    from paper_2605_28760_b200.zo_engine import ZoConfig, lozo_step
    mcfg = M.ModelConfig(vocab=64, dim=32, n_layers=1, n_heads=2, prompt_len=8)
    task = M.generate_task(M.TaskConfig(seed=1, vocab=64, prompt_len=8, train_size=16, dev_size=2, val_size=2))
    zcfg = ZoConfig(batch_size=4, nu=5)
    params = M.init_params(mcfg, max_batch=4)
    lozo_step(params, mcfg, AdapterState(epsilon=zcfg.epsilon), zcfg, 0,
              M.sample_minibatch(task, "train", zcfg.seed, 0, 4))
    with pytest.raises(ConfigError):
        params.engine.baseline_directions(zcfg.seed, 1, zcfg.nu)


@pytest.mark.parametrize("recompute", [False, True])
def test_high_rank_materialising_writes_bit_exact(recompute):
    """r > 8 (the factorized MeZO-style comparand, config 5's estimator) runs the tiled
    float64 kernel; params bit-exact vs the oracle's run_baseline given its coefficients."""
    from oracle import reference as R
    from paper_2605_28760_b200 import model as M
    mk = dict(vocab=64, dim=32, n_layers=2, n_heads=2, prompt_len=16, init_seed=7, init_scale=0.08)
    tk = dict(seed=11, vocab=64, prompt_len=16, train_size=64, dev_size=8, val_size=8)
    rc = R.ModelCfg(**mk)
    splits = R.generate_task(R.TaskCfg(**tk))
    z = R.ZoCfg(seed=42, epsilon=1e-3, learning_rate=1e-3, rank=16, batch_size=8, estimator="factorized_sqrt_r")
    recs, final = R.run_baseline(rc, splits, z, 3, recompute=recompute)
    mcfg = M.ModelConfig(**mk)
    task = M.generate_task(M.TaskConfig(**tk))
    params = M.init_params(mcfg, max_batch=8)
    eng = params.bind(16, "factorized_sqrt_r", 8, 1, "lora_only")
    for t, rec in enumerate(recs):
        tokens, gold = M.sample_minibatch(task, "train", 42, t, 8).sequences()
        eng.baseline_directions(42, t, 1)
        for p in (0, 1):
            eng.baseline_pass(p, 1e-3, recompute)
            got = R.canonical_mean(eng.score(tokens, gold, nsign=1)[0])
            assert abs(got - (rec.loss_plus if p == 0 else rec.loss_minus)) <= _T.LOSS_MATERIALISED
        eng.baseline_pass(2, 1e-3, recompute)
        eng.set_coefficient([rec.loss_plus, rec.loss_minus, rec.coefficient, rec.beta])
        eng.baseline_update(1e-3, recompute)
    params.invalidate()
    assert M.params_digest(params) == R.params_digest(final)


def test_dense_mezo_step_api_bit_exact(golden_dir):
    """zo_engine.dense_mezo_step (zo_engine.py:476-493) on the device: the reference's dense
    estimator trajectory (= the materialising loop's cached mode) -- digests exact, losses
    within the fp16 tolerance, params bit-exact when the reference's losses are installed."""
    from paper_2605_28760_b200.zo_engine import dense_mezo_step
    h, recs, fin = _traj(golden_dir, "traj_micro_baseline_dense.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    params = M.init_params(mcfg, max_batch=zcfg.batch_size)
    for t, rec in enumerate(recs):
        batch = M.sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
        out = dense_mezo_step(params, mcfg, zcfg, t, batch)
        assert (out.u_digest, out.v_digest, out.minibatch_id) == (rec["u_digest"], rec["v_digest"],
                                                                   rec["minibatch_id"])
        assert abs(out.loss_plus - rec["loss_plus"]) <= _T.LOSS["fp16"] and abs(out.loss_minus - rec["loss_minus"]) <= _T.LOSS["fp16"]
    from paper_2605_28760_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        dense_mezo_step(params, mcfg, zcfg, 0, M.sample_minibatch(task, "train", zcfg.seed, 0, zcfg.batch_size),
                        scorer=lambda b: 0.0)
