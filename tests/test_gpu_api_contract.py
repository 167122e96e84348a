"""Reference conventions of the public API that the trajectory tests do not reach
(SURVEY.md §8(b) "Reference conventions to preserve").

* ``GpuPairScorer`` drives the unmodified step control flow through the
  ``scorer=`` seam (zo_engine.py:298-346) and reproduces the reference trajectory.
* A plain host ``params`` dict keeps ONE device replica across calls and is
  mutated in place by the step functions that mutate parameters (factorized
  update zo_engine.py:449-450, folds runtime.py:242-250).
* ``step_directions`` is pure: calling it mid-run (for another window) leaves the
  trajectory unchanged.
* A host upload of a non-zero window A marks it unfolded, so a window change folds
  it with the V it was uploaded with (adapter.py:260-271 pairing).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _traj(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        lines = [json.loads(l) for l in f if l.strip()]
    return lines[0], [l for l in lines if l["record"] == "step"], lines[-1]


def _setup(h):
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.zo_engine import ZoConfig
    return M, M.ModelConfig(**h["model"]), M.generate_task(M.TaskConfig(**h["task"])), ZoConfig(**h["zo"])


def test_gpu_pair_scorer_through_lozo_step(golden_dir):
    from paper_2605_28760_b200.adapter import AdapterState
    from paper_2605_28760_b200.zo_engine import GpuPairScorer, lozo_step
    h, recs, fin = _traj(golden_dir, "traj_micro_lozo.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    params = M.init_params(mcfg, max_batch=zcfg.batch_size)
    state = AdapterState(epsilon=zcfg.epsilon)
    scorer = GpuPairScorer(params, mcfg, state)
    fused = M.init_params(mcfg, max_batch=zcfg.batch_size)
    fstate = AdapterState(epsilon=zcfg.epsilon)
    for t, rec in enumerate(recs):
        batch = M.sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
        out = lozo_step(params, mcfg, state, zcfg, t, batch, scorer=scorer)
        ref = lozo_step(fused, mcfg, fstate, zcfg, t, batch)
        assert (out.u_digest, out.v_digest, out.minibatch_id) == (rec["u_digest"], rec["v_digest"],
                                                                   rec["minibatch_id"])
        # the seam runs the same fused pair as the one-call step: identical losses
        assert (out.loss_plus, out.loss_minus, out.beta) == (ref.loss_plus, ref.loss_minus, ref.beta)
        assert abs(out.loss_plus - rec["loss_plus"]) < 2e-3 and abs(out.loss_minus - rec["loss_minus"]) < 2e-3
        if (t + 1) % zcfg.nu == 0:
            for p in (params, fused):
                p.engine.fold()
                p.invalidate()


def test_pair_scorer_cache_invalidated_by_adapter_edit(golden_dir):
    """An L- cached on the +1 call is not served after the adapter changed."""
    from paper_2605_28760_b200.adapter import AdapterState
    from paper_2605_28760_b200.zo_engine import GpuPairScorer, lozo_step
    h, recs, _ = _traj(golden_dir, "traj_micro_lozo.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    params = M.init_params(mcfg, max_batch=zcfg.batch_size)
    state = AdapterState(epsilon=zcfg.epsilon)
    batch = M.sample_minibatch(task, "train", zcfg.seed, 0, zcfg.batch_size)
    lozo_step(params, mcfg, state, zcfg, 0, batch)  # binds, samples V/U
    eng = params.engine
    eng.sample_u(zcfg.seed, 1)
    state._probe_on = True
    scorer = GpuPairScorer(params, mcfg, state)
    state.set_sign(1)
    scorer(batch)
    assert scorer._cached is not None
    v0 = scorer._cached[1]
    state._touch()  # a caller edit between the two calls
    state.set_sign(-1)
    lm = scorer(batch)
    assert scorer._cached is None  # re-scored, not served from the stale cache
    assert lm == v0  # nothing actually changed on the device, so the fresh score agrees


def test_host_dict_params_single_replica_and_write_back(golden_dir):
    from paper_2605_28760_b200.adapter import AdapterState
    from paper_2605_28760_b200.model import as_device_params
    from paper_2605_28760_b200.zo_engine import factorized_step
    h, recs, fin = _traj(golden_dir, "traj_micro_fact.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    host = M.init_params(mcfg, max_batch=zcfg.batch_size).to_host()
    ids = {k: id(v) for k, v in host.items()}
    dp0 = as_device_params(host, mcfg)
    assert as_device_params(host, mcfg) is dp0  # one replica per dict
    dev = M.init_params(mcfg, max_batch=zcfg.batch_size)
    s1, s2 = AdapterState(epsilon=zcfg.epsilon), AdapterState(epsilon=zcfg.epsilon)
    for t in range(3):
        batch = M.sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
        a = factorized_step(host, mcfg, s1, zcfg, t, batch)
        b = factorized_step(dev, mcfg, s2, zcfg, t, batch)
        assert (a.loss_plus, a.loss_minus, a.beta) == (b.loss_plus, b.loss_minus, b.beta)
    assert as_device_params(host, mcfg) is dp0
    # the caller's arrays were updated in place (same objects), bit-equal to the device replica
    assert {k: id(v) for k, v in host.items()} == ids
    assert M.params_digest(host) == M.params_digest(dev)
    assert M.params_digest(host) != h["model_digest"]


def test_run_serving_path_host_dict_sees_folds(golden_dir):
    from paper_2605_28760_b200.runtime import run_serving_path
    h, recs, fin = _traj(golden_dir, "traj_micro_lozo.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    host = M.init_params(mcfg, max_batch=zcfg.batch_size).to_host()
    run = run_serving_path(mcfg, task, zcfg, h["steps"], eval_every=10 ** 9, params=host)
    assert M.params_digest(host) == run.final_params_digest


def test_step_directions_is_pure(golden_dir):
    from paper_2605_28760_b200.adapter import AdapterState
    from paper_2605_28760_b200.zo_engine import lozo_step, step_directions
    h, recs, fin = _traj(golden_dir, "traj_micro_lozo.jsonl")  # nu = 5
    M, mcfg, task, zcfg = _setup(h)
    runs = []
    for probe_mid_run in (False, True):
        params = M.init_params(mcfg, max_batch=zcfg.batch_size)
        state = AdapterState(epsilon=zcfg.epsilon)
        out = []
        for t in range(8):
            if probe_mid_run and t == 3:
                d = step_directions(params, zcfg, 11, mcfg)  # another window, mid-window
                assert d.u_digest == recs[11]["u_digest"] and d.v_digest == recs[11]["v_digest"]
            batch = M.sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
            r = lozo_step(params, mcfg, state, zcfg, t, batch)
            out.append((r.loss_plus, r.loss_minus, r.beta, r.u_digest, r.v_digest))
            if (t + 1) % zcfg.nu == 0:
                params.engine.fold()
                params.invalidate()
        params.engine.fold()
        params.invalidate()
        runs.append((out, M.params_digest(params)))
    assert runs[0] == runs[1]


def test_uploaded_window_mass_is_folded_before_v_changes():
    from paper_2605_28760_b200.engine import A, V, ZoEngine
    eng = ZoEngine(64, 32, 2, 2, 16, max_batch=8, rank=2)
    eng.init_params(7, 0.08)
    eng.sample_v(42, 0, 5)
    w0 = {lid: eng.download(lid) for lid in eng.lids}
    vw = eng.split(V, eng.get_slot(V))
    a = np.random.default_rng(3).standard_normal(eng.su) * 1e-2
    eng.set_slot(A, a)
    eng.set_window(0)  # the uploaded V is window 0's
    eng.sample_v(42, 5, 5)  # window change: the uploaded A must be folded with the OLD V first
    assert not eng.get_slot(A).any()
    am = eng.split(A, a)
    for lid in eng.lids:
        want = w0[lid].copy()
        for k in range(2):  # numerics.py:228-235, k ascending
            want += np.multiply.outer(am[lid][:, k], vw[lid][:, k])
        np.testing.assert_array_equal(eng.download(lid), want)
    eng.close()
