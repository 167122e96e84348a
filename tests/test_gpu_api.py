"""The reference-shaped public API on the GPU, against the reference's golden
trajectories (tests/golden/traj_*.jsonl).

* With the reference's own coefficients injected through the `scorer=` seam,
  the device update (K8) and folds (K9) must reproduce the reference's float64
  parameters BIT-EXACTLY (final params_digest equal), and every step's U/V
  digests must match.
* run_serving_path end to end: digests exact, losses within the fp16 tolerance.
"""
import json
import os

import numpy as np
import pytest

import zo_tolerances as TOL

pytestmark = pytest.mark.gpu


def _traj(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        lines = [json.loads(l) for l in f if l.strip()]
    return lines[0], [l for l in lines if l["record"] == "step"], lines[-1]


def _setup(h):
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.zo_engine import ZoConfig
    mcfg = M.ModelConfig(**h["model"])
    task = M.generate_task(M.TaskConfig(**h["task"]))
    zcfg = ZoConfig(**h["zo"])
    return M, mcfg, task, zcfg


class _ReplayScorer:
    """scorer(batch) returning the reference's recorded L+ then L- (zo_engine.py:318-326)."""

    def __init__(self, recs):
        self.recs, self.i, self.calls = recs, 0, 0

    def __call__(self, batch):
        r = self.recs[self.i]
        v = r["loss_plus"] if self.calls % 2 == 0 else r["loss_minus"]
        self.calls += 1
        if self.calls % 2 == 0:
            self.i += 1
        return v


@pytest.mark.parametrize("name", ["micro_lozo", "small_lozo", "micro_full"])
def test_update_and_fold_bit_exact_with_reference_coefficients(golden_dir, name):
    from paper_2605_28760_b200.adapter import AdapterState
    from paper_2605_28760_b200.zo_engine import lozo_step
    h, recs, fin = _traj(golden_dir, f"traj_{name}.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    params = M.init_params(mcfg, max_batch=zcfg.batch_size)
    assert M.params_digest(params) == h["model_digest"]
    state = AdapterState(epsilon=zcfg.epsilon)
    scorer = _ReplayScorer(recs)
    for t, rec in enumerate(recs):
        batch = M.sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
        out = lozo_step(params, mcfg, state, zcfg, t, batch, scorer=scorer)
        assert (out.u_digest, out.v_digest, out.minibatch_id) == (rec["u_digest"], rec["v_digest"],
                                                                   rec["minibatch_id"])
        assert out.beta == rec["beta"] and out.coefficient == rec["coefficient"]
        if (t + 1) % zcfg.nu == 0:
            params.engine.fold()
            params.invalidate()
    assert M.params_digest(params) == fin["pre_fold_params_digest"]
    params.engine.fold()
    params.invalidate()
    assert M.params_digest(params) == fin["final_params_digest"]


@pytest.mark.parametrize("name", ["micro_fact", "micro_fact_full"])
def test_factorized_dense_update_bit_exact(golden_dir, name):
    from paper_2605_28760_b200.engine import U, V, ZoEngine
    from paper_2605_28760_b200.numerics import canonical_mean, digest_hex
    h, recs, fin = _traj(golden_dir, f"traj_{name}.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    eng = ZoEngine(mcfg.vocab, mcfg.dim, mcfg.n_layers, mcfg.n_heads, mcfg.prompt_len, max_batch=zcfg.batch_size,
                   rank=zcfg.rank, estimator="factorized_sqrt_r", scope=zcfg.scope)
    eng.init_params(mcfg.init_seed, mcfg.init_scale)
    dl = []
    for t, rec in enumerate(recs):
        batch = M.sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
        eng.sample_v(zcfg.seed, t, 1)
        eng.sample_u(zcfg.seed, t)
        assert digest_hex(eng.digest(U)) == rec["u_digest"]
        assert digest_hex(eng.digest(V)) == rec["v_digest"]
        tokens, gold = batch.sequences()
        eng.prepare_probe(zcfg.epsilon, 0)
        nll = eng.score(tokens, np.stack([gold, gold]), nsign=2)
        dl.append(max(abs(canonical_mean(nll[0]) - rec["loss_plus"]), abs(canonical_mean(nll[1]) - rec["loss_minus"])))
        eng.set_coefficient(np.array([rec["loss_plus"], rec["loss_minus"], rec["coefficient"], rec["beta"]]))
        eng.update_dense(zcfg.learning_rate)
    assert max(dl) <= TOL.LOSS["fp16"], dl
    params = {lid: eng.download(lid) for lid in eng.lids}
    params.update({k: eng.download_vector(k) for k in eng.vids})
    assert M.params_digest(params) == fin["final_params_digest"]


@pytest.mark.parametrize("name", ["micro_lozo", "micro_full"])
def test_run_serving_path_public_api(golden_dir, name):
    from paper_2605_28760_b200.runtime import run_serving_path
    h, recs, fin = _traj(golden_dir, f"traj_{name}.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    run = run_serving_path(mcfg, task, zcfg, h["steps"], eval_every=10 ** 9)
    assert run.model_digest == h["model_digest"] and run.task_digest == h["task_digest"]
    assert run.steps_completed == len(recs) and not run.aborted
    for a, b in zip(recs, run.trajectory):
        assert (a["u_digest"], a["v_digest"], a["minibatch_id"]) == (b.u_digest, b.v_digest, b.minibatch_id)
        assert abs(a["loss_plus"] - b.loss_plus) <= TOL.LOSS["fp16"]
        assert abs(a["loss_minus"] - b.loss_minus) <= TOL.LOSS["fp16"]
        if abs(a["loss_plus"] - a["loss_minus"]) >= TOL.HIGH_SIGNAL:
            assert abs(b.coefficient - a["coefficient"]) <= TOL.C_REL * abs(a["coefficient"]), (a, b)
    assert abs(run.eval_curve[-1].loss - fin["eval_loss"]) <= TOL.LOSS["fp16"]
    # the reference's wire format round-trips
    from paper_2605_28760_b200.zo_engine import read_trajectory, write_trajectory
    os.makedirs("gpurun_out", exist_ok=True)
    out = f"gpurun_out/parity_traj_{name}_b200.jsonl"
    write_trajectory(out, {"model_digest": run.model_digest}, run.trajectory, {"eval_loss": run.eval_curve[-1].loss})
    _, back, _ = read_trajectory(out)
    assert [r.to_dict() for r in back] == [r.to_dict() for r in run.trajectory]
    # the reference's acceptance checks (verify.py): strict compare at the fp16 tolerance,
    # sign agreement of L+ - L- on every high-signal step
    from paper_2605_28760_b200.verify import record_deltas, sign_match, strict_compare
    ref = read_trajectory(os.path.join(golden_dir, f"traj_{name}.jsonl"))
    sc = strict_compare(ref, read_trajectory(out), loss_tol=TOL.LOSS["fp16"])
    sm = sign_match(record_deltas(ref[1]), record_deltas(back))
    os.makedirs("gpurun_out/parity", exist_ok=True)
    with open(f"gpurun_out/parity/verify_{name}.json", "w") as f:
        json.dump({"strict_compare": sc.to_dict(), "sign_match": sm.to_dict()}, f, indent=1)
    assert sc.accepted == sc.steps, sc.to_dict()
    assert sm.high_signal_fraction == 1.0 and sm.overall_fraction >= 0.9, sm.to_dict()


def test_run_serving_path_abort_is_transactional(golden_dir):
    from paper_2605_28760_b200.runtime import run_serving_path
    h, recs, fin = _traj(golden_dir, "traj_micro_lozo.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    run = run_serving_path(mcfg, task, zcfg, 8, eval_every=10 ** 9, abort_at=3)
    assert run.aborted and run.steps_completed == 3 and len(run.trajectory) == 3


def test_evaluate_split_vs_oracle():
    from oracle import reference as R
    from paper_2605_28760_b200 import model as M
    mcfg = M.ModelConfig(vocab=512, dim=128, n_layers=2, n_heads=2, prompt_len=63, init_seed=7, init_scale=0.02)
    task = M.generate_task(M.TaskConfig(seed=11, vocab=512, prompt_len=63, train_size=16, dev_size=40, val_size=4))
    params = M.init_params(mcfg, max_batch=16)
    loss, acc = M.evaluate_split(params, mcfg, task, "dev")
    # oracle: base weights, gold-option NLL over the dev split (model.py:444-460)
    cfg = R.ModelCfg(**{k: getattr(mcfg, k) for k in R.ModelCfg.__dataclass_fields__})
    p = R.init_params(cfg)
    prompts, golds = task.splits["dev"]
    opts = np.array([[510], [511]])
    per = [R.forward_nll(p, cfg, np.concatenate([prompts, np.tile(o, (len(prompts), 1))], axis=1),
                         np.tile(o, (len(prompts), 1))) for o in opts]
    ref_loss = R.canonical_mean(np.choose(golds, per))
    ref_acc = float(np.mean(np.argmax(-np.stack(per, axis=1), axis=1) == golds))
    assert abs(loss - ref_loss) <= TOL.LOSS["fp16"]
    assert abs(acc - ref_acc) <= 1.0 / len(golds) + 1e-12


def test_score_options_one_forward_equals_per_option():
    """zo_score_options: every single-token option from one forward is bitwise the
    per-option forward (the scored row never attends the option token)."""
    from paper_2605_28760_b200.engine import ZoEngine
    eng = ZoEngine(512, 128, 2, 2, 63, max_batch=16, rank=2)
    eng.init_params(7, 0.02)
    rng = np.random.default_rng(4)
    prompts = rng.integers(0, 510, size=(16, 63))
    eng.prepare_probe(0.0, 1)
    both = eng.score_options(np.concatenate([prompts, np.full((16, 1), 510)], axis=1), [510, 511, 7])
    for j, o in enumerate((510, 511, 7)):
        tok = np.concatenate([prompts, np.full((16, 1), o)], axis=1)
        np.testing.assert_array_equal(both[j], eng.score(tok, np.full((16, 1), o), nsign=1)[0])
    eng.close()


def test_checkpoint_resume_bit_identical(golden_dir, tmp_path):
    """Checkpoint mid-window (ZOAD adapter + float64 masters), resume on a fresh
    engine: the continued trajectory and final parameters equal an uninterrupted
    run bit for bit (counter-keyed streams)."""
    from paper_2605_28760_b200.adapter_io import load_adapter
    from paper_2605_28760_b200.runtime import load_checkpoint, run_serving_path, save_checkpoint
    h, _, _ = _traj(golden_dir, "traj_micro_lozo.jsonl")
    M, mcfg, task, zcfg = _setup(h)  # nu = 5
    full = run_serving_path(mcfg, task, zcfg, 9, eval_every=10 ** 9)
    part = run_serving_path(mcfg, task, zcfg, 7, eval_every=10 ** 9, final_fold=False)  # stops mid-window
    meta = save_checkpoint(str(tmp_path / "ck"), part.params, part.state, 7, mcfg, zcfg)
    assert load_adapter(str(tmp_path / "ck" / "adapter.zoad")).entries["blk0.qkv"].window_slot.rank == zcfg.rank
    params, state, nxt, meta2 = load_checkpoint(str(tmp_path / "ck"))
    assert nxt == 7 and meta2 == meta
    rest = run_serving_path(mcfg, task, zcfg, 2, eval_every=10 ** 9, params=params, state=state, start_step=7)
    for a, b in zip(full.trajectory[7:], rest.trajectory):
        assert (a.step, a.loss_plus, a.loss_minus, a.beta, a.u_digest, a.v_digest) == \
               (b.step, b.loss_plus, b.loss_minus, b.beta, b.u_digest, b.v_digest)
    assert rest.final_params_digest == full.final_params_digest


@pytest.mark.parametrize("name", ["micro_lozo", "micro_full", "micro_fact", "micro_baseline_dense"])
def test_step_directions_match_reference(golden_dir, name):
    """zo_engine.step_directions (zo_engine.py:224-261) on the device: the chained U/V digests of
    the reference's records, matrices / vectors of the right shapes (dense_mezo: a dense z per
    weight, no V part)."""
    from oracle import reference as R
    from paper_2605_28760_b200.zo_engine import step_directions
    h, recs, _ = _traj(golden_dir, f"traj_{name}.jsonl")
    M, mcfg, task, zcfg = _setup(h)
    params = M.init_params(mcfg, max_batch=zcfg.batch_size)
    for t in (0, 1):
        d = step_directions(params, zcfg, t, mcfg)
        assert (d.u_digest, d.v_digest) == (recs[t]["u_digest"], recs[t]["v_digest"])
    if zcfg.estimator == "dense_mezo":
        lid = "blk1.ff_up"
        np.testing.assert_array_equal(d.matrices[lid], R.gaussian(zcfg.seed, 1, lid, R.ROLE_DENSE_Z,
                                                                  *d.matrices[lid].shape))
        assert set(d.vectors) == set(params.engine.vids)
    elif zcfg.scope == "full":
        assert all(v.shape == (mcfg.dim,) for v in d.vectors.values())


def test_slot_snapshot_ring():
    """zo_slot_snapshot / zo_slot_snapshot_wait (the digest path's asynchronous U / V copies):
    a landed snapshot equals the arena at snapshot time even after the arena moves on, ring
    slots are independent, and waiting on a slot never snapshotted is an InputError."""
    from paper_2605_28760_b200.engine import ZoEngine, U, V
    from paper_2605_28760_b200.errors import InputError
    eng = ZoEngine(512, 128, 2, 2, 63, max_batch=16, rank=2)
    eng.init_params(7, 0.02)
    eng.sample_u(42, 0)
    eng.sample_v(42, 0, 50)
    u0, v0 = eng.get_slot(U), eng.get_slot(V)
    eng.snapshot(U, 0)
    eng.snapshot(V, 0)
    eng.sample_u(42, 1)  # the arena moves on in stream order after the device copy
    u1 = eng.get_slot(U)
    assert not np.array_equal(u0, u1)
    eng.snapshot(U, 1)
    np.testing.assert_array_equal(eng.snapshot_wait(U, 0), u0)
    np.testing.assert_array_equal(eng.snapshot_wait(U, 1), u1)
    np.testing.assert_array_equal(eng.snapshot_wait(V, 0), v0)
    with pytest.raises(InputError):
        eng.snapshot_wait(U, 2)  # allocated with the ring, never written
    with pytest.raises(InputError):
        eng.snapshot(U, 4)  # past the ring depth (zob200.h SNAP_RING)
