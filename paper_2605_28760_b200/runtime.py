"""Serving-style driver of ``zoserve.runtime`` (runtime.py:253-359) on the engine.

``run_serving_path`` keeps the reference's loop and return type: per step a
host minibatch (16 indices), one fused device ``lozo_step``, a fold at every
nu boundary and at run end, evals at the reference cadence (excluded from
``train_wall_s``).  U/V digests are computed off the critical path by a host
thread pool from device copies of the slot arenas.
"""
from __future__ import annotations

import concurrent.futures as cf
import time

import numpy as np
from dataclasses import dataclass, field

from .adapter import AdapterState
from .engine import U as SLOT_U, V as SLOT_V, Z as SLOT_Z
from .errors import ConfigError, ScoringAbort
from .engine import resolve_precision
from .model import (EvalPoint, ModelConfig, TaskData, as_device_params, evaluate_split, init_params,
                    params_digest, sample_minibatch)
from .numerics import digest_hex
from .zo_engine import ZoConfig, ZoStepRecord, factorized_step, lozo_step

__all__ = ["CostMeter", "ServingRun", "ScoringAbort", "run_serving_path", "save_checkpoint", "load_checkpoint"]


@dataclass
class CostMeter:
    """Phase accounting (runtime.py:84-136).  Weight-write counts are a CPU
    cost proxy in the reference; here the device phases are timed with CUDA
    events (sample / score / update) and folds by wall clock."""
    scoring_calls: int = 0
    scoring_cost_units: int = 0
    writes_probe: int = 0
    time_sample_s: float = 0.0
    time_scoring_s: float = 0.0
    time_update_s: float = 0.0
    time_fold_s: float = 0.0

    def to_dict(self) -> dict:
        return dict(self.__dict__)


@dataclass
class ServingRun:
    config: ZoConfig
    model_config: ModelConfig
    trajectory: list[ZoStepRecord]
    eval_curve: list[EvalPoint]
    meter: CostMeter
    final_params_digest: str
    params: object
    state: AdapterState
    train_wall_s: float
    precision: str
    steps_completed: int
    model_digest: str
    task_digest: str
    aborted: bool = False
    kind: str = "serving-b200"
    extra: dict = field(default_factory=dict)


SNAP_RING = 4  # zob200.h zo_slot_snapshot ring depth


class _SnapRing:
    """Pinned host ring of asynchronous U / V arena snapshots (zob200.h zo_slot_snapshot): the
    device copy is stream-ordered, the host copy overlaps the next step, and a slot is reused
    only after the digest reading it has finished."""

    def __init__(self, eng, which: int):
        self.eng, self.which, self.next, self.busy = eng, which, 0, [None] * SNAP_RING

    def digest(self, pool, z_arena=None):
        slot = self.next
        self.next = (slot + 1) % SNAP_RING
        if self.busy[slot] is not None:
            self.busy[slot].result()
        self.eng.snapshot(self.which, slot)
        eng, which = self.eng, self.which
        fut = pool.submit(lambda: eng.digest(which, eng.snapshot_wait(which, slot), z_arena))
        self.busy[slot] = fut
        return fut


def run_serving_path(mcfg: ModelConfig, task: TaskData, zcfg: ZoConfig, steps: int, precision: str = "real64",
                     eval_every: int = 50, fold_on_eval: bool = False, abort_at: int | None = None,
                     params=None, digests: bool = True, compute_param_digests: bool = True,
                     state: AdapterState | None = None, start_step: int = 0, final_fold: bool = True,
                     digest_every: int = 1) -> ServingRun:
    """ZO fine-tuning the serving way (runtime.py:253-359), device-resident.

    Extensions over the reference signature (all defaulted to its behaviour):
    ``state`` / ``start_step`` resume a run from ``load_checkpoint`` (steps
    start_step .. start_step+steps-1, the counter-keyed streams make the
    continuation bit-identical to an uninterrupted run), ``final_fold=False``
    leaves the window unfolded so the run can be checkpointed mid-window, and
    ``digest_every = k > 1`` audits the U/V digests of every k-th step only (the others
    carry empty digests, which verify.strict_compare skips): the reference chains every
    step's full direction arena through FNV-1a, a byte-serial hash -- at rank 128 on 13B
    that is 1.5 GB of U per step, read back and hashed on the host."""
    if steps < 1:
        raise ConfigError("steps must be >= 1")
    if digest_every < 1:
        raise ConfigError("digest_every must be >= 1")
    if zcfg.estimator == "dense_mezo":
        raise ConfigError("dense_mezo has no serving-path form (no compact update factor); "
                          "use the baseline path for it")
    params = init_params(mcfg, precision=resolve_precision(precision),
                         max_batch=max(16, zcfg.batch_size)) if params is None else params
    dp = as_device_params(params, mcfg)
    opt_len = len(task.config.options[0])
    eng = dp.bind(zcfg.rank, zcfg.estimator, zcfg.batch_size, opt_len, zcfg.scope)
    model_digest = params_digest(dp) if compute_param_digests else ""
    state = AdapterState(epsilon=zcfg.epsilon) if state is None else state
    state._bind(eng)
    state._sync_to_engine(eng)
    meter = CostMeter()
    step_fn = lozo_step if zcfg.estimator == "lozo_lazy" else factorized_step
    pool = cf.ThreadPoolExecutor(max_workers=4) if digests else None
    rings = {SLOT_U: _SnapRing(eng, SLOT_U), SLOT_V: _SnapRing(eng, SLOT_V)}
    pending: list[tuple[ZoStepRecord, cf.Future, cf.Future | None]] = []
    vfut = {"key": None, "fut": None}
    trajectory: list[ZoStepRecord] = []
    evals: list[EvalPoint] = []
    wall = 0.0
    aborted = False

    def do_eval(at: int) -> None:
        if fold_on_eval and zcfg.estimator == "lozo_lazy":
            eng.fold()
            dp.invalidate()
        loss, acc = evaluate_split(dp, mcfg, task, "dev", state.view(), precision)
        evals.append(EvalPoint(at, wall * 1e3, loss, acc))

    do_eval(start_step)
    done = start_step
    loop_t0 = time.perf_counter()
    eval_in_loop = 0.0
    # the next step's minibatch is drawn on a host thread while the device runs this step (the
    # engine call releases the GIL); the draw is a pure function of (seed, step)
    prefetch = cf.ThreadPoolExecutor(max_workers=1)
    nxt = prefetch.submit(sample_minibatch, task, "train", zcfg.seed, start_step, zcfg.batch_size)
    for t in range(start_step, start_step + steps):
        batch = nxt.result()
        if t + 1 < start_step + steps:
            nxt = prefetch.submit(sample_minibatch, task, "train", zcfg.seed, t + 1, zcfg.batch_size)
        t0 = time.perf_counter()
        try:
            if abort_at is not None and t == abort_at:
                raise ScoringAbort(f"injected failure at step {t}")
            rec = step_fn(dp, mcfg, state, zcfg, t, batch, precision, digests="off")
        except ScoringAbort:
            aborted = True
            break
        wall += time.perf_counter() - t0
        ms = eng.last_step_ms()
        meter.time_sample_s += ms[0] * 1e-3
        meter.time_scoring_s += ms[1] * 1e-3
        meter.time_update_s += ms[2] * 1e-3
        meter.scoring_calls += 2
        meter.scoring_cost_units += 2 * zcfg.batch_size
        if pool is not None and (t - start_step) % digest_every == 0:
            # U (and a new window's V) leave through asynchronous snapshots into a pinned ring:
            # the device copy is stream-ordered, the host copy overlaps the next step, and the
            # digest thread waits for it (a ring slot is reused only after its digest is done)
            z_arena = eng.get_slot(SLOT_Z) if zcfg.scope == "full" else None
            ufut = rings[SLOT_U].digest(pool, z_arena)
            wkey = (t // zcfg.nu) * zcfg.nu if zcfg.estimator == "lozo_lazy" else t
            if vfut["key"] != wkey:
                vfut["key"], vfut["fut"] = wkey, rings[SLOT_V].digest(pool)
            pending.append((rec, ufut, vfut["fut"]))
        trajectory.append(rec)
        done = t + 1
        if zcfg.estimator == "lozo_lazy" and (t + 1) % zcfg.nu == 0:
            f0 = time.perf_counter()
            eng.fold()
            dp.invalidate()
            dt = time.perf_counter() - f0
            meter.time_fold_s += dt
            wall += dt
        if (t + 1) % eval_every == 0 and (t + 1) != start_step + steps:
            e0 = time.perf_counter()
            do_eval(t + 1)
            eval_in_loop += time.perf_counter() - e0
    loop_wall = time.perf_counter() - loop_t0 - eval_in_loop
    prefetch.shutdown(wait=False)
    if not aborted and final_fold and zcfg.estimator == "lozo_lazy":
        f0 = time.perf_counter()
        eng.fold()
        dp.invalidate()
        dt = time.perf_counter() - f0
        meter.time_fold_s += dt
        wall += dt
    if not aborted:
        do_eval(done)
    dp.sync_host()  # a caller's host dict sees the folds, as in the reference (runtime.py:242-250)
    d0 = time.perf_counter()
    for rec, uf, vf in pending:  # unaudited steps (digest_every > 1) keep empty digests
        rec.u_digest = digest_hex(uf.result())
        rec.v_digest = digest_hex(vf.result())
    if pool is not None:
        pool.shutdown()
    digest_wait = time.perf_counter() - d0
    return ServingRun(config=zcfg, model_config=mcfg, trajectory=trajectory, eval_curve=evals, meter=meter,
                      final_params_digest=params_digest(dp) if compute_param_digests else "", params=dp,
                      state=state, train_wall_s=wall, precision=precision, steps_completed=done,
                      model_digest=model_digest, task_digest=task.digest(), aborted=aborted,
                      extra={"loop_wall_s": loop_wall, "digest_wait_s": digest_wait})


# ---------------------------------------------------------------- checkpoint / resume
def save_checkpoint(path: str, params, state: AdapterState, next_step: int, mcfg: ModelConfig,
                    zcfg: ZoConfig) -> dict:
    """Checkpoint a (possibly mid-window) device run into directory ``path``:

    * ``adapter.zoad`` (+ manifest) -- the window slots (A, V_win) in the
      reference's ZOAD format (adapter.py:305-328);
    * ``params/<layer id>.npy`` -- the float64 master weights with every fold
      applied so far, and the LN vectors;
    * ``meta.json`` -- next step, configs, digests.

    Resuming needs nothing else: U, V and minibatches are counter-keyed by
    (seed, step), so ``run_serving_path(..., state=, start_step=next_step)``
    continues bit-identically."""
    import json
    import os
    from dataclasses import asdict

    from .adapter_io import save_adapter
    os.makedirs(os.path.join(path, "params"), exist_ok=True)
    dp = as_device_params(params, mcfg)
    for k in dp:
        np.save(os.path.join(path, "params", k + ".npy"), np.asarray(dp[k], dtype=np.float64))
    man = save_adapter(state, os.path.join(path, "adapter.zoad"))
    meta = {"format": "zob200-checkpoint-1", "next_step": int(next_step), "model": asdict(mcfg),
            "zo": asdict(zcfg), "params_digest": params_digest(dp), "adapter_state_digest": man["state_digest"]}
    with open(os.path.join(path, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    return meta


def load_checkpoint(path: str, precision: str = "fp16", max_batch: int = 16, device: int = 0):
    """Inverse of ``save_checkpoint``: returns (params, state, next_step, meta) with
    the params re-uploaded to a fresh device engine on first use and the digests
    verified."""
    import json
    import os

    from .adapter_io import load_adapter
    from .errors import InputError
    with open(os.path.join(path, "meta.json")) as f:
        meta = json.load(f)
    if meta.get("format") != "zob200-checkpoint-1":
        raise InputError("not a zob200 checkpoint")
    mcfg = ModelConfig(**meta["model"])
    host = {}
    for fn in sorted(os.listdir(os.path.join(path, "params"))):
        if fn.endswith(".npy"):
            host[fn[:-4]] = np.load(os.path.join(path, "params", fn))
    if params_digest(host) != meta["params_digest"]:
        raise InputError("checkpoint params digest mismatch")
    from .model import DeviceParams
    params = DeviceParams(mcfg, host=host, precision=resolve_precision(precision),
                          max_batch=max_batch, device=device)
    state = load_adapter(os.path.join(path, "adapter.zoad"))
    for e in state._host_entries.values():
        e.perturb_slot = None  # probes are per-step and never carried across steps
    state._probe_on = False
    nxt = int(meta["next_step"])
    if meta["zo"].get("estimator", "lozo_lazy") == "lozo_lazy":
        nu = int(meta["zo"]["nu"])
        state._window_hint = (nxt // nu) * nu  # the saved V is this window's (mid-window resume)
    return params, state, nxt, meta
