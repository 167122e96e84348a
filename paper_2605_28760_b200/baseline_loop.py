"""The conventional training loop (``zoserve.baseline_loop``, baseline_loop.py:1-271)
on the same device replica: the cost comparand of the serving path.

Per step and matrix the loop writes the probe into the weights (W += eps*P,
score L+; W += -2eps*P, score L-), restores them and writes the update
(W += -(eta*c_used)*P) -- four m*n weight writes -- and scores each sign with
its own forward over the materialised weights (no LoRA extension, two
launches of every GEMM instead of one).  ``recompute_products`` selects the
reference's two _Probe modes (baseline_loop.py:68-104): cached (dense product
applied with axpy_dense, bit-exact restore) or recompute (axpy_outer per term,
arithmetic restore), and all three estimators run (dense_mezo: a dense z per weight,
regenerated every step, _DenseProbe).  The float64 arithmetic is the reference's, so the
parameters are bit-exact given the coefficients (tests/test_gpu_baseline.py);
the scoring runs on the 16-bit tensor-core path like the serving scorer.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

from .engine import U as SLOT_U, V as SLOT_V
from .errors import ConfigError
from .engine import resolve_precision
from .model import (EvalPoint, ModelConfig, TaskData, as_device_params, evaluate_split, init_params,
                    params_digest, sample_minibatch)
from .numerics import canonical_mean, digest_hex
from .runtime import CostMeter
from .zo_engine import ZoConfig, ZoStepRecord, make_step_record, write_trajectory

__all__ = ["BaselineRun", "run_baseline", "compare_ready_export", "run_header"]


@dataclass
class BaselineRun:  # baseline_loop.py:49-65
    config: ZoConfig
    model_config: ModelConfig
    trajectory: list[ZoStepRecord]
    eval_curve: list[EvalPoint]
    weight_write_count: int
    meter: CostMeter
    final_params_digest: str
    params: object
    train_wall_s: float
    precision: str
    steps_completed: int
    model_digest: str
    task_digest: str
    recompute_products: bool
    kind: str = "baseline"
    probe_pairs: list = field(default_factory=list)  # symmetry with ServingRun


def run_baseline(mcfg: ModelConfig, task: TaskData, zcfg: ZoConfig, steps: int, precision: str = "real64",
                 eval_every: int = 50, recompute_products: bool = False, params=None,
                 digests: bool = True, compute_param_digests: bool = True) -> BaselineRun:
    """Full-weight perturb / score / restore / update loop (baseline_loop.py:122-239).

    Same signature, return type and records as the reference; ``digests`` /
    ``compute_param_digests`` (defaults = the reference's behaviour) switch the
    host-side fingerprints off for long timing runs."""
    if steps < 1:
        raise ConfigError("steps must be >= 1")
    params = init_params(mcfg, precision=resolve_precision(precision),
                         max_batch=max(16, zcfg.batch_size)) if params is None else params
    dp = as_device_params(params, mcfg)
    opt_len = len(task.config.options[0])
    eng = dp.bind(zcfg.rank, zcfg.estimator, zcfg.batch_size, opt_len, zcfg.scope)
    model_digest = params_digest(dp) if compute_param_digests else ""
    meter = CostMeter()
    eps, eta = zcfg.epsilon, zcfg.learning_rate
    rec_mode = bool(recompute_products)
    # 4 counted writes per perturbed element per step (baseline_loop.py:131-135)
    per_step = sum(m * n for m, n in eng.shapes.values())
    if zcfg.scope == "full" or zcfg.estimator == "dense_mezo":
        per_step += sum(eng.vlens.values())
    trajectory: list[ZoStepRecord] = []
    evals: list[EvalPoint] = []
    wall = 0.0

    def do_eval(at: int) -> None:
        dp.invalidate()
        loss, acc = evaluate_split(dp, mcfg, task, "dev", None, precision)
        evals.append(EvalPoint(at, wall * 1e3, loss, acc))

    do_eval(0)
    for t in range(steps):
        batch = sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
        tokens, gold = batch.sequences()
        t0 = time.perf_counter()
        eng.baseline_directions(zcfg.seed, t, zcfg.nu)
        eng.baseline_pass(0, eps, rec_mode)
        s0 = time.perf_counter()
        lp = canonical_mean(eng.score(tokens, gold, nsign=1)[0])
        s1 = time.perf_counter()
        eng.baseline_pass(1, eps, rec_mode)
        s2 = time.perf_counter()
        lm = canonical_mean(eng.score(tokens, gold, nsign=1)[0])
        s3 = time.perf_counter()
        eng.baseline_pass(2, eps, rec_mode)
        c = (lp - lm) / (2.0 * eps)
        c_used = c / zcfg.rank if (zcfg.divide_by_r and zcfg.estimator == "lozo_lazy") else c
        beta = -(eta * c_used)
        eng.set_coefficient([lp, lm, c, beta])
        eng.baseline_update(eta, rec_mode)
        t1 = time.perf_counter()
        wall += t1 - t0
        meter.scoring_calls += 2
        meter.scoring_cost_units += 2 * batch.prompts.shape[0]
        meter.writes_probe += 3 * per_step
        meter.time_scoring_s += (s1 - s0) + (s3 - s2)
        meter.time_update_s += (t1 - t0) - (s1 - s0) - (s3 - s2)
        ud = digest_hex(eng.digest(SLOT_U)) if digests else ""
        vd = digest_hex(eng.digest(SLOT_V)) if digests else ""
        trajectory.append(make_step_record(zcfg, t, lp, lm, beta, ud, vd, batch))
        if (t + 1) % eval_every == 0 and (t + 1) != steps:
            do_eval(t + 1)
    do_eval(steps)
    dp.invalidate()
    dp.sync_host()  # the reference mutates the caller's params dict in place
    return BaselineRun(config=zcfg, model_config=mcfg, trajectory=trajectory, eval_curve=evals,
                       weight_write_count=4 * per_step * steps, meter=meter,
                       final_params_digest=params_digest(dp) if compute_param_digests else "", params=dp,
                       train_wall_s=wall, precision=precision, steps_completed=steps, model_digest=model_digest,
                       task_digest=task.digest(), recompute_products=rec_mode)


def run_header(run, path_name: str, extra: dict | None = None) -> dict:
    """Trajectory-file header shared by both execution paths (baseline_loop.py:242-257)."""
    header = {
        "path": path_name,
        "precision": run.precision,
        "steps": run.steps_completed,
        "seed": run.config.seed,
        "estimator": run.config.estimator,
        "scope": run.config.scope,
        "zo_digest": run.config.digest(),
        "model_digest": run.model_digest,
        "task_digest": run.task_digest,
    }
    if extra:
        header.update(extra)
    return header


def compare_ready_export(run, path: str, extra_header: dict | None = None) -> str:
    """Shared JSON-lines trajectory (header, step records, final summary),
    baseline_loop.py:260-271.  Serving runs carry no write count."""
    final_eval = run.eval_curve[-1]
    final = {
        "eval_loss": final_eval.loss,
        "eval_acc": final_eval.acc,
        "params_digest": run.final_params_digest,
        "weight_writes": getattr(run, "weight_write_count", 0),
    }
    write_trajectory(path, run_header(run, run.kind, extra_header), run.trajectory, final)
    return path
