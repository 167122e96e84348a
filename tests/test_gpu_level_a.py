"""Level A of the drop-in boundary against the UNMODIFIED reference.

``oracle/stage_ref.sh`` (run by ``__graft_entry__.build()``) copies the reference package
into oracle/_ref/zoserve, which travels to the GPU box.  Here its own
``zoserve.runtime.run_serving_path`` (runtime.py:253-359) runs with the B200 scorer
installed by ``plugin.install_into_zoserve``: the reference samples its directions,
keeps its AdapterState, applies accumulate_on_U and folds on the host, and calls
``forward_score`` / ``evaluate_split`` -- which now score on the device.  The resulting
trajectory is judged by the reference's own ``verify.strict_compare`` / ``sign_match``
against the golden trajectory the reference wrote in float64.

Skipped (not failed) when oracle/_ref was not staged (no /root/reference at build time).
"""
import json
import os
import sys

import numpy as np
import pytest

import zo_tolerances as TOL

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref")


def _zoserve():
    if not os.path.isfile(os.path.join(REF, "zoserve", "runtime.py")):
        pytest.skip("oracle/_ref/zoserve not staged (oracle/stage_ref.sh needs /root/reference at build time)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import zoserve
    import zoserve.runtime  # noqa: F401
    import zoserve.verify  # noqa: F401
    assert os.path.dirname(zoserve.__file__).startswith(REF)
    return zoserve


def _golden(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        lines = [json.loads(l) for l in f if l.strip()]
    return lines[0]


@pytest.mark.parametrize("name", ["traj_micro_lozo.jsonl", "traj_small_lozo.jsonl", "traj_opt125m_lozo.jsonl"])
def test_unmodified_run_serving_path_with_b200_scorer(golden_dir, name, tmp_path):
    zs = _zoserve()
    from zoserve.model import ModelConfig, TaskConfig, generate_task
    from zoserve.zo_engine import ZoConfig, read_trajectory, write_trajectory
    from zoserve.verify import record_deltas, sign_match, strict_compare

    from paper_2605_28760_b200.plugin import install_into_zoserve
    h = _golden(golden_dir, name)
    mcfg = ModelConfig(**h["model"])
    task = generate_task(TaskConfig(**h["task"]))
    zcfg = ZoConfig(**h["zo"])
    uninstall = install_into_zoserve(zs, rank=zcfg.rank, batch_size=zcfg.batch_size)
    try:
        run = zs.runtime.run_serving_path(mcfg, task, zcfg, h["steps"], eval_every=10 ** 9)
    finally:
        uninstall()
    assert not run.aborted and run.steps_completed == h["steps"]
    assert (run.model_digest, run.task_digest) == (h["model_digest"], h["task_digest"])
    out = str(tmp_path / "level_a.jsonl")
    final = {"eval_loss": run.eval_curve[-1].loss, "eval_acc": run.eval_curve[-1].acc,
             "final_params_digest": run.final_params_digest}
    write_trajectory(out, {"model_digest": run.model_digest, "task_digest": run.task_digest}, run.trajectory, final)
    ref = read_trajectory(os.path.join(golden_dir, name))
    got = read_trajectory(out)
    sc = strict_compare(ref, got, loss_tol=TOL.LOSS["fp16"])
    sm = sign_match(record_deltas(ref[1]), record_deltas(got[1]))
    rel_dc = [abs(b.coefficient - a.coefficient) / abs(a.coefficient) for a, b in zip(ref[1], got[1])
              if abs(a.loss_plus - a.loss_minus) >= TOL.HIGH_SIGNAL]
    rep = {"golden": name, "strict_compare": sc.to_dict(), "sign_match": sm.to_dict(),
           "max_rel_dc_high_signal": max(rel_dc, default=0.0), "eval_loss": final["eval_loss"],
           "eval_loss_ref": ref[2]["eval_loss"], "scorer_calls": run.meter.scoring_calls,
           "probe_writes": run.meter.writes_probe}
    os.makedirs("gpurun_out/parity", exist_ok=True)
    with open(f"gpurun_out/parity/level_a_{name.replace('.jsonl', '')}.json", "w") as f:
        json.dump(rep, f, indent=1, default=str)
    # the reference's own acceptance: every step accepted (seeds, U/V digests, losses)
    assert sc.accepted == sc.steps == h["steps"], rep
    assert sm.high_signal_fraction in (None, 1.0), rep
    assert max(rel_dc, default=0.0) <= TOL.C_REL, rep
    assert abs(final["eval_loss"] - ref[2]["eval_loss"]) <= TOL.LOSS["fp16"], rep
    # zero-write probing, the serving path's defining property (test_paths.py:114)
    assert run.meter.writes_probe == 0
