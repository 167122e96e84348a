"""The reference's "real32" precision (model.py:149-154) on the device: the float32
forward as 3xTF32 tcgen05 GEMMs (kind::tf32, fp32 accumulate) + fp32 LN / attention /
GELU / loss (csrc/precise.cu).  SURVEY.md §8(c) fp32-mode bounds: |dL+-| <= 1e-5 absolute,
|dc|/|c| <= 1e-3, against the reference's own real32 and real64 outputs."""
import json
import os

import numpy as np
import pytest

import zo_tolerances as TOL
from oracle import reference as R

pytestmark = pytest.mark.gpu


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _traj(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        lines = [json.loads(l) for l in f if l.strip()]
    return lines[0], [l for l in lines if l["record"] == "step"], lines[-1]


def _report(name, data):
    os.makedirs("gpurun_out/parity", exist_ok=True)
    with open(os.path.join("gpurun_out/parity", name + ".json"), "w") as f:
        json.dump(data, f, indent=1)


def test_tf32x3_gemm_accuracy():
    from paper_2605_28760_b200.engine import test_gemm_tf32x3
    rng = np.random.default_rng(0)
    for M, N, K in [(200, 384, 768), (2048, 256, 3072), (33, 1000, 96)]:
        A = rng.standard_normal((M, K)).astype(np.float32)
        W = 0.02 * rng.standard_normal((K, N))
        got = test_gemm_tf32x3(A, W).astype(np.float64)
        ref = A.astype(np.float64) @ W
        scale = np.sqrt(K) * 0.02  # |A . W| ~ sqrt(K) * std(W)
        err = np.max(np.abs(got - ref)) / scale
        # fp32-class (measured 1.9e-6 at K = 4096 with 4-block K chunks); 16-bit operands land at ~1e-3
        assert err < 4e-6, (M, N, K, err)


@pytest.mark.parametrize("name", ["micro", "small", "opt125m"])
def test_real32_forward_nll(golden_dir, name):
    from paper_2605_28760_b200.engine import ZoEngine
    g = _load(golden_dir, f"forward_{name}.json")
    m = g["model"]
    eng = ZoEngine(m["vocab"], m["dim"], m["n_layers"], m["n_heads"], m["prompt_len"], max_batch=16, rank=g["rank"],
                   precision="real32")
    eng.init_params(m["init_seed"], m["init_scale"])
    step, r = g["step"], g["rank"]
    eng.sample_v(g["zseed"], step, 50)
    eng.sample_u(g["zseed"], step)
    A = {lid: g["a_scale"] * R.gaussian(g["a_seed"], step, lid, R.ROLE_U, eng.shapes[lid][0], r) for lid in eng.lids}
    eng.set_slot(2, eng.join(2, A))
    tokens = np.asarray(g["tokens"])
    gold = tokens[:, m["prompt_len"]:]
    eng.prepare_probe(g["epsilon"], 0)
    nll = eng.score(tokens, np.stack([gold, gold]), nsign=2)
    eng.prepare_probe(g["epsilon"], 1)
    nll0 = eng.score(tokens, gold, nsign=1)[0]
    eng.close()
    got = {1: nll[0], -1: nll[1], 0: nll0}
    rep = {}
    for prec in ("real32", "real64"):
        ref = {s: np.array(g["nll"][f"{prec}:{s}"]) for s in (1, -1, 0)}
        rep[prec] = {"max_abs_nll": max(float(np.max(np.abs(got[s] - ref[s]))) for s in (1, -1, 0)),
                     "dL_ref": R.canonical_mean(ref[1]) - R.canonical_mean(ref[-1]),
                     "dL_got": R.canonical_mean(got[1]) - R.canonical_mean(got[-1])}
        rep[prec]["rel_err_dL"] = abs(rep[prec]["dL_got"] - rep[prec]["dL_ref"]) / abs(rep[prec]["dL_ref"])
    _report(f"real32_forward_{name}", rep)
    for prec in ("real32", "real64"):
        assert rep[prec]["max_abs_nll"] <= TOL.REAL32_NLL, rep
        assert rep[prec]["rel_err_dL"] <= TOL.REAL32_C_REL, rep


@pytest.mark.parametrize("name", ["micro_lozo_real32", "small_lozo_real32", "micro_lozo", "opt125m_lozo"])
def test_real32_run_serving_path(golden_dir, name):
    """run_serving_path(precision="real32") against the reference's real32 (and real64) runs."""
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.runtime import run_serving_path
    from paper_2605_28760_b200.zo_engine import ZoConfig
    h, recs, fin = _traj(golden_dir, f"traj_{name}.jsonl")
    mcfg = M.ModelConfig(**h["model"])
    task = M.generate_task(M.TaskConfig(**h["task"]))
    zcfg = ZoConfig(**h["zo"])
    run = run_serving_path(mcfg, task, zcfg, h["steps"], precision="real32", eval_every=10 ** 9)
    rows = []
    for a, b in zip(recs, run.trajectory):
        assert (a["u_digest"], a["v_digest"], a["minibatch_id"]) == (b.u_digest, b.v_digest, b.minibatch_id)
        rows.append({"dLp": b.loss_plus - a["loss_plus"], "dLm": b.loss_minus - a["loss_minus"],
                     "rel_dc": abs(b.coefficient - a["coefficient"]) / abs(a["coefficient"]),
                     "d_diff": abs((b.loss_plus - b.loss_minus) - (a["loss_plus"] - a["loss_minus"])),
                     "high_signal": abs(a["loss_plus"] - a["loss_minus"]) >= TOL.HIGH_SIGNAL})
    rep = {"golden": name, "precision": h["precision"],
           "max_dL": max(max(abs(r["dLp"]), abs(r["dLm"])) for r in rows),
           "max_rel_dc_high_signal": max((r["rel_dc"] for r in rows if r["high_signal"]), default=0.0),
           "max_rel_dc": max(r["rel_dc"] for r in rows), "eval_loss": run.eval_curve[-1].loss,
           "eval_loss_ref": fin["eval_loss"], "rows": rows}
    _report(f"real32_traj_{name}", rep)
    assert rep["max_dL"] <= TOL.REAL32_LOSS, rep
    assert rep["max_rel_dc_high_signal"] <= TOL.REAL32_C_REL, rep
    # low-signal steps: the probe difference itself within two loss tolerances (an fp32 loss
    # of ~5 has a 4.8e-7 ulp, so c of a 1e-4 difference is only known to ~1e-3 relative)
    assert max(r["d_diff"] for r in rows) <= 2 * TOL.REAL32_LOSS, rep
    assert abs(rep["eval_loss"] - rep["eval_loss_ref"]) <= TOL.REAL32_LOSS, rep
