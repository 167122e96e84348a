"""CPU-only tests: the C ABI library loads and exports every declared symbol,
host logic (digests, canonical mean, task/minibatch data prep, configs) matches
the reference's golden vectors, and the multi-rank NLL exchange reproduces the
single-process coefficient (gloo, world_size 2)."""
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from oracle import reference as R

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(REPO, "include", "zob200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(zo_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_28760_b200 import build
    build.build()
    from paper_2605_28760_b200 import _lib
    return _lib.lib()


def test_library_exports_every_declared_symbol(lib):
    syms = _header_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (zo_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    from paper_2605_28760_b200 import _lib
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(syms) <= bound, sorted(set(syms) - bound)


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib._name], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs
    sass = subprocess.run(["cuobjdump", "-sass", lib._name], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05.mma, TMA, tcgen05.ld


def test_no_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_28760_b200.engine import ZoEngine
    with pytest.raises(RuntimeError):
        ZoEngine(64, 32, 2, 2, 16)


def test_fnv_and_digest_chain(lib, golden_dir):
    from paper_2605_28760_b200 import numerics as N
    v = json.load(open(os.path.join(golden_dir, "fnv.json")))
    assert N.digest_hex(N.digest_bytes(b"")) == v["empty"]
    assert N.digest_hex(N.digest_bytes(b"foobar")) == v["foobar"]
    assert N.digest_hex(N.digest_text("params")) == v["params"]
    assert N.digest_hex(N.digest_array(np.arange(8, dtype=np.float64))) == v["arange8"]
    assert N.digest_hex(N.digest_array(np.array([1.5, -2.25]), N.digest_text("blk0.qkv"))) == v["chain"]
    # zo_digest_chain == the reference's _chain over sorted ids (zo_engine.py:220-221)
    import ctypes
    rng = np.random.default_rng(0)
    lids = ["blk0.attn_out", "blk0.ff_down", "embed"]
    arrs = [rng.standard_normal((5, 2)), rng.standard_normal((7, 2)), rng.standard_normal((3, 2))]
    arena = np.concatenate([a.reshape(-1) for a in arrs])
    offs = np.cumsum([0] + [a.size for a in arrs[:-1]])
    got = lib.zo_digest_chain((ctypes.c_char_p * 3)(*[l.encode() for l in lids]), arena.ctypes.data,
                              (ctypes.c_int64 * 3)(*offs), (ctypes.c_int64 * 3)(*[a.size for a in arrs]), 3,
                              R.FNV_OFFSET_BASIS)
    h = R.FNV_OFFSET_BASIS
    for lid, a in zip(lids, arrs):
        h = R.digest_array(a, R.digest_text(lid, h))
    assert got == h


def test_canonical_mean_matches_oracle(lib):
    from paper_2605_28760_b200.numerics import canonical_mean
    rng = np.random.default_rng(1)
    for n in (1, 2, 3, 7, 16, 33):
        v = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 8, n)
        assert canonical_mean(v) == R.canonical_mean(v)
        assert canonical_mean(np.concatenate([v, v])) == canonical_mean(v)


@pytest.mark.parametrize("name", ["micro_lozo", "small_lozo"])
def test_task_minibatch_and_config_digests(lib, golden_dir, name):
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.zo_engine import ZoConfig
    lines = [json.loads(l) for l in open(os.path.join(golden_dir, f"traj_{name}.jsonl"))]
    h, recs = lines[0], [l for l in lines if l["record"] == "step"]
    task = M.generate_task(M.TaskConfig(**h["task"]))
    assert task.digest() == h["task_digest"]
    z = ZoConfig(**h["zo"])
    assert z.digest() == h["zo_digest"]
    for r in recs:
        mb = M.sample_minibatch(task, "train", z.seed, r["step"], z.batch_size)
        assert mb.batch_id == r["minibatch_id"]
    assert M.ModelConfig(**h["model"]).digest() == R.digest_hex(
        R.digest_text(json.dumps(dict(sorted(h["model"].items())), sort_keys=True)))


def test_pos_encoding_matches_oracle(lib):
    from paper_2605_28760_b200.model import pos_encoding
    np.testing.assert_array_equal(pos_encoding(64, 768), R.pos_encoding(64, 768))


def test_config_validation_mirrors_reference(lib):
    from paper_2605_28760_b200 import ConfigError
    from paper_2605_28760_b200.model import ModelConfig
    from paper_2605_28760_b200.zo_engine import ZoConfig
    with pytest.raises(ConfigError):
        ModelConfig(dim=30, n_heads=4)
    with pytest.raises(ConfigError):
        ZoConfig(epsilon=0)
    with pytest.raises(ConfigError):
        ZoConfig(scope="everything")


def test_canonical_order_layout():
    from paper_2605_28760_b200.dist import canonical_order
    world, bl = 4, 4
    # rank r holds [sign][b] for examples r*bl .. r*bl+bl-1, value = sign*100 + example
    g = np.array([[[s * 100 + r * bl + b for b in range(bl)] for s in range(2)] for r in range(world)], float)
    out = canonical_order(g.reshape(-1), world, bl)
    np.testing.assert_array_equal(out, [[s * 100 + e for e in range(world * bl)] for s in range(2)])


_WORKER = r"""
import os, sys, json
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {repo!r})
from paper_2605_28760_b200.dist import exchange_nll, shard_range
from paper_2605_28760_b200.numerics import canonical_mean
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]), world_size=2)
rank = dist.get_rank()
B = 16
rng = np.random.default_rng(123)
full = rng.standard_normal((2, B)) * 0.1 + 4.0        # the NLLs a single GPU would produce
lo, hi = shard_range(B, rank, 2)
local = torch.from_numpy(np.ascontiguousarray(full[:, lo:hi])).double()
glob = exchange_nll(local, 2).numpy()
lp, lm = canonical_mean(glob[0]), canonical_mean(glob[1])
c = (lp - lm) / (2.0 * 1e-3)
ref = (canonical_mean(full[0]) - canonical_mean(full[1])) / (2.0 * 1e-3)
print(json.dumps({{"rank": rank, "c": c, "ref": ref}}))
dist.destroy_process_group()
"""


def test_exact_mode_exchange_gloo_world2(tmp_path):
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    script = tmp_path / "w.py"
    script.write_text(_WORKER.format(repo=REPO, port=port))
    procs = [subprocess.Popen([sys.executable, str(script), str(r)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for r in range(2)]
    outs = [p.communicate(timeout=240) for p in procs]
    res = [json.loads(o[0].strip().splitlines()[-1]) for o in outs]
    assert res[0]["c"] == res[1]["c"] == res[0]["ref"]  # bitwise: identical c on every rank


_QDIR_WORKER = r"""
import os, sys, json
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {repo!r})
from oracle import reference as R
from paper_2605_28760_b200.dist import exchange_out4, qdir_steps, fold_due, check_qdir
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]), world_size=2)
g, G, nu = dist.get_rank(), 2, 4
check_qdir(G, nu)
cfg = R.ModelCfg(vocab=64, dim=16, n_layers=1, n_heads=2, prompt_len=7, init_seed=7, init_scale=0.08)
splits = R.generate_task(R.TaskCfg(seed=11, vocab=64, prompt_len=7, train_size=32, dev_size=4, val_size=4))
z = R.ZoCfg(seed=42, epsilon=1e-3, learning_rate=1e-2, rank=2, nu=nu, batch_size=4)
params = R.init_params(cfg)
st = R.LozoState()
def batch(s):
    p, gl, idx = R.sample_minibatch(splits, "train", z.seed, s, z.batch_size)
    gold = np.array([[cfg.vocab - 2], [cfg.vocab - 1]])[gl]
    return np.concatenate([p, gold], axis=1), gold, idx
for t in range(4):
    s = qdir_steps(t, G)[g]
    # this rank's direction only (the CPU stand-in for zo_qdir_score_async)
    sg = R.LozoState({{k: v.copy() for k, v in st.A.items()}}, R.window_v(params, z, s) if st.A else {{}})
    rec, _ = R.lozo_step(params, cfg, sg, z, s, *batch(s))
    out4 = torch.tensor([rec.loss_plus, rec.loss_minus, rec.coefficient, rec.beta], dtype=torch.float64)
    allc = exchange_out4(out4, G).numpy()
    st.V = sg.V
    for gg in range(G):  # zo_qdir_apply_async: every U regenerated, g order
        dirs, _, _ = R.step_dirs({{k: v.shape for k, v in params.items() if v.ndim == 2}}, z, t * G + gg)
        for lid, (u, _v) in dirs.items():
            st.A.setdefault(lid, np.zeros((params[lid].shape[0], z.rank)))
            st.A[lid] = st.A[lid] + allc[gg, 3] * u
    if fold_due(t, G, nu):
        R.fold_all(params, st)
print(json.dumps({{"rank": g, "digest": R.params_digest(params),
                  "a": float(sum(np.abs(a).sum() for a in st.A.values()))}}))
dist.destroy_process_group()
"""


def test_qdir_mode_exchange_gloo_world2(tmp_path):
    """Two ranks each score one direction per macro-step, exchange [L+,L-,c,beta] over
    gloo and apply both updates: both replicas end bit-identical to the single-process
    q-direction oracle (oracle.reference.qdir_macro_step)."""
    import socket
    sys.path.insert(0, REPO)
    from oracle import reference as R
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    script = tmp_path / "q.py"
    script.write_text(_QDIR_WORKER.format(repo=REPO, port=port))
    procs = [subprocess.Popen([sys.executable, str(script), str(r)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for r in range(2)]
    outs = [p.communicate(timeout=240) for p in procs]
    res = [json.loads(o[0].strip().splitlines()[-1]) for o in outs]
    assert res[0] == {**res[1], "rank": 0}
    # single-process restatement
    G, nu = 2, 4
    cfg = R.ModelCfg(vocab=64, dim=16, n_layers=1, n_heads=2, prompt_len=7, init_seed=7, init_scale=0.08)
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=64, prompt_len=7, train_size=32, dev_size=4, val_size=4))
    z = R.ZoCfg(seed=42, epsilon=1e-3, learning_rate=1e-2, rank=2, nu=nu, batch_size=4)
    params = R.init_params(cfg)
    st = R.LozoState()
    for t in range(4):
        bs = []
        for s in range(t * G, t * G + G):
            p, gl, idx = R.sample_minibatch(splits, "train", z.seed, s, z.batch_size)
            gold = np.array([[cfg.vocab - 2], [cfg.vocab - 1]])[gl]
            bs.append((np.concatenate([p, gold], axis=1), gold, idx))
        R.qdir_macro_step(params, cfg, st, z, t, G, bs)
        if ((t + 1) * G) % nu == 0:
            R.fold_all(params, st)
    assert res[0]["digest"] == R.params_digest(params)
    assert res[0]["a"] == float(sum(np.abs(a).sum() for a in st.A.values()))


def test_qdir_G1_oracle_is_lozo_step():
    """qdir_macro_step with G = 1 reproduces the reference's lozo_step exactly."""
    sys.path.insert(0, REPO)
    from oracle import reference as R
    cfg = R.ModelCfg(vocab=64, dim=16, n_layers=1, n_heads=2, prompt_len=7, init_seed=7, init_scale=0.08)
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=64, prompt_len=7, train_size=32, dev_size=4, val_size=4))
    z = R.ZoCfg(seed=42, epsilon=1e-3, learning_rate=1e-2, rank=2, nu=2, batch_size=4)
    pa, pb = R.init_params(cfg), R.init_params(cfg)
    sa, sb = R.LozoState(), R.LozoState()
    for t in range(4):
        p, gl, idx = R.sample_minibatch(splits, "train", z.seed, t, z.batch_size)
        gold = np.array([[cfg.vocab - 2], [cfg.vocab - 1]])[gl]
        tok = np.concatenate([p, gold], axis=1)
        ra, _ = R.lozo_step(pa, cfg, sa, z, t, tok, gold, idx)
        (rb,) = R.qdir_macro_step(pb, cfg, sb, z, t, 1, [(tok, gold, idx)])
        assert ra == rb
        if (t + 1) % z.nu == 0:
            R.fold_all(pa, sa)
            R.fold_all(pb, sb)
    assert R.params_digest(pa) == R.params_digest(pb)
