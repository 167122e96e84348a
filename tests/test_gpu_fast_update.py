"""The tensor-core factorized dense update (zo_set_update_mode 1; BASELINE config 5):
W += (-(lr*c)/sqrt(r)) U V^T (zo_engine.py:449-450) with U V^T on tcgen05 (16-bit operands,
fp32 accumulate) fused into the master / 16-bit-shadow read-modify-write.  In this mode the
projection and embedding masters are held as fp32 (10 instead of 18 bytes per weight per
update); switching modes converts them in place.

Stated tolerance: each step's update agrees with the reference's float64 axpy_outer to
1e-2 of its own magnitude (16-bit rounding of the N(0,1) directions, ~3e-3 RMS); the exact
mode stays bit-exact (test_gpu_api.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
UPDATE_REL = 1e-2


@pytest.mark.parametrize("rank", [16, 128])
def test_tensor_update_matches_float64(rank):
    from paper_2605_28760_b200.engine import ZoEngine
    eng = ZoEngine(256, 64, 2, 2, 16, max_batch=8, rank=rank, estimator="factorized_sqrt_r")
    eng.init_params(7, 0.08)
    eng.set_update_mode("tensor")
    eng.sample_v(42, 3, 1)
    eng.sample_u(42, 3)
    U = eng.split(0, eng.get_slot(0))
    V = eng.split(1, eng.get_slot(1))
    before = {lid: eng.download(lid) for lid in eng.lids}
    lr, c = 1e-3, 37.5
    eng.set_coefficient(np.array([4.0, 3.9, c, -(lr * c)]))
    eng.update_dense(lr)
    alpha = -(lr * c) / np.sqrt(rank)
    for lid in eng.lids:
        want_delta = alpha * (U[lid] @ V[lid].T)
        got_delta = eng.download(lid) - before[lid]
        err = np.max(np.abs(got_delta - want_delta)) / np.max(np.abs(want_delta))
        assert err <= UPDATE_REL, (lid, err)
    eng.close()


def test_tensor_update_trajectory_close_to_exact():
    """Three factorized steps (r = 32) in both modes: same losses within the fp16 scorer noise,
    parameters within the per-step update tolerance."""
    from paper_2605_28760_b200.engine import ZoEngine
    from oracle import reference as R
    cfg = R.ModelCfg(vocab=256, dim=64, n_layers=2, n_heads=2, prompt_len=15, init_seed=7, init_scale=0.08)
    splits = R.generate_task(R.TaskCfg(seed=11, vocab=256, prompt_len=15, train_size=64, dev_size=4, val_size=4))
    engs = {}
    for mode in ("exact", "tensor"):
        e = ZoEngine(256, 64, 2, 2, 15, max_batch=8, rank=32, estimator="factorized_sqrt_r")
        e.init_params(cfg.init_seed, cfg.init_scale)
        e.set_update_mode(mode)
        engs[mode] = e
    before = {lid: engs["exact"].download(lid) for lid in engs["exact"].lids}
    outs = {m: [] for m in engs}
    for t in range(3):
        p, gl, idx = R.sample_minibatch(splits, "train", 42, t, 8)
        gold = np.array([[254], [255]])[gl]
        tokens = np.concatenate([p, gold], axis=1)
        for m, e in engs.items():
            outs[m].append(e.step(42, t, 1, 1e-3, 1e-3, False, tokens, gold))
    for a, b in zip(outs["exact"], outs["tensor"]):
        assert abs(a[0] - b[0]) < 1e-3 and abs(a[1] - b[1]) < 1e-3
    for lid in engs["exact"].lids:
        de = engs["exact"].download(lid) - before[lid]
        dt = engs["tensor"].download(lid) - before[lid]
        assert np.max(np.abs(dt - de)) <= 2 * UPDATE_REL * np.max(np.abs(de)), lid
    for e in engs.values():
        e.close()


def test_fp32_master_mode_switch():
    """Entering the tensor mode narrows the masters to fp32 in place (downloads read them back
    widened), the scorer's embedding gather then reads the fp32 master -- the same fp32 values
    the float64 path rounds to, so the NLLs are bitwise unchanged -- and leaving the mode widens
    them again exactly."""
    from paper_2605_28760_b200.engine import ZoEngine
    eng = ZoEngine(256, 64, 2, 2, 15, max_batch=8, rank=32, estimator="factorized_sqrt_r")
    eng.init_params(7, 0.08)
    before = {lid: eng.download(lid) for lid in eng.lids}
    rng = np.random.default_rng(0)
    tok = rng.integers(0, 256, size=(8, 16)).astype(np.int32)
    gold = tok[:, -1:].copy()
    eng.prepare_probe(1e-3, 1)
    nll64 = eng.score(tok, gold, nsign=1)
    eng.set_update_mode("tensor")
    for lid in eng.lids:
        assert np.array_equal(eng.download(lid), before[lid].astype(np.float32).astype(np.float64)), lid
    eng.prepare_probe(1e-3, 1)
    assert np.array_equal(eng.score(tok, gold, nsign=1), nll64)
    # an upload in fp32-master mode lands rounded to fp32
    w = before["blk0.qkv"] * 1.5
    eng.upload({"blk0.qkv": w})
    assert np.array_equal(eng.download("blk0.qkv"), w.astype(np.float32).astype(np.float64))
    eng.set_update_mode("exact")
    for lid in eng.lids:
        want = (w if lid == "blk0.qkv" else before[lid]).astype(np.float32).astype(np.float64)
        assert np.array_equal(eng.download(lid), want), lid
    eng.close()
