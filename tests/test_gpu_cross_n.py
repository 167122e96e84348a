"""Determinism across GPU counts (SURVEY.md §7 H6, §8(e) exact mode) on one GPU.

Exact-trajectory mode slices the global minibatch over N ranks: rank g scores
examples [g*B/N, (g+1)*B/N) for both probe signs, so each GPU runs the layer
GEMMs at M = 2*(B/N)*(T-1) rows.  Here the N ranks are emulated on one device by
scoring the N slices one after the other with the same engine state.

* ``row_invariant`` schedule (zo_set_schedule(1), what exact mode runs): the
  per-example NLLs of every slicing (N = 1, 2, 4, 8) are BITWISE equal -- so c
  and the update are too -- although M changes the tile width, the CTA pairing
  and the half-width tail of every GEMM.
* ``fast`` schedule (the N = 1 default, stream-K tails on the 13B ff_down and the 4-way
  tails on attn_out / qkv): the tails' fp32 partial sums change the last bits of the
  residual stream, which flips an occasional 16-bit rounding of the next LN output --
  observed up to 1.2e-3 relative (2.5e-2 absolute on NLLs of ~21) per-example NLL vs the
  row-invariant schedule, i.e. the fp16 scorer's own noise; bounded at 2.5e-3 relative.

Shape: OPT-13B dims (d = 5120, H = 40), two decoder blocks (the first runs every row --
the last block's attn_out / ff_up / ff_down only see the scored rows), B = 16, T = 64 -- the
configuration whose ff_down GEMM takes the stream-K tail at N = 1.
"""
import os
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

D, H, L, V, T, B = 5120, 40, 2, 4096, 64, 16
# fast vs row-invariant schedule, relative per-example NLL: observed 2.7e-4 with the stream-K
# tail on ff_down only, 1.2e-3 once the 4-way tail also covers qkv / attn_out (N = 2: 1008 rows)
# -- fp16 rounding flips in differently-summed tail tiles, amplified by this random-init
# model's NLLs of ~21 (the GEMMs themselves match fp32 torch, test_gemm_streamk_four_way_tail)
FAST_REL = 2.5e-3


@pytest.fixture(scope="module")
def eng13():
    import torch

    from paper_2605_28760_b200.engine import ZoEngine
    eng = ZoEngine(V, D, L, H, T - 1, max_batch=B, rank=2)
    eng.set_stream(torch.cuda.current_stream().cuda_stream)
    eng.init_params(7, 0.02)
    # a non-zero window A so the +-eps probes differ from W0 in every extension column
    eng.step(42, 0, 50, 1e-3, 1e-3, False, *_batch(np.random.default_rng(3)))
    yield eng
    eng.close()


def _batch(rng):
    tok = rng.integers(0, V, size=(B, T), dtype=np.int32)
    return tok, tok[:, -1:].copy()


def _score_sliced(eng, tok, gold, world, step=1):
    """Per-example NLLs [2, B] with the batch sliced over `world` emulated ranks."""
    import torch
    bl = B // world
    out = torch.empty(world, 2, bl, dtype=torch.float64, device="cuda")
    for g in range(world):
        d_tok = torch.from_numpy(np.ascontiguousarray(tok[g * bl:(g + 1) * bl])).cuda()
        d_gold = torch.from_numpy(np.ascontiguousarray(gold[g * bl:(g + 1) * bl])).cuda()
        eng.step_score_async(42, step, 50, 1e-3, d_tok.data_ptr(), d_gold.data_ptr(), bl)
        eng.nll_io(out[g].data_ptr(), 2 * bl, False)
        torch.cuda.synchronize()
    return out.transpose(0, 1).reshape(2, B).cpu().numpy()  # canonical [sign][example]


def test_row_invariant_schedule_is_bitwise_across_gpu_counts(eng13):
    tok, gold = _batch(np.random.default_rng(5))
    eng13.set_schedule("row_invariant")
    try:
        ref = _score_sliced(eng13, tok, gold, 1)
        assert np.isfinite(ref).all()
        for world in (2, 4, 8):
            got = _score_sliced(eng13, tok, gold, world)
            bad = np.flatnonzero(got.reshape(-1) != ref.reshape(-1))
            assert bad.size == 0, (world, bad[:8], np.abs(got - ref).max())
    finally:
        eng13.set_schedule("fast")


def test_fast_schedule_tolerance_across_gpu_counts(eng13):
    tok, gold = _batch(np.random.default_rng(6))
    eng13.set_schedule("row_invariant")
    inv = _score_sliced(eng13, tok, gold, 1)
    eng13.set_schedule("fast")
    rep = {}
    for world in (1, 2, 4, 8):
        got = _score_sliced(eng13, tok, gold, world)
        dif = float(np.max(np.abs(got - inv)))
        rep[world] = {"max_abs_vs_row_invariant": dif, "max_rel_vs_row_invariant": float(np.max(np.abs(got - inv) / np.abs(inv))),
                      "bitwise_equal": bool(np.array_equal(got, inv))}
    os.makedirs("gpurun_out/parity", exist_ok=True)
    with open("gpurun_out/parity/cross_n_opt13b_block.json", "w") as f:
        json.dump(rep, f, indent=1)
    for world, r in rep.items():
        assert r["max_rel_vs_row_invariant"] <= FAST_REL, (world, r)
