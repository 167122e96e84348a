"""One fused LoZO step at a shape that exercises the whole 13B GEMM schedule -- CTA-pair
tiles, the stream-K tail (ff_down at d = 5120, M = 2016), half-width tail tiles, the
fused extension partials -- plus the split-vocabulary loss, the sampler, the device
update/fold, a factorized step through the fp32-master tensor update (EPI_UPDATE32),
the split-step graphs and a non-finite abort.  Run under compute-sanitizer
(scripts/sanitize.sh); prints "sanitize shapes ok".

    python scripts/sanitize_shapes.py [--small]
--small: d = 1024 (CTA pairs + half tails, no stream-K) for the slow racecheck/synccheck tools.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true")
    args = ap.parse_args()
    import torch

    from paper_2605_28760_b200.engine import ZoEngine
    from paper_2605_28760_b200.errors import ScoringAbort
    D, H, L = (1024, 8, 2) if args.small else (5120, 40, 2)
    V, T, B = 4096, 64, 16
    rng = np.random.default_rng(0)
    tok = rng.integers(0, V, size=(B, T)).astype(np.int32)
    gold = tok[:, -1:].copy()
    # LoZO r = 2: eager step (fold at the window end), graph step, split-step graphs
    eng = ZoEngine(V, D, L, H, T - 1, max_batch=B, rank=2)
    eng.init_params(7, 0.02)
    for t in range(3):
        eng.step(42, t, 2, 1e-3, 1e-5, False, tok, gold)
    eng.fold()
    d_tok = torch.from_numpy(tok).cuda()
    d_gold = torch.from_numpy(np.stack([gold, gold])).cuda()
    eng.step_graph(42, 3, 2, 1e-3, 1e-5, False, d_tok.data_ptr(), d_gold.data_ptr(), B)
    eng.step_graph(42, 4, 2, 1e-3, 1e-5, False, d_tok.data_ptr(), d_gold.data_ptr(), B)
    eng.step_score_graph(42, 5, 2, 1e-3, d_tok.data_ptr(), d_gold.data_ptr(), B)
    eng.step_apply_graph(1e-3, 1e-5, False, B)
    eng.set_schedule("row_invariant")
    eng.step(42, 6, 2, 1e-3, 1e-5, False, tok, gold)
    eng.prepare_probe(0.0, 1)
    eng.score_options(tok, [1, 2, 3])
    eng.synchronize()
    eng.close()
    # factorized r = 32 (high-rank extension GEMMs, merged signs) with the fp32-master update
    eng = ZoEngine(V, D, L, H, T - 1, max_batch=B, rank=32, estimator="factorized_sqrt_r")
    eng.init_params(7, 0.02)
    eng.set_update_mode("tensor")
    for t in range(2):
        eng.step(42, t, 1, 1e-3, 1e-5, False, tok, gold)
    E = eng.download("embed")
    E[tok[0, 3], :] = np.inf
    eng.upload({"embed": E})
    try:
        eng.step(42, 2, 1, 1e-3, 1e-5, False, tok, gold)
        raise SystemExit("expected ScoringAbort")
    except ScoringAbort:
        pass
    eng.set_update_mode("exact")
    eng.synchronize()
    eng.close()
    print("sanitize shapes ok")


if __name__ == "__main__":
    main()
