"""Time the factorized dense update alone (zo_update_dense) at 13B layer dims.
    python scripts/bench_update.py [--layers 4] [--rank 128] [--mode tensor]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--rank", type=int, default=128)
    ap.add_argument("--mode", default="tensor")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    from paper_2605_28760_b200.engine import ZoEngine
    eng = ZoEngine(50272, 5120, a.layers, 40, 63, max_batch=16, rank=a.rank, estimator="factorized_sqrt_r")
    eng.init_params(7, 0.02)
    eng.set_update_mode(a.mode)
    eng.sample_v(42, 1, 1)
    eng.sample_u(42, 1)
    eng.set_coefficient(np.array([4.0, 3.9, 10.0, -1e-6]))
    eng.update_dense(1e-7)
    torch.cuda.synchronize()
    weights = sum(m * n for m, n in eng.shapes.values())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        eng.update_dense(1e-7)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    bpw = 10 if a.mode == "tensor" else 18
    print(json.dumps({"mode": a.mode, "weights": weights, "ms": ms,
                      "GBps_algorithmic": bpw * weights / ms / 1e6}))


if __name__ == "__main__":
    main()
