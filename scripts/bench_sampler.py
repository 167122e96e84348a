"""Direction-sampler throughput (zo_sample_u: k_keys + k_spec + k_scan + k_emit_copy) at 13B
layer dims, factorized r = 128 (the config-5 U plan per layer set):
    python scripts/bench_sampler.py [--layers 4] [--rank 128] [--reps 10]
Prints ms per U-plan sample and normals/s."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--rank", type=int, default=128)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    from paper_2605_28760_b200.engine import ZoEngine
    eng = ZoEngine(50272, 5120, a.layers, 40, 63, max_batch=16, rank=a.rank, estimator="factorized_sqrt_r")
    eng.init_params(7, 0.02)
    eng.sample_u(42, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(a.reps):
        eng.sample_u(42, i + 1)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / a.reps
    print(json.dumps({"layers": a.layers, "rank": a.rank, "normals": int(eng.su), "ms": round(ms, 3),
                      "normals_per_s": eng.su / (ms * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
