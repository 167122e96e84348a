"""Isolated layer-GEMM times (zo_bench_gemm) for env-switched A/B runs, 13B dims by default:
    ZO_RES_TMA=0 python scripts/ab_gemm.py ; ZO_RES_TMA=1 python scripts/ab_gemm.py
    python scripts/ab_gemm.py --dim 2048 --heads 32      (OPT-1.3B layer shapes)
Prints us per launch and the achieved TF/s of each of the four layer GEMMs."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=5120)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--iters", type=int, default=40)
    a = ap.parse_args()
    from paper_2605_28760_b200.engine import ZoEngine
    eng = ZoEngine(50272, a.dim, 2, a.heads, 63, max_batch=a.batch, rank=2)
    eng.init_params(7, 0.02)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("ZO_")}, "dim": a.dim}
    for name, which in (("qkv", 0), ("attn_out", 1), ("ff_up", 2), ("ff_down", 3)):
        eng.bench_gemm(which, a.batch, 5)
        ms, tf = eng.bench_gemm(which, a.batch, a.iters)
        out[name] = round(ms * 1e3, 1)
        out[name + "_tf"] = round(tf / (ms * 1e-3) / 1e12, 0)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
