"""Isolated layer-GEMM times at 13B dims (zo_bench_gemm), for env-switched A/B runs:
    ZO_RES_TMA=0 python scripts/ab_gemm.py ; ZO_RES_TMA=1 python scripts/ab_gemm.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2605_28760_b200.engine import ZoEngine
    eng = ZoEngine(50272, 5120, 2, 40, 63, max_batch=16, rank=2)
    eng.init_params(7, 0.02)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("ZO_")}}
    for name, which in (("qkv", 0), ("attn_out", 1), ("ff_up", 2), ("ff_down", 3)):
        eng.bench_gemm(which, 16, 5)
        ms, tf = eng.bench_gemm(which, 16, 40)
        out[name] = round(ms * 1e3, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
