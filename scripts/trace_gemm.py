#!/usr/bin/env python
"""Per-CTA timeline of the four layer GEMMs at a BASELINE shape (zo_trace_gemm): for every
persistent CTA the MMA window and the epilogue window of each tile segment (globaltimer),
summarised as the launch span, the tiles per CTA, the idle tail (CTAs that finished early)
and the exposed last epilogue.

    python scripts/trace_gemm.py [--model opt-13b] [--json gpurun_out/gemm_trace.json]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def summarise(tr):
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    us = lambda x: (int(x) - int(t0)) / 1000.0
    rows = []
    for c in range(tr.shape[0]):
        mma = [(us(tr[c, 2 + 2 * i]), us(tr[c, 3 + 2 * i])) for i in range(15) if tr[c, 2 + 2 * i] > 0]
        epi = [(us(tr[c, 32 + 2 * i]), us(tr[c, 33 + 2 * i])) for i in range(15)
               if tr[c, 32 + 2 * i] > 0 and tr[c, 33 + 2 * i] > 0]
        rows.append({"cta": c, "start": us(tr[c, 0]), "end": us(tr[c, 1]), "mma": mma, "epi": epi})
    leaders = [r for r in rows if r["mma"]]
    span = max(r["end"] for r in rows)
    last_mma = [r["mma"][-1][1] for r in leaders]
    last_epi = [r["epi"][-1][1] for r in rows if r["epi"]]
    return {"span_us": span, "segments_per_leader": sorted({len(r["mma"]) for r in leaders}),
            "mma_busy_us_mean": float(np.mean([sum(b - a for a, b in r["mma"]) for r in leaders])),
            "last_mma_end_us": [float(min(last_mma)), float(np.mean(last_mma)), float(max(last_mma))],
            "last_epilogue_end_us": [float(min(last_epi)), float(np.mean(last_epi)), float(max(last_epi))],
            "sample": rows[:2] + rows[-2:]}


def main():
    from bench import MODELS
    from paper_2605_28760_b200.engine import ZoEngine
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-13b", choices=sorted(MODELS))
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    mdl = MODELS[a.model]
    eng = ZoEngine(mdl["vocab"], mdl["dim"], mdl["n_layers"], mdl["n_heads"], 63, max_batch=a.batch, rank=2)
    eng.init_params(7, 0.02)
    out = {}
    for w, name in enumerate(["qkv", "attn_out", "ff_up", "ff_down"]):
        s = summarise(eng.trace_gemm(w, a.batch).astype(np.int64))
        out[name] = s
        print(f"{name:8s} span {s['span_us']:7.1f} us  segments/CTA {s['segments_per_leader']}  "
              f"MMA busy {s['mma_busy_us_mean']:6.1f} us  last MMA end min/mean/max "
              f"{s['last_mma_end_us'][0]:.1f}/{s['last_mma_end_us'][1]:.1f}/{s['last_mma_end_us'][2]:.1f}  "
              f"last epilogue end {s['last_epilogue_end_us'][0]:.1f}/{s['last_epilogue_end_us'][1]:.1f}/"
              f"{s['last_epilogue_end_us'][2]:.1f}", flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
