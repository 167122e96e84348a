#!/usr/bin/env python
"""The paper's Phase 3 table on one B200: core-step time of the serving path vs the
materialising training loop (baseline_loop.py, the "official baseline" structure) by
model and batch size, both through bench.py (CUDA events, device-resident inputs).

    python scripts/phase3_sweep.py [--models opt-125m,opt-1.3b,opt-6.7b,opt-13b] [--batches 8,16,32]
Writes one JSON object per (model, batch) to stdout and the table to gpurun_out/phase3.json.
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="opt-125m,opt-1.3b,opt-6.7b,opt-13b")
    ap.add_argument("--batches", default="8,16,32")
    ap.add_argument("--steps", type=int, default=30)
    a = ap.parse_args()
    rows = []
    for model in a.models.split(","):
        for b in a.batches.split(","):
            cmd = [sys.executable, os.path.join(HERE, "bench.py"), "--model", model, "--batch", b,
                   "--steps", str(a.steps), "--no-cpu-baseline", "--no-e2e", "--materialising-steps", "6"]
            out = subprocess.run(cmd, capture_output=True, text=True, cwd=HERE, timeout=900)
            try:
                d = json.loads(out.stdout.strip().splitlines()[-1])
            except Exception:
                print(json.dumps({"model": model, "batch": int(b), "error": out.stderr[-400:]}), flush=True)
                continue
            m = d.get("materialising_loop", {})
            row = {"model": model, "batch": int(b), "serving_ms": d["ms_per_step"],
                   "serving_steps_per_s": d["value"], "materialising_ms": m.get("ms_per_step"),
                   "speedup": m.get("speedup_of_serving_path"), "sm_mhz": d["clocks"]["sm_mhz"]}
            rows.append(row)
            print(json.dumps(row), flush=True)
    os.makedirs(os.path.join(HERE, "gpurun_out"), exist_ok=True)
    with open(os.path.join(HERE, "gpurun_out", "phase3.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
