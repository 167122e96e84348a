import sys, time, subprocess
sys.path.insert(0, '.')
from paper_2605_28760_b200.engine import ZoEngine
eng = ZoEngine(50272, 5120, 40, 40, 63, max_batch=16, rank=2)
eng.init_params(7, 0.02)
for reps in (20, 200, 2000, 20):
    ms, fl = eng.bench_gemm(0, 16, reps)
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(f"qkv reps={reps}: {ms*1e3:.1f} us  {fl/(ms*1e-3)/1e12:.0f} TF/s   after: {clk}", flush=True)
for w, name in ((1, "attn_out"), (2, "ff_up"), (3, "ff_down")):
    for reps in (20, 1000):
        ms, fl = eng.bench_gemm(w, 16, reps)
        print(f"{name} reps={reps}: {ms*1e3:.1f} us  {fl/(ms*1e-3)/1e12:.0f} TF/s", flush=True)
