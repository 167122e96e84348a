#!/usr/bin/env python
"""bench.py -- ZO steps/s + scored tokens/s of the LoZO serving step
(BASELINE.json metric) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--model opt-13b] [--impl ours|reference]

Workload (N=1): OPT-13B-shaped decoder (d=5120, L=40, H=40, V=50272; the
reference's architecture, model.py:170-199), LoZO rank-2 LoRA-only, SST-2
shape B=16 x T=64 (prompt 63 + 1 option token), nu=50, eps=1e-3, lr=1e-7,
random init (Role.INIT streams, init_scale 0.02) on synthetic marker-task
batches.  One step = directions (U; V + fold at window boundaries) + both
probes scored in one fused forward + canonical-mean coefficient + rank-r
update, exactly lozo_step + run_serving_path's fold policy.

value : steps/s over K device-timed steps (CUDA events on the engine stream,
        inputs resident in HBM, weights 25.7 GB >> 126 MB L2 so no flush).
e2e   : the same through the public API (sample_minibatch + lozo_step with
        host batches: H2D tokens from pinned staging, D2H of L+/L-/c) -- wall clock.
N > 1 : --mode qdir (default; BASELINE config 3 "query directions sharded") --
        rank g scores the direction and minibatch of reference step t*N+g on a
        full B=16 batch at the shared state of macro-step t; the [L+,L-,c,beta]
        of every rank are all-gathered over NCCL (32 B/rank) and every rank
        regenerates the N counter-keyed U's and applies the N updates in rank
        order (identical replicas, no weight traffic); value = reference steps/s
        of the whole job, "weak".  nu is rounded down to a multiple of N.
        --mode exact -- the 16 examples are split over ranks (both signs on every
        rank), the per-example NLLs are all-gathered (256 B/step) and every rank
        applies the identical update: the reference trajectory itself; "strong".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

MODELS = {
    "opt-125m": dict(vocab=50272, dim=768, n_layers=12, n_heads=12),
    "opt-1.3b": dict(vocab=50272, dim=2048, n_layers=24, n_heads=32),
    "opt-6.7b": dict(vocab=50272, dim=4096, n_layers=32, n_heads=32),
    "opt-13b": dict(vocab=50272, dim=5120, n_layers=40, n_heads=40),
}
METRIC = "ZO steps/sec + scored tokens/s, OPT-13B LoZO SST-2 shape, 1/2/4/8 B200"
UNIT = "ZO steps/s"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    """(HBM GB/s, bf16 TF/s burst, bf16 TF/s sustained, source)."""
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        burst = d.get("bf16_tflops", 1590.0)
        return d.get("hbm_gbs", 6650.0), burst, d.get("bf16_tflops_sustained", burst), "measured"
    return 6650.0, 1590.0, 1590.0, "fallback"


def layer_gemms(eng, B):
    """Per-launch device time of the four layer GEMMs + LM head (CUDA events on the
    engine stream, 20 back-to-back launches each, weights streamed from HBM)."""
    names = ["qkv", "attn_out", "ff_up", "ff_down", "lm_head"]
    g = {}
    for w in range(5):
        gms, gfl = eng.bench_gemm(w, B, 20)
        g[names[w]] = {"ms": gms, "tflops": gfl / (gms * 1e-3) / 1e12}
    lay_ms = sum(g[n]["ms"] for n in names[:4])
    lay_fl = sum(g[n]["tflops"] * g[n]["ms"] * 1e-3 * 1e12 for n in names[:4])
    return g, lay_ms, lay_fl / (lay_ms * 1e-3) / 1e12


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines = gpu, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(model):
    """DRAM bytes (read + write) of one launch of each of the four layer GEMMs, from the
    committed `ncu --set full` capture (profiles/), or None when not captured for this model."""
    import csv
    if model != "opt-13b":
        return None
    # the newest committed capture (profiles/capture.sh)
    cands = [os.path.join(HERE, "profiles", n) for n in ("r02_final/ncu_gemm_opt13b.csv", "r01g_ncu_gemm_opt13b.csv")]
    p = next((c for c in cands if os.path.exists(c)), None)
    if p is None:
        return None
    tot = 0.0
    with open(p) as f:
        rows = list(csv.DictReader(f))[:4]  # qkv, attn_out, ff_up, ff_down of layer 1
        for row in rows:
            tot += (float(row["dram__bytes_read.sum [Mbyte]"]) + float(row["dram__bytes_write.sum [Mbyte]"])) * 1e6
    return tot


def launches_per_step(L: int, n_mats: int, window: bool) -> int:
    # set_step + sampler(U) 5 + prep + embed + 9/layer (+2 gathers of the pruned last layer)
    # + final LN + LM GEMM + loss + coefficient + update
    n = 1 + 5 + 1 + 1 + 9 * L + 2 + 4 + 1
    if window:
        n += 5 + n_mats + n_mats  # sampler(V) + V extension writes + fold kernels
    return n


def dense_flops(dim, L, B, T, V, r, opt_len=1):
    tok = 2 * B * T
    dense = 24.0 * dim * dim * L * tok
    attn = 2 * B * L * 4 * T * T * dim * 2 / 2  # QK^T + AV, both signs
    head = 2.0 * (2 * B * opt_len) * dim * V
    lora = 2.0 * tok * r * (L * (dim + 3 * dim + dim + dim + dim + 4 * dim + 4 * dim + dim))
    return dense, dense + attn + head + lora


# --------------------------------------------------------------------------- CPU arms
def workload_config(args, world: int) -> tuple[dict, str, bool]:
    """The bench line's `config` (identical for both arms), `scaling`, and whether the
    N>1 run is in q-direction mode."""
    qdir = world > 1 and args.mode == "qdir"
    fact = args.estimator == "factorized_sqrt_r"
    B, T = args.batch, args.seq
    nu = args.nu
    if qdir and nu % world:
        nu = max(world, nu // world * world)
    upd = ("float64 dense update every step (bit-exact)" if args.dense_update == "exact" else
           "dense update every step as tcgen05 U V^T fused into the float64-master / 16-bit-shadow RMW")
    workload = (f"{args.model} factorized_sqrt_r (MeZO-style) r={args.rank} LoRA-only SST-2 shape, B={B} x T={T}, "
                f"{upd}" if fact else
                f"{args.model} LoZO r={args.rank} LoRA-only SST-2 shape, B={B} x T={T}, nu={nu}, "
                f"timed span centred on a window boundary (fold + V resample inside)")
    if args.arch == "opt":
        workload += ", OPT decoder (ReLU FFN, learned positions, projection biases)"
    cfg = {"workload": workload, "model": args.model, "global_batch": B, "seq_len": T,
           "parallelism": (f"qdir{world}" if qdir else f"exact-dp{world}") if world > 1 else "single",
           "l2": "inputs larger than L2 (25.7 GB 16-bit weights/step at 13B); no flush"}
    return cfg, ("strong" if (world > 1 and not qdir) else "weak"), qdir


def run_reference(args, mdl):
    """--impl reference: the reference's own path on host cores -- the unmodified zoserve
    staged in oracle/_ref (whole lozo_step calls at the model's dims with 1 and 2 blocks,
    depth-extrapolated), else the oracle port."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.cpu_bench import BlockSample, host_threads, reference_layers
    B, T = args.batch, args.seq
    got = reference_layers(mdl["dim"], mdl["n_layers"], mdl["n_heads"], mdl["vocab"], B, T) \
        if args.estimator == "lozo_lazy" and args.rank == 2 else None
    if got is not None:
        v, sample = got
        cfg, scaling, _ = workload_config(args, world)
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference", "config": cfg,
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": host_threads(), "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "scored_tokens_per_s": v * 2 * B * T}
        print(json.dumps(line), flush=True)
        return
    n_ex = 1
    bs = BlockSample(mdl["dim"], mdl["n_heads"], mdl["vocab"], T, n_ex)
    t_head = bs.run_head() * B
    for _ in range(args.warmup):
        bs.run()
    times = [bs.run() for _ in range(args.steps)]
    tc = float(np.mean([t[0] for t in times]))
    tf = float(np.mean([t[1] for t in times]))
    per_step = mdl["n_layers"] * (tc + B * tf) + t_head
    v = 1.0 / per_step
    sample = (f"oracle float64 port: per step 1 of {mdl['n_layers']} blocks, paired +-eps forward of 1 of {B} "
              f"sequences (T={T}, scaled x{B}) + the block's per-call composition; x{mdl['n_layers']} + LM-head rows")
    cfg, scaling, _ = workload_config(args, world)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference", "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": host_threads(), "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "scored_tokens_per_s": v * 2 * B * T}
    print(json.dumps(line), flush=True)


def config1_gpu(args, M, ZoEngine, torch, stream, steps: int = 50, warmup: int = 5) -> dict:
    """BASELINE config 1 (OPT-125m dims, B = 16, T = 64, r = 2, nu = 50) on this GPU: the fused
    step graph over device-resident batches, CUDA events, the window boundary inside."""
    mdl = MODELS["opt-125m"]
    mcfg = M.ModelConfig(vocab=mdl["vocab"], dim=mdl["dim"], n_layers=mdl["n_layers"], n_heads=mdl["n_heads"],
                         prompt_len=63, init_seed=7, init_scale=0.02)
    task = M.generate_task(M.TaskConfig(seed=11, vocab=mdl["vocab"], prompt_len=63, train_size=1000, dev_size=4,
                                        val_size=4))
    eng = ZoEngine(mcfg.vocab, mcfg.dim, mcfg.n_layers, mcfg.n_heads, 63, max_batch=16, rank=2,
                   precision=args.precision)
    eng.set_stream(stream.cuda_stream)
    eng.init_params(mcfg.init_seed, mcfg.init_scale)
    t0 = 50 - steps // 2 - warmup
    toks, golds = [], []
    for t in range(t0, t0 + warmup + steps):
        seq, gold = M.sample_minibatch(task, "train", 42, t, 16).sequences()
        toks.append(seq)
        golds.append(gold)
    d_tok = torch.from_numpy(np.asarray(toks, dtype=np.int32)).cuda()
    d_gold = torch.from_numpy(np.asarray(golds, dtype=np.int32)).cuda()

    def step(i):
        t = t0 + i
        eng.step_graph(42, t, 50, 1e-3, 1e-7, False, d_tok[i].data_ptr(), d_gold[i].data_ptr(), 16)
        if (t + 1) % 50 == 0:
            eng.fold_async()
    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(warmup, warmup + steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    eng.close()
    return {"value": 1000.0 / ms, "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "workload": "opt-125m LoZO r=2 LoRA-only SST-2 shape, B=16 x T=64, nu=50 (BASELINE config 1), "
                        f"timed steps {t0 + warmup}..{t0 + warmup + steps - 1} incl. the window boundary"}


# --------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--model", default="opt-13b", choices=sorted(MODELS))
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--seq", type=int, default=64)
    ap.add_argument("--rank", type=int, default=2)
    ap.add_argument("--estimator", default="lozo_lazy", choices=["lozo_lazy", "factorized_sqrt_r"],
                    help="factorized_sqrt_r = BASELINE config 5 (MeZO-style high-rank, e.g. --rank 128): "
                         "probe U V^T/sqrt(r), dense float64 update of every weight each step")
    ap.add_argument("--nu", type=int, default=50)
    ap.add_argument("--dense-update", default="exact", choices=["exact", "tensor"],
                    help="factorized_sqrt_r dense update: float64 bit-exact (default) or the tcgen05 U V^T "
                         "fused into the master/shadow update (HBM-bound, ~1e-3 of each step's update)")
    ap.add_argument("--precision", default="fp16", choices=["fp16", "bf16"])
    ap.add_argument("--arch", default="zoserve", choices=["zoserve", "opt"],
                    help="decoder: the reference's (default, parity-backed) or the OPT family's "
                         "(ReLU, learned positions, biases; real checkpoints load into it)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="launch kernels eagerly (no CUDA graph)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-materialising", dest="materialising", action="store_false",
                    help="skip the materialising training-loop comparand (baseline_loop.py) on the same GPU")
    ap.add_argument("--materialising-steps", type=int, default=6)
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no e2e/cpu/gemm microbench")
    ap.add_argument("--mode", default="qdir", choices=["qdir", "exact"],
                    help="N>1: qdir = query directions sharded (rank g scores reference step t*N+g on a full "
                         "batch, weak scaling); exact = the 16 examples split over ranks (strong scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    mdl = MODELS[args.model]
    if args.impl == "reference":
        run_reference(args, mdl)
        return

    import torch
    rank, world, local = dist_env()
    # ZO_BENCH_SAME_DEVICE=1 puts every rank on cuda:0 with gloo (a one-GPU functional test
    # of the N>1 path; timing meaningless) -- the real runs use NCCL, one GPU per rank
    same_dev = os.environ.get("ZO_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def all_gather(out, inp):
        import torch.distributed as dist
        if same_dev:  # gloo: exchange through host memory (a few bytes)
            o = out.cpu()
            dist.all_gather_into_tensor(o, inp.cpu())
            out.copy_(o)
        else:
            dist.all_gather_into_tensor(out, inp)
    from paper_2605_28760_b200 import model as M
    from paper_2605_28760_b200.adapter import AdapterState
    from paper_2605_28760_b200.engine import ZoEngine
    from paper_2605_28760_b200.zo_engine import ZoConfig, factorized_step, lozo_step

    B, T = args.batch, args.seq
    qdir = world > 1 and args.mode == "qdir"
    if qdir and args.nu % world:
        # the G directions of a macro-step must share one window (G | nu): round nu down
        # to a multiple of G (50 -> 48 at 4 and 8 GPUs; the fold is ~1% of a step)
        args.nu = max(world, args.nu // world * world)
    if not qdir and B % world:
        raise SystemExit("global batch must divide over ranks")
    Bl = B if qdir else B // world
    G = world if qdir else 1  # reference steps (directions) per timed step
    prompt_len = T - 1
    mcfg = M.ModelConfig(arch=args.arch, vocab=mdl["vocab"], dim=mdl["dim"], n_layers=mdl["n_layers"],
                         n_heads=mdl["n_heads"],
                         prompt_len=prompt_len, init_seed=7, init_scale=0.02)
    tcfg = M.TaskConfig(seed=11, vocab=mdl["vocab"], prompt_len=prompt_len, train_size=1000, dev_size=4,
                        val_size=4)
    fact = args.estimator == "factorized_sqrt_r"
    if fact:
        args.nu = 1
    zcfg = ZoConfig(seed=42, epsilon=1e-3, learning_rate=1e-7, rank=args.rank, nu=args.nu, batch_size=B,
                    estimator=args.estimator)
    task = M.generate_task(tcfg)
    t_init = time.perf_counter()
    eng = ZoEngine(mcfg.vocab, mcfg.dim, mcfg.n_layers, mcfg.n_heads, prompt_len, opt_len=1, max_batch=Bl,
                   rank=args.rank, estimator=args.estimator, precision=args.precision, device=local,
                   arch=args.arch, max_pos=mcfg.max_positions)
    stream = torch.cuda.current_stream()
    eng.set_stream(stream.cuda_stream)
    eng.init_params(mcfg.init_seed, mcfg.init_scale)
    if fact and args.dense_update == "tensor":
        eng.set_update_mode("tensor")
    if args.mode == "exact":
        # exact-trajectory mode: row-invariant GEMM schedule, so every slicing of the batch over
        # the ranks gives the N = 1 NLLs bit for bit (tests/test_gpu_cross_n.py)
        eng.set_schedule("row_invariant")
    torch.cuda.synchronize()
    t_init = time.perf_counter() - t_init

    # step schedule: the timed span is centred on a window boundary, so it contains the fold
    # of one window and the V resample of the next (runtime.py:327-330 / zo_engine.py:389-400)
    # -- with K < nu the boundary is over-represented (conservative for `value`)
    nu_m = max(1, zcfg.nu // G)  # macro-steps per window
    t_first = nu_m * -(-(args.warmup + args.steps // 2) // nu_m) - args.steps // 2
    t0_run = t_first - args.warmup
    nsteps = args.warmup + args.steps
    toks = np.zeros((nsteps, Bl, T), dtype=np.int32)
    golds = np.zeros((nsteps, Bl, 1), dtype=np.int32)
    for i in range(nsteps):
        t = t0_run + i
        if qdir:  # this rank's direction: reference step t*G + rank, full batch
            seq, gold = M.sample_minibatch(task, "train", zcfg.seed, t * G + rank, B).sequences()
            toks[i], golds[i] = seq, gold
            continue
        mb = M.sample_minibatch(task, "train", zcfg.seed, t, B)
        seq, gold = mb.sequences()
        toks[i] = seq[rank * Bl:(rank + 1) * Bl]
        golds[i] = gold[rank * Bl:(rank + 1) * Bl]
    d_tok = torch.from_numpy(toks).cuda()
    d_gold = torch.from_numpy(golds).cuda()
    nll_local = torch.zeros(2 * Bl, dtype=torch.float64, device="cuda")
    nll_all = torch.zeros(world * 2 * Bl, dtype=torch.float64, device="cuda")
    nll_full = torch.zeros(2 * B, dtype=torch.float64, device="cuda")  # canonical [sign][example]
    out4_local = torch.zeros(4, dtype=torch.float64, device="cuda")
    out4_all = torch.zeros(world * 4, dtype=torch.float64, device="cuda")

    def one_step(t, tp=None, gp=None):
        if tp is None:
            tp, gp = d_tok[t - t0_run].data_ptr(), d_gold[t - t0_run].data_ptr()
        if qdir:
            # score half and apply half as captured CUDA graphs (args.graph), the 32 B
            # all-gather between them
            score = eng.qdir_score_graph if args.graph else eng.qdir_score_async
            apply = eng.qdir_apply_graph if args.graph else eng.qdir_apply_async
            score(zcfg.seed, t, G, rank, zcfg.nu, zcfg.epsilon, zcfg.learning_rate, False, tp, gp, B)
            eng.out4_io(out4_local.data_ptr(), False)
            all_gather(out4_all, out4_local)  # 32 B per rank
            apply(zcfg.seed, t, G, zcfg.learning_rate, out4_all.data_ptr())
            if not fact and ((t + 1) * G) % zcfg.nu == 0:
                eng.fold_async()
            return
        if world == 1:
            if args.graph:
                eng.step_graph(zcfg.seed, t, zcfg.nu, zcfg.epsilon, zcfg.learning_rate, False, tp, gp, Bl)
            else:
                eng.step_async(zcfg.seed, t, zcfg.nu, zcfg.epsilon, zcfg.learning_rate, False, tp, gp, Bl)
        else:
            score = eng.step_score_graph if args.graph else eng.step_score_async
            apply = eng.step_apply_graph if args.graph else eng.step_apply_async
            score(zcfg.seed, t, zcfg.nu, zcfg.epsilon, tp, gp, Bl)
            eng.nll_io(nll_local.data_ptr(), 2 * Bl, False)
            all_gather(nll_all, nll_local)
            # [rank][sign][b] -> [sign][rank*Bl + b] (canonical example order)
            nll_full.view(2, world, Bl).copy_(nll_all.view(world, 2, Bl).transpose(0, 1))
            eng.nll_io(nll_full.data_ptr(), 2 * B, True)
            apply(zcfg.epsilon, zcfg.learning_rate, False, B)
        if not fact and (t + 1) % zcfg.nu == 0:
            eng.fold_async()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    cold = layer_gemms(eng, Bl) if (rank == 0 and not args.profile) else None
    for t in range(t0_run, t_first):
        one_step(t)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for t in range(t_first, t_first + args.steps):
            one_step(t)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    out4 = eng.read_out4()
    replicas_identical = None
    if world > 1:
        # every replica must hold the identical window A after the run (no weight traffic)
        import torch.distributed as dist
        from paper_2605_28760_b200.engine import A as SLOT_A
        dg = torch.tensor([eng.digest(SLOT_A) & ((1 << 62) - 1)], dtype=torch.int64,
                          device="cpu" if same_dev else "cuda")
        allg = [torch.zeros_like(dg) for _ in range(world)]
        dist.all_gather(allg, dg)
        replicas_identical = len({int(x.item()) for x in allg}) == 1
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device="cpu" if same_dev else "cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    value = 1000.0 * G / ms_step  # reference steps (ZO directions) per second, whole job
    windows = sum(1 for t in range(t_first, t_first + args.steps) if (t * G) % zcfg.nu == 0)
    per_step, per_window = eng.graph_kernel_count()
    split = eng.split_graph_kernels()  # [score, apply, qdir score, qdir apply] graph kernels
    if world > 1 and args.graph:
        # + the eager step-index write in front of the score graph (+ the macro-step base)
        per_step = (split[2] + split[3] + 2) if qdir else (split[0] + split[1] + 1)
        G_extra = 0
    else:
        G_extra = G - 1
        if not (world == 1 and args.graph) or per_step <= 1:
            per_step = launches_per_step(mcfg.n_layers, 4 * mcfg.n_layers + 1, False)  # eager paths: estimate
    launches = args.steps * (per_step + G_extra * 6) + (0 if fact else windows * per_window)

    hbm_peak, tf_peak, tf_sust, peak_kind = peaks()
    cfg, scaling, _ = workload_config(args, world)
    cfg["timed_steps"] = [t_first, t_first + args.steps - 1]
    cfg["window_boundaries_timed"] = windows
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None,
            "dtype": args.precision,
            "data": "synthetic (marker task, random-init Role.INIT weights)",
            "config": cfg,
            "scored_tokens_per_s": value * 2 * B * T, "option_tokens_per_s": value * 2 * B,
            "gpu_launches": launches, "clocks": clk.summary(), "init_s": t_init,
            **({"replicas_identical": replicas_identical} if world > 1 else {}),
            **({"split_graphs": {"score_kernels": split[2] if qdir else split[0],
                                 "apply_kernels": split[3] if qdir else split[1]}} if world > 1 and args.graph else {}),
            "last_losses": [float(out4[0]), float(out4[1]), float(out4[2])]}
    dense, total = dense_flops(mcfg.dim, mcfg.n_layers, B, T, mcfg.vocab, args.rank)
    line["step_tflops"] = total / 1e12
    line["step_tensor_util"] = {"achieved_tflops": total / (ms_step * 1e-3) / 1e12 / world,
                                "of": f"{tf_peak} TF/s {peak_kind} bf16 burst / {tf_sust} sustained"}

    if rank == 0 and not args.profile:
        # roofline of the dominant kernel family, the per-layer tcgen05 GEMMs, measured INSIDE
        # steps: one eager step right after the timed region (same clocks / power state) with
        # a CUDA event in front of every kernel group on the engine stream; the GEMMs' device
        # time over their algorithmic FLOPs, against the SUSTAINED measured bf16 peak
        if not qdir and world == 1:
            t_prof = t_first + args.steps
            eng.profile_step(zcfg.seed, t_prof, zcfg.nu, zcfg.epsilon, zcfg.learning_rate,
                             d_tok[0].data_ptr(), d_gold[0].data_ptr(), Bl)  # plans warm
            # a hot lead-in of captured steps queued right in front of the profiled step (no
            # host sync between them), so it runs in the timed region's power / clock state
            # -- a step started from an idle GPU runs ~10% faster under the power cap
            lead = 20
            for i in range(lead):
                one_step(t_prof + 1 + i, d_tok[i % len(d_tok)].data_ptr(), d_gold[i % len(d_gold)].data_ptr())
            fam = eng.profile_step(zcfg.seed, t_prof + 1 + lead, zcfg.nu, zcfg.epsilon, zcfg.learning_rate,
                                   d_tok[0].data_ptr(), d_gold[0].data_ptr(), Bl)
        else:
            fam = None
        d, Lr, Mr = mcfg.dim, mcfg.n_layers, 2 * Bl * (T - 1)  # rows the forward computes
        gemm_fl = 2.0 * Mr * d * d * (3 * Lr + (1 + 4 + 4) * (Lr - 1))  # qkv x L; out/up/down x (L-1)
        with ClockSampler(local) as gclk:
            g, lay_ms, iso = layer_gemms(eng, Bl)
        if fam is not None:
            gemm_ms = fam["qkv"] + fam["attn_out"] + fam["ff_up"] + fam["ff_down"]
            achieved = gemm_fl / (gemm_ms * 1e-3) / 1e12
            prof_total = sum(fam.values())
        else:
            achieved = iso
        line["roofline"] = {"bound": "tensor", "achieved": achieved, "peak": tf_sust, "unit": "TFLOP/s",
                            "frac": achieved / tf_sust, "traffic": ncu_traffic(args.model),
                            "kernel": "k_gemm (tcgen05 kind::f16, layer GEMMs qkv+attn_out+ff_up+ff_down)",
                            "peak_kind": f"{peak_kind} bf16 sustained (MEASURED_PEAKS.json): GEMMs timed inside "
                                         f"an eager step right after the timed region",
                            "share_of_step": (gemm_ms / prof_total) if fam is not None else None}
        # DRAM bytes of one launch each of the four layer GEMMs (ncu, layer 1) beside their
        # algorithmic bytes: weights once, A operands once, outputs (RMW for the residual ones)
        line["roofline"]["traffic_scope"] = "one launch each of qkv, attn_out, ff_up, ff_down (ncu --set full)"
        line["roofline"]["algorithmic_bytes"] = (2.0 * 12 * d * d + 2.0 * Mr * 7 * d
                                                 + Mr * d * (2 * 3 + 8 + 2 * 4 + 8))
        if fam is not None:
            line["roofline"]["in_step_ms"] = {k: round(v, 4) for k, v in fam.items()}
            line["roofline"]["in_step_total_ms"] = prof_total
        line["roofline"]["isolated"] = {
            "achieved": iso, "frac_of_sustained": iso / tf_sust, "per_gemm": g, "clocks": gclk.summary(),
            "when": "each layer GEMM alone, 20 back-to-back launches, right after the timed steps"}
        if cold is not None:
            line["roofline"]["burst_check"] = {
                "achieved": cold[2], "peak": tf_peak, "frac": cold[2] / tf_peak,
                "per_gemm_ms": {k: v["ms"] for k, v in cold[0].items()},
                "when": "same isolated launches on the cold GPU before the warm-up (burst clocks)"}

    if not args.no_e2e and not args.profile and world == 1:
        # the public API end to end: run_serving_path (runtime.py:253-359, row a1) on host
        # minibatches -- per step sample_minibatch, the H2D copy of tokens/golds from pinned
        # staging, one fused lozo_step, the D2H read of [L+, L-, c, beta], the U arena copied
        # back for the U/V digests the reference's records carry (FNV on a host thread pool)
        # and the fold at the window boundary.  Timed by wall clock over the step loop plus
        # the final digest wait, evals excluded (train_wall_s semantics).
        from paper_2605_28760_b200.runtime import run_serving_path
        params = M.DeviceParams(mcfg, precision=args.precision, max_batch=B)
        params._engine = eng  # reuse the initialised replica
        state = AdapterState(epsilon=zcfg.epsilon)
        base = t_first + args.steps + 2
        e_first = nu_m * -(-(base + args.warmup + args.steps // 2) // nu_m) - args.steps // 2
        # rank > 8 (config 5): audit the U/V digests of every 50th step -- the full arenas are
        # 3.4 GB per step there and FNV-1a is byte-serial (runtime.run_serving_path digest_every)
        dig_every = 1 if args.rank <= 8 else 50
        kw = dict(eval_every=10 ** 9, params=params, state=state, compute_param_digests=False, final_fold=False,
                  digests=True, digest_every=dig_every)
        run_serving_path(mcfg, task, zcfg, args.warmup, start_step=e_first - args.warmup, **kw)
        torch.cuda.synchronize()
        run = run_serving_path(mcfg, task, zcfg, args.steps, start_step=e_first, **kw)
        torch.cuda.synchronize()
        e2e_s = (run.extra["loop_wall_s"] + run.extra["digest_wait_s"]) / args.steps
        assert all(r.u_digest and r.v_digest for i, r in enumerate(run.trajectory) if i % dig_every == 0)
        v_reads = (1.0 / dig_every) if fact else (1.0 / zcfg.nu)  # V arena copies per step
        line["e2e"] = {"value": 1.0 / e2e_s, "unit": UNIT,
                       "h2d_bytes_per_step": B * T * 4 + 2 * B * 4 + 8,
                       "d2h_bytes_per_step": 32 + 8 * eng.su / dig_every + 8 * eng.sv * v_reads,
                       "digest_every": dig_every,
                       "api": "runtime.run_serving_path (host minibatches, fused lozo_step, U/V digests on the "
                              "host pool" + (f", audited every {dig_every} steps" if dig_every > 1 else "")
                              + ", folds at window boundaries)",
                       "timed_steps": [e_first, e_first + args.steps - 1],
                       "digest_wait_s": run.extra["digest_wait_s"],
                       "phase_ms_last_step": dict(zip(["sample", "score", "update"], eng.last_step_ms()))}

    if not args.no_e2e and not args.profile and world > 1:
        # end to end at N GPUs: every step each rank draws its minibatch on the host (its own
        # direction's in q-direction mode, its slice in exact mode), copies it from pinned
        # memory, runs score -> all-gather -> apply, and reads the gathered coefficients back
        # (the losses the public API returns); wall clock, max over ranks
        import torch.distributed as dist
        h_tok = torch.empty((Bl, T), dtype=torch.int32).pin_memory()
        h_gold = torch.empty((Bl, 1), dtype=torch.int32).pin_memory()
        e_tok = torch.empty((Bl, T), dtype=torch.int32, device="cuda")
        e_gold = torch.empty((Bl, 1), dtype=torch.int32, device="cuda")

        def e2e_step(t):
            if qdir:
                seq, gold = M.sample_minibatch(task, "train", zcfg.seed, t * G + rank, B).sequences()
            else:
                seq, gold = M.sample_minibatch(task, "train", zcfg.seed, t, B).sequences()
                seq, gold = seq[rank * Bl:(rank + 1) * Bl], gold[rank * Bl:(rank + 1) * Bl]
            h_tok.copy_(torch.from_numpy(np.ascontiguousarray(seq, dtype=np.int32)))
            h_gold.copy_(torch.from_numpy(np.ascontiguousarray(gold, dtype=np.int32)))
            e_tok.copy_(h_tok, non_blocking=True)
            e_gold.copy_(h_gold, non_blocking=True)
            one_step(t, e_tok.data_ptr(), e_gold.data_ptr())
            return out4_all.cpu() if qdir else torch.from_numpy(eng.read_out4())

        t_e0 = nsteps + 2
        for t in range(t_e0, t_e0 + args.warmup):
            e2e_step(t)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for t in range(t_e0 + args.warmup, t_e0 + args.warmup + args.steps):
            e2e_step(t)
        torch.cuda.synchronize()
        el = torch.tensor([time.perf_counter() - t0], device="cpu" if same_dev else "cuda")
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e_s = float(el.item()) / args.steps
        line["e2e"] = {"value": G / e2e_s, "unit": UNIT, "h2d_bytes_per_step": Bl * T * 4 + Bl * 4,
                       "d2h_bytes_per_step": (G * 32) if qdir else 32,
                       "api": ("model.sample_minibatch + zo_qdir_score_async / all-gather / zo_qdir_apply_async"
                               if qdir else "model.sample_minibatch + zo_step_score_async / all-gather of NLLs / "
                                            "zo_step_apply_async") + " (host batch per rank, wall clock, max over ranks)"}

    if args.materialising and not args.profile and world == 1:
        # the conventional training loop (baseline_loop.py:122-239) on the same replica: probe
        # written into the weights, one forward per sign, restore, update -- the paper's
        # "official baseline" structure, timed the same way (CUDA events, device inputs)
        eng.fold_async()  # the comparand starts from folded weights (no window mass)
        nb = args.materialising_steps
        bw = min(3, nb)
        rc = False  # cached products: the reference's default mode
        for t in range(bw):
            eng.baseline_step_async(zcfg.seed, t, zcfg.nu, zcfg.epsilon, zcfg.learning_rate, False, rc,
                                    d_tok[t].data_ptr(), d_gold[t].data_ptr(), Bl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t in range(bw, bw + nb):
            eng.baseline_step_async(zcfg.seed, t, zcfg.nu, zcfg.epsilon, zcfg.learning_rate, False, rc,
                                    d_tok[t % nsteps].data_ptr(), d_gold[t % nsteps].data_ptr(), Bl)
        e1.record(stream)
        torch.cuda.synchronize()
        bms = e0.elapsed_time(e1) / nb
        line["materialising_loop"] = {
            "value": 1000.0 / bms, "unit": UNIT, "ms_per_step": bms, "steps": nb,
            "speedup_of_serving_path": (1000.0 / ms_step) / (1000.0 / bms),
            "mode": "cached products (restore = copy of the saved bits)",
            "weight_writes_per_step": 4 * (sum(mcfg.dim * n for n in (3 * mcfg.dim, mcfg.dim, 4 * mcfg.dim))
                                           * mcfg.n_layers + mcfg.vocab * mcfg.dim),
            "what": "baseline_loop.py:122-239 on this GPU: W+=eps*P, score L+, W-=2eps*P, score L-, restore, "
                    "W-=eta*c*P (zo_baseline_step_async, float64 master + 16-bit serving copy)"}

    if rank == 0 and not args.no_cpu_baseline and not args.profile:
        from oracle.cpu_bench import estimate_step, host_threads, reference_config1
        step_s, desc, _ = estimate_step(mcfg.dim, mcfg.n_layers, mcfg.n_heads, mcfg.vocab, B, T,
                                        n_examples=4 if mcfg.dim >= 4096 else B)
        line["cpu_baseline"] = {"value": 1.0 / step_s, "unit": UNIT, "cores": host_threads(), "kind": "port",
                                "sample": desc + " (extrapolated: the 13B step does not fit a bounded CPU run)"}
        if world == 1:
            # BASELINE config 1 measured in whole steps on both sides, no extrapolation: the
            # reference's own lozo_step on the host cores and the same step on this B200
            ref1 = reference_config1(steps=2, warmup=0)
            g1 = config1_gpu(args, M, ZoEngine, torch, stream)
            if ref1 is not None:
                line["cpu_baseline"]["config1_reference"] = {
                    "value": ref1[0], "unit": UNIT, "cores": host_threads(), "kind": "reference",
                    "sample": ref1[1]}
            line["config1_b200"] = g1
            if ref1 is not None:
                line["config1_b200"]["speedup_vs_reference"] = g1["value"] / ref1[0]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
