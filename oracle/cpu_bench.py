"""oracle/cpu_bench.py -- TEST INFRASTRUCTURE ONLY: the CPU baseline leg of bench.py.

Times the oracle port (oracle/reference.py, float64 numpy, the reference's
algorithm: compose-then-matmul, model.py:157-199 + adapter.py:200-234) on a
BOUNDED sample of one LoZO step and extrapolates to the whole step:

  sample  = one decoder block of the paired (+eps, -eps) scoring forward for
            `n_examples` sequences of T tokens, including the per-call dense
            composition W0 + A V^T +- eps U V^T of the block's four matrices
            (the reference materialises these every scorer call);
  step    = n_layers * (composition + (B / n_examples) * forward)
            + the LM-head rows and option NLLs of both probes (timed once)
            + direction sampling for every matrix (timed, C oracle sampler).

Never used as the product path; bench.py reports it as ``cpu_baseline``
(kind "port") and as the ``--impl reference`` arm.
"""
from __future__ import annotations

import math
import os
import time

import numpy as np

from . import reference as R


def _block_forward(x, w, H):
    B, T, d = x.shape
    dh = d // H
    mask = np.triu(np.ones((T, T), dtype=bool), k=1)
    h = R._ln(x, 1.0, 0.0)
    qkv = h @ w["qkv"]
    q, k, v = (qkv[..., j * d:(j + 1) * d].reshape(B, T, H, dh).transpose(0, 2, 1, 3) for j in range(3))
    s = q @ k.transpose(0, 1, 3, 2) / math.sqrt(dh)
    s = np.where(mask, -np.inf, s)
    s = s - s.max(axis=-1, keepdims=True)
    a = np.exp(s)
    a = a / a.sum(axis=-1, keepdims=True)
    ctx = (a @ v).transpose(0, 2, 1, 3).reshape(B, T, d)
    x = x + ctx @ w["attn_out"]
    h = R._ln(x, 1.0, 0.0)
    return x + R._gelu(h @ w["ff_up"]) @ w["ff_down"]


class BlockSample:
    def __init__(self, dim: int, n_heads: int, vocab: int, T: int, n_examples: int, rank: int = 2, seed: int = 0):
        rng = np.random.default_rng(seed)
        d = dim
        self.H, self.T, self.n = n_heads, T, n_examples
        self.shapes = {"qkv": (d, 3 * d), "attn_out": (d, d), "ff_up": (d, 4 * d), "ff_down": (4 * d, d)}
        self.W = {k: 0.02 * rng.standard_normal(s) for k, s in self.shapes.items()}
        self.A = {k: 1e-4 * rng.standard_normal((s[0], rank)) for k, s in self.shapes.items()}
        self.U = {k: rng.standard_normal((s[0], rank)) for k, s in self.shapes.items()}
        self.V = {k: rng.standard_normal((s[1], rank)) for k, s in self.shapes.items()}
        self.x = rng.standard_normal((n_examples, T, d))
        self.head_x = rng.standard_normal((n_examples, d))
        self.E = 0.02 * rng.standard_normal((vocab, d))

    def run(self, eps: float = 1e-3) -> tuple[float, float]:
        """(composition seconds, forward seconds) for the sample, both probe signs.
        Composition is per scorer call (independent of batch size), the forward
        scales with the number of sequences."""
        tc = tf = 0.0
        for sign in (+1, -1):
            t0 = time.perf_counter()
            w = {k: R.compose(self.W[k], self.A[k], self.V[k], self.U[k], sign, eps) for k in self.W}
            t1 = time.perf_counter()
            _block_forward(self.x, w, self.H)
            t2 = time.perf_counter()
            tc += t1 - t0
            tf += t2 - t1
        return tc, tf

    def run_head(self) -> float:
        t0 = time.perf_counter()
        for _ in (+1, -1):
            row = self.head_x @ self.E.T
            m = row.max(axis=-1)
            _ = m + np.log(np.exp(row - m[:, None]).sum(axis=-1))
        return time.perf_counter() - t0


def sampler_seconds(shapes: dict, rank: int) -> float:
    t0 = time.perf_counter()
    for lid, (m, n) in shapes.items():
        R.gaussian(42, 7, lid, R.ROLE_U, m, rank)
    return time.perf_counter() - t0


def estimate_step(dim, n_layers, n_heads, vocab, B, T, n_examples, rank=2, reps=1):
    """(seconds per full step estimated, sample description, sample seconds)."""
    bs = BlockSample(dim, n_heads, vocab, T, n_examples, rank)
    bs.run()  # warm (page in, BLAS threads)
    tc, tf = min((bs.run() for _ in range(reps)), key=lambda p: p[0] + p[1])
    t_block = tc + tf * (B / n_examples)
    t_head = bs.run_head() * (B / n_examples)
    shapes = {"embed": (vocab, dim)}
    for i in range(n_layers):
        shapes.update({f"blk{i}.qkv": (dim, 3 * dim), f"blk{i}.attn_out": (dim, dim),
                       f"blk{i}.ff_up": (dim, 4 * dim), f"blk{i}.ff_down": (4 * dim, dim)})
    t_samp = sampler_seconds(dict(list(shapes.items())[:5]), rank) * len(shapes) / 5
    step = n_layers * t_block + t_head + t_samp
    desc = (f"oracle float64 port: 1 of {n_layers} decoder blocks, paired +-eps forward of {n_examples}/{B} "
            f"sequences x T={T} ({tf:.3f} s, scaled x{B // n_examples}) + the block's per-call W0+AV^T+-eps UV^T "
            f"composition ({tc:.3f} s); x{n_layers} blocks + LM-head rows + direction sampling")
    return step, desc, t_block


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_config1(steps: int = 2, warmup: int = 1):
    """The UNMODIFIED reference (oracle/_ref/zoserve, staged by oracle/stage_ref.sh) timed on
    BASELINE config 1 -- OPT-125m dims, V = 50272, B = 16, T = 64, r = 2, nu = 50, lr 1e-7,
    real64: whole ``zoserve.zo_engine.lozo_step`` calls (directions, both composed float64
    forwards, coefficient, update), the state carried across steps exactly as
    run_serving_path does (runtime.py:303-330).  Returns (steps/s, description) or None when
    the reference was not staged."""
    import sys
    ref = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
    if not os.path.isfile(os.path.join(ref, "zoserve", "zo_engine.py")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from zoserve.adapter import AdapterState
    from zoserve.model import ModelConfig, TaskConfig, generate_task, init_params, sample_minibatch
    from zoserve.zo_engine import ZoConfig, lozo_step
    mcfg = ModelConfig(vocab=50272, dim=768, n_layers=12, n_heads=12, prompt_len=63, init_seed=7, init_scale=0.02)
    task = generate_task(TaskConfig(seed=11, vocab=50272, prompt_len=63, train_size=1000, dev_size=64, val_size=64))
    zcfg = ZoConfig(seed=42, epsilon=1e-3, learning_rate=1e-7, rank=2, nu=50, batch_size=16)
    params = init_params(mcfg)
    state = AdapterState(epsilon=zcfg.epsilon)
    times = []
    for t in range(warmup + steps):
        batch = sample_minibatch(task, "train", zcfg.seed, t, zcfg.batch_size)
        t0 = time.perf_counter()
        rec = lozo_step(params, mcfg, state, zcfg, t, batch, "real64")
        if t >= warmup:
            times.append(time.perf_counter() - t0)
    s = float(np.mean(times))
    desc = (f"the reference itself (zoserve.zo_engine.lozo_step, real64, oracle/_ref) at BASELINE config 1 "
            f"(OPT-125m dims, B=16, T=64): {steps} whole steps timed after {warmup} warm-up, "
            f"{s:.2f} s/step; last step L+ = {rec.loss_plus:.6f}")
    return 1.0 / s, desc


def reference_layers(dim: int, n_layers: int, n_heads: int, vocab: int, B: int = 16, T: int = 64,
                     layer_counts=(1, 2)):
    """The UNMODIFIED reference (oracle/_ref/zoserve) at a large model's own dims, bounded by
    depth: one whole ``lozo_step`` (real64: directions, both composed float64 forwards,
    coefficient, update) of the same model with 1 and with 2 decoder blocks; the block cost is
    the difference, the rest (embedding, LM head, loss, sampling) the remainder, and the full
    model's step = remainder + n_layers x block (every block has the same shape).  Returns
    (steps/s, description) or None when the reference was not staged."""
    import sys
    ref = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
    if not os.path.isfile(os.path.join(ref, "zoserve", "zo_engine.py")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from zoserve.adapter import AdapterState
    from zoserve.model import ModelConfig, TaskConfig, generate_task, init_params, sample_minibatch
    from zoserve.zo_engine import ZoConfig, lozo_step
    task = generate_task(TaskConfig(seed=11, vocab=vocab, prompt_len=T - 1, train_size=64, dev_size=2, val_size=2))
    zcfg = ZoConfig(seed=42, epsilon=1e-3, learning_rate=1e-7, rank=2, nu=50, batch_size=B)
    secs = {}
    for L in layer_counts:
        mcfg = ModelConfig(vocab=vocab, dim=dim, n_layers=L, n_heads=n_heads, prompt_len=T - 1, init_seed=7,
                           init_scale=0.02)
        params = init_params(mcfg)
        state = AdapterState(epsilon=zcfg.epsilon)
        batch = sample_minibatch(task, "train", zcfg.seed, 0, B)
        t0 = time.perf_counter()
        lozo_step(params, mcfg, state, zcfg, 0, batch, "real64")
        secs[L] = time.perf_counter() - t0
        del params
    l1, l2 = layer_counts[0], layer_counts[-1]
    block = (secs[l2] - secs[l1]) / (l2 - l1)
    if block <= 0:  # timing noise on a tiny model: split the deeper step evenly
        block = secs[l2] / (l2 + 1)
    rest = max(secs[l1] - l1 * block, 0.0)
    step = rest + n_layers * block
    desc = (f"the reference itself (zoserve.zo_engine.lozo_step, real64, oracle/_ref) at the model's own dims "
            f"(d={dim}, H={n_heads}, V={vocab}, B={B}, T={T}) with {l1} and {l2} decoder blocks: "
            f"{secs[l1]:.1f} s / {secs[l2]:.1f} s per whole step -> {block:.1f} s per block + {rest:.1f} s "
            f"embedding/LM head/loss/sampling; {n_layers} blocks -> {step:.0f} s per step "
            f"(depth-extrapolated: the full model's step does not fit a bounded CPU run)")
    return 1.0 / step, desc
