"""Two-point zeroth-order estimators of ``zoserve.zo_engine`` (zo_engine.py:46-65)
on the B200 engine.

``lozo_step`` / ``factorized_step`` keep the reference signatures and return
the same ``ZoStepRecord``; with the default scorer the whole step (directions,
paired scoring, coefficient, update) runs on the device in one call
(``zo_step``).  A caller-supplied ``scorer`` keeps the reference's seam
(zo_engine.py:298-346): directions are still sampled on the device and the
update is applied there with the coefficient the scorer produced.
"""
from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass

import numpy as np

from .adapter import AdapterState, LoraSlot
from .engine import V as SLOT_V, U as SLOT_U
from .errors import ConfigError, InputError
from .model import Minibatch, ModelConfig, as_device_params, matrix_ids, vector_ids
from .engine import resolve_precision
from .numerics import (FNV_OFFSET_BASIS, Role, StreamKey, canonical_mean, digest_array, digest_hex, digest_text,
                       gaussian_vector, sample_gaussian)

__all__ = ["SCOPES", "ESTIMATORS", "ZoConfig", "ZoStepRecord", "write_trajectory", "read_trajectory",
           "lozo_direction", "factorized_direction", "StepDirections", "step_directions",
           "estimate_coefficient", "make_step_record", "lozo_step", "factorized_step", "dense_mezo_step"]

SCOPES = ("lora_only", "full")
ESTIMATORS = ("dense_mezo", "lozo_lazy", "factorized_sqrt_r")


@dataclass(frozen=True)
class ZoConfig:
    """zo_engine.py:71-98."""
    seed: int = 42
    epsilon: float = 1e-3
    learning_rate: float = 1e-3
    rank: int = 2
    nu: int = 50
    divide_by_r: bool = False
    scope: str = "lora_only"
    estimator: str = "lozo_lazy"
    batch_size: int = 16

    def __post_init__(self) -> None:
        if self.epsilon <= 0:
            raise ConfigError("epsilon must be > 0")
        if self.nu < 1 or self.rank < 1:
            raise ConfigError("nu and rank must be >= 1")
        if self.learning_rate < 0:
            raise ConfigError("learning_rate must be >= 0")
        if self.scope not in SCOPES:
            raise ConfigError(f"scope must be one of {SCOPES}, got {self.scope!r}")
        if self.estimator not in ESTIMATORS:
            raise ConfigError(f"estimator must be one of {ESTIMATORS}, got {self.estimator!r}")
        if self.batch_size < 1:
            raise ConfigError("batch_size must be >= 1")

    def digest(self) -> str:
        return digest_hex(digest_text(json.dumps(asdict(self), sort_keys=True)))


@dataclass
class ZoStepRecord:
    """zo_engine.py:101-127."""
    step: int
    loss_plus: float
    loss_minus: float
    coefficient: float
    beta: float
    seed: int
    u_digest: str
    v_digest: str
    minibatch_id: str

    def to_dict(self) -> dict:
        d = {"record": "step"}
        d.update(asdict(self))
        return d

    @classmethod
    def from_dict(cls, d: dict) -> "ZoStepRecord":
        return cls(**{k: d[k] for k in ("step", "loss_plus", "loss_minus", "coefficient", "beta", "seed",
                                        "u_digest", "v_digest", "minibatch_id")})


def write_trajectory(path: str, header: dict, records: list[ZoStepRecord], final: dict | None = None) -> None:
    """JSON-lines trajectory, the reference's wire format (zo_engine.py:130-144)."""
    with open(path, "w") as f:
        head = {"record": "header", "schema": 1}
        head.update(header)
        f.write(json.dumps(head, sort_keys=True) + "\n")
        for r in records:
            f.write(json.dumps(r.to_dict(), sort_keys=True) + "\n")
        if final is not None:
            tail = {"record": "final"}
            tail.update(final)
            f.write(json.dumps(tail, sort_keys=True) + "\n")


def read_trajectory(path: str):
    with open(path) as f:
        lines = [json.loads(l) for l in f if l.strip()]
    if not lines or lines[0].get("record") != "header":
        raise InputError(f"{path}: not a trajectory file (missing header line)")
    recs = [ZoStepRecord.from_dict(d) for d in lines[1:] if d.get("record") == "step"]
    finals = [d for d in lines[1:] if d.get("record") == "final"]
    return lines[0], recs, finals[-1] if finals else None


# --------------------------------------------------------------------------- directions
def lozo_direction(seed: int, step: int, layer_id: str, m: int, n: int, rank: int, nu: int):
    """(U, V) of one matrix (zo_engine.py:163-178), sampled on the device."""
    if rank > min(m, n):
        raise ConfigError(f"rank {rank} exceeds min dim of {m}x{n} matrix")
    if rank < 1 or nu < 1:
        raise ConfigError("rank and nu must be >= 1")
    v = sample_gaussian(StreamKey(seed, (step // nu) * nu, layer_id, Role.V), n, rank)
    u = sample_gaussian(StreamKey(seed, step, layer_id, Role.U), m, rank)
    return u, v


def factorized_direction(seed: int, step: int, layer_id: str, m: int, n: int, rank: int) -> LoraSlot:
    """U V^T / sqrt(r) (zo_engine.py:181-191)."""
    if rank < 1:
        raise ConfigError("rank must be >= 1")
    u = sample_gaussian(StreamKey(seed, step, layer_id, Role.U), m, rank)
    v = sample_gaussian(StreamKey(seed, step, layer_id, Role.V), n, rank)
    return LoraSlot(u, v, 1.0 / math.sqrt(rank))


@dataclass
class StepDirections:
    matrices: dict
    vectors: dict
    u_digest: str
    v_digest: str
    scale: float = 1.0


def _engine_for(params, mcfg: ModelConfig, zcfg: ZoConfig, batch: Minibatch):
    if zcfg.estimator == "dense_mezo":
        raise ConfigError("dense_mezo has no B200 engine path (no compact update factor)")
    dp = as_device_params(params, mcfg)
    eng = dp.bind(zcfg.rank, zcfg.estimator, zcfg.batch_size, batch.option_array().shape[1], zcfg.scope)
    return dp, eng


def _chain(h: int, layer_id: str, a: np.ndarray) -> int:
    return digest_array(a, digest_text(layer_id, h))


def _dense_direction(seed: int, step: int, layer_id: str, shape) -> np.ndarray:
    """zo_engine.py:193-198: Role.DENSE_Z stream of one parameter."""
    key = StreamKey(seed, step, layer_id, Role.DENSE_Z)
    if len(shape) == 1:
        return gaussian_vector(key, shape[0])
    return sample_gaussian(key, shape[0], shape[1])


def step_directions(params, zcfg: ZoConfig, step: int, mcfg: ModelConfig | None = None) -> StepDirections:
    """Every direction of one step plus chained digests (zo_engine.py:224-261).

    Pure, like the reference: each stream is drawn by the device sampler into a
    fresh host array (``zo_sample_stream``); the engine's U/V/A arenas, its
    window and its float64 masters are not touched, so calling this mid-run
    leaves the trajectory unchanged.  ``mcfg`` is accepted for symmetry with the
    other entry points and unused (shapes come from ``params``)."""
    def shape_of(lid):
        return params.shape_of(lid) if hasattr(params, "shape_of") else np.shape(params[lid])

    mids, vids = matrix_ids(params), vector_ids(params)
    hu = hv = FNV_OFFSET_BASIS
    matrices: dict = {}
    vectors: dict = {}
    scale = 1.0
    if zcfg.estimator == "dense_mezo":
        for lid in mids:
            z = _dense_direction(zcfg.seed, step, lid, shape_of(lid))
            matrices[lid] = z
            hu = _chain(hu, lid, z)
        for lid in vids:
            z = _dense_direction(zcfg.seed, step, lid, shape_of(lid))
            vectors[lid] = z
            hu = _chain(hu, lid, z)
        return StepDirections(matrices, vectors, digest_hex(hu), digest_hex(hv))
    for lid in mids:
        m, n = shape_of(lid)
        if zcfg.estimator == "lozo_lazy":
            u, v = lozo_direction(zcfg.seed, step, lid, m, n, zcfg.rank, zcfg.nu)
        else:
            slot = factorized_direction(zcfg.seed, step, lid, m, n, zcfg.rank)
            u, v, scale = slot.A, slot.B, slot.scale
        matrices[lid] = (u, v)
        hu = _chain(hu, lid, u)
        hv = _chain(hv, lid, v)
    if zcfg.scope == "full":
        for lid in vids:
            z = _dense_direction(zcfg.seed, step, lid, shape_of(lid))
            vectors[lid] = z
            hu = _chain(hu, lid, z)
    return StepDirections(matrices, vectors, digest_hex(hu), digest_hex(hv), scale)


# --------------------------------------------------------------------------- coefficient
def estimate_coefficient(scorer, state: AdapterState, epsilon: float, batch, on_sign=None):
    """c = (L+ - L-) / (2 eps) from exactly two scorer calls at sign +1 then -1,
    sign restored to 0 in all cases (zo_engine.py:298-332)."""
    if epsilon <= 0:
        raise ConfigError("epsilon must be > 0")
    if not state._probe_on and not any(e.perturb_slot is not None for e in state._host_entries.values()):
        raise ConfigError("no active perturbation slot installed")
    try:
        state.set_sign(+1)
        if on_sign is not None:
            on_sign(+1)
        lp = float(scorer(batch))
        state.set_sign(-1)
        if on_sign is not None:
            on_sign(-1)
        lm = float(scorer(batch))
    finally:
        state.set_sign(0)
        if on_sign is not None:
            on_sign(0)
    return (lp - lm) / (2.0 * epsilon), lp, lm


def make_step_record(zcfg: ZoConfig, step: int, lp: float, lm: float, beta: float, u_digest: str, v_digest: str,
                     batch) -> ZoStepRecord:
    """Coefficient recomputed from the recorded losses (zo_engine.py:349-365)."""
    return ZoStepRecord(step, lp, lm, (lp - lm) / (2.0 * zcfg.epsilon), beta, zcfg.seed, u_digest, v_digest,
                        batch.batch_id)


class _DigestCache:
    """Per-state V digest cache (V only changes at window starts)."""

    def __init__(self):
        self.key = None
        self.value = None


def _digests(state: AdapterState, eng, zcfg: ZoConfig, step: int, mode: str):
    if mode == "off":
        return "", ""
    u = digest_hex(eng.digest(SLOT_U))
    wkey = (step // zcfg.nu) * zcfg.nu if zcfg.estimator == "lozo_lazy" else step
    cache = getattr(state, "_vdig", None)
    if cache is None:
        cache = state._vdig = _DigestCache()
    if cache.key != wkey:
        cache.key, cache.value = wkey, digest_hex(eng.digest(SLOT_V))
    return u, cache.value


class GpuPairScorer:
    """The reference's ``scorer`` protocol (zo_engine.py:340-346) on the engine:
    the +1 call scores both probes in one fused launch and caches L-; the -1
    call returns the cached value only if neither the minibatch nor the adapter
    changed in between (batch id + ``AdapterState.version``).  Pure: writes no
    weights."""

    def __init__(self, params, mcfg: ModelConfig, state: AdapterState):
        self.dp = as_device_params(params, mcfg)
        self.mcfg = mcfg
        self.state = state
        self._cached = None

    def __call__(self, batch: Minibatch) -> float:
        eng = self.dp.engine
        sign = self.state.perturb_sign
        key = (batch.batch_id, self.state.version)
        if sign == -1 and self._cached is not None and self._cached[0] == key:
            v = self._cached[1]
            self._cached = None
            return v
        self._cached = None
        tokens, gold = batch.sequences()
        self.state._sync_to_engine(eng)
        if sign == 0 or not self.state._probe_on:
            eng.prepare_probe(self.state.epsilon, 1)
            return canonical_mean(eng.score(tokens, gold, nsign=1)[0])
        eng.prepare_probe(self.state.epsilon, 0)
        nll = eng.score(tokens, np.stack([gold, gold]), nsign=2)  # one gold block per probe half
        lp, lm = canonical_mean(nll[0]), canonical_mean(nll[1])
        if sign == 1:
            self._cached = (key, lm)
            return lp
        return lm


# --------------------------------------------------------------------------- steps
def lozo_step(params, mcfg: ModelConfig, state: AdapterState, zcfg: ZoConfig, step: int, batch: Minibatch,
              precision: str = "real64", scorer=None, digests: str = "sync") -> ZoStepRecord:
    """One lazy low-rank step (zo_engine.py:368-417): V keyed by the window
    start, U by the step, paired probes, c, A += -(eta*c_used)*U.  Dense
    weights are untouched; folds are the caller's policy."""
    if zcfg.estimator != "lozo_lazy":
        raise ConfigError("lozo_step needs estimator='lozo_lazy'")
    dp, eng = _engine_for(params, mcfg, zcfg, batch)
    state._bind(eng)
    state._sync_to_engine(eng)
    tokens, gold = batch.sequences()
    if scorer is None:
        out = eng.step(zcfg.seed, step, zcfg.nu, zcfg.epsilon, zcfg.learning_rate, zcfg.divide_by_r, tokens, gold)
        lp, lm, beta = float(out[0]), float(out[1]), float(out[3])
        if zcfg.scope == "full":
            dp.invalidate()
    else:
        window = (step // zcfg.nu) * zcfg.nu
        if getattr(state, "_window", None) != window:
            eng.sample_v(zcfg.seed, step, zcfg.nu)  # folds unfolded window mass first
            dp.invalidate()
            state._window = window
        eng.sample_u(zcfg.seed, step)
        state._probe_on = True
        state._touch()  # new probe U on the device
        try:
            c, lp, lm = estimate_coefficient(scorer, state, zcfg.epsilon, batch)
        finally:
            state.clear_probes()
        c_used = c / zcfg.rank if zcfg.divide_by_r else c
        beta = -(zcfg.learning_rate * c_used)
        eng.set_coefficient(np.array([lp, lm, c, beta]))
        eng.update_u()
        eng.update_vectors(zcfg.learning_rate)  # full scope: VectorProbe.update (zo_engine.py:412-416)
        dp.invalidate()
    state._touch()  # the window A moved
    if zcfg.scope == "full":
        dp.sync_host(matrices=False)  # VectorProbe.update mutated the caller's 1-D params
    ud, vd = _digests(state, eng, zcfg, step, digests)
    return make_step_record(zcfg, step, lp, lm, beta, ud, vd, batch)


def factorized_step(params, mcfg: ModelConfig, state: AdapterState, zcfg: ZoConfig, step: int, batch: Minibatch,
                    precision: str = "real64", scorer=None, digests: str = "sync") -> ZoStepRecord:
    """sqrt(r)-normalised factorized step (zo_engine.py:420-453): probe U V^T/sqrt(r),
    then W += (-(eta*c)/sqrt(r)) U V^T into the float64 master (+16-bit shadow)."""
    if zcfg.estimator != "factorized_sqrt_r":
        raise ConfigError("factorized_step needs estimator='factorized_sqrt_r'")
    if scorer is not None:
        raise ConfigError("factorized_step on the B200 engine uses its fused scorer")
    dp, eng = _engine_for(params, mcfg, zcfg, batch)
    state._bind(eng)
    tokens, gold = batch.sequences()
    out = eng.step(zcfg.seed, step, 1, zcfg.epsilon, zcfg.learning_rate, False, tokens, gold)
    dp.invalidate()
    dp.sync_host()  # the dense update wrote every matrix (zo_engine.py:449-450)
    state._touch()
    ud, vd = _digests(state, eng, zcfg, step, digests)
    return make_step_record(zcfg, step, float(out[0]), float(out[1]), -(zcfg.learning_rate * float(out[2])),
                            ud, vd, batch)


def dense_mezo_step(params, mcfg: ModelConfig, zcfg: ZoConfig, step: int, batch: Minibatch,
                    precision: str = "real64", scorer=None, digests: str = "sync") -> ZoStepRecord:
    """One dense two-point step (zo_engine.py:476-493): z ~ N(0,1) for every parameter
    (Role.DENSE_Z, scope ignored), in-place probing of the device weights with bit-exact
    restore (_dense_probe_coefficient, 456-473), then theta <- theta - eta*c*z -- the device
    materialising loop's cached mode (baseline_loop.run_baseline), float64 exact given c.
    A custom ``scorer`` cannot see device-resident probed weights and is rejected."""
    if zcfg.estimator != "dense_mezo":
        raise ConfigError("dense_mezo_step needs estimator='dense_mezo'")
    if scorer is not None:
        raise ConfigError("dense_mezo_step scores the device weights; a host scorer cannot see them")
    resolve_precision(precision)
    dp = as_device_params(params, mcfg)
    eng = dp.bind(zcfg.rank, "dense_mezo", batch.prompts.shape[0], batch.option_array().shape[1], zcfg.scope)
    tokens, gold = batch.sequences()
    eng.baseline_directions(zcfg.seed, step, zcfg.nu)
    eng.baseline_pass(0, zcfg.epsilon, False)
    lp = canonical_mean(eng.score(tokens, gold, nsign=1)[0])
    eng.baseline_pass(1, zcfg.epsilon, False)
    lm = canonical_mean(eng.score(tokens, gold, nsign=1)[0])
    eng.baseline_pass(2, zcfg.epsilon, False)
    c = (lp - lm) / (2.0 * zcfg.epsilon)
    beta = -(zcfg.learning_rate * c)
    eng.set_coefficient([lp, lm, c, beta])
    eng.baseline_update(zcfg.learning_rate, False)
    dp.invalidate()
    dp.sync_host()
    u = digest_hex(eng.digest(SLOT_U)) if digests != "off" else ""
    v = digest_hex(eng.digest(SLOT_V)) if digests != "off" else ""
    return make_step_record(zcfg, step, lp, lm, beta, u, v, batch)
