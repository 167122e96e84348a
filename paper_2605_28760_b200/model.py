"""Model / task surface of ``zoserve.model`` (model.py:34-53) on the B200 engine.

Configs, the synthetic marker task and minibatch sampling are host data prep
(numpy streams, exactly as the reference).  Parameters live on the device:
``init_params`` returns a :class:`DeviceParams` mapping whose float64 master is
regenerated on the GPU from the Role.INIT streams (bit-exact), and
``forward_score`` / ``eval_accuracy`` / ``evaluate_split`` run the tcgen05
scorer.
"""
from __future__ import annotations

import json
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np

from .engine import ZoEngine, resolve_precision, vector_shapes
from .errors import ConfigError, DimensionError, InputError
from .numerics import (Role, StreamKey, canonical_mean, digest_array, digest_bytes, digest_hex, digest_text,
                       sample_indices)

__all__ = [
    "ModelConfig", "init_params", "params_digest", "matrix_ids", "vector_ids", "pos_encoding",
    "forward_score", "forward_nll", "eval_accuracy", "TaskConfig", "TaskData", "generate_task", "save_task",
    "load_task", "Minibatch", "sample_minibatch", "EvalPoint", "evaluate_split", "DeviceParams",
]


@dataclass(frozen=True)
class ModelConfig:
    """Decoder shape (model.py:62-81): pre-LN, packed qkv, GELU-tanh FFN (4d),
    sinusoidal positions, no biases, tied head.

    ``arch="opt"`` (no reference counterpart) is the OPT
    family's decoder that real checkpoints load into (opt_io.py): ReLU FFN,
    learned positions ``pos_embed`` [max_positions + 2, dim] read at offset 2,
    biases on qkv / attn_out / ff_up / ff_down, pre-LN, tied head.  Its extra 2-D
    param joins the LoRA scope like every other matrix (matrix_ids rule,
    model.py:120-121); the biases are 1-D (full scope)."""
    vocab: int = 64
    dim: int = 32
    n_layers: int = 2
    n_heads: int = 2
    prompt_len: int = 16
    init_seed: int = 7
    init_scale: float = 0.08
    arch: str = "zoserve"
    max_positions: int = 2048

    def __post_init__(self) -> None:
        if self.arch not in ("zoserve", "opt"):
            raise ConfigError(f"arch must be 'zoserve' or 'opt', got {self.arch!r}")
        if self.arch == "opt" and self.max_positions <= self.prompt_len:
            raise ConfigError("max_positions must exceed prompt_len")
        if self.dim % self.n_heads != 0:
            raise ConfigError(f"dim {self.dim} not divisible by n_heads {self.n_heads}")
        if self.vocab < 8:
            raise ConfigError("vocab must leave room for control tokens (>= 8)")
        if min(self.dim, self.n_layers, self.n_heads, self.prompt_len) < 1:
            raise ConfigError("model dimensions must be positive")

    def digest(self) -> str:
        d = dict(self.__dict__)
        if d["arch"] == "zoserve":  # the reference's ModelConfig fields only (model.py:62-81)
            d.pop("arch")
            d.pop("max_positions")
        return digest_hex(digest_text(json.dumps(d, sort_keys=True)))


def matrix_shapes(cfg: ModelConfig) -> dict[str, tuple[int, int]]:
    d = cfg.dim
    out = {"embed": (cfg.vocab, d)}
    if cfg.arch == "opt":
        out["pos_embed"] = (cfg.max_positions + 2, d)
    for i in range(cfg.n_layers):
        out[f"blk{i}.qkv"] = (d, 3 * d)
        out[f"blk{i}.attn_out"] = (d, d)
        out[f"blk{i}.ff_up"] = (d, 4 * d)
        out[f"blk{i}.ff_down"] = (4 * d, d)
    return out


def _vector_defaults(cfg: ModelConfig) -> dict[str, np.ndarray]:
    """LN scale 1 / shift 0 (model.py:100-107); OPT biases 0."""
    return {k: (np.ones(n) if k.endswith(".scale") else np.zeros(n))
            for k, n in vector_shapes(cfg.n_layers, cfg.dim, cfg.arch).items()}


class DeviceParams(Mapping):
    """``params`` dict of the reference, backed by a device-resident engine.

    Matrices are read back (float64, reference (in, out) layout) on access and
    cached until the next device mutation (fold / dense update).  The engine is
    created on first use with the ZoConfig it must serve (rank, estimator) --
    the reference's params dict is likewise untyped until a step uses it.
    """

    def __init__(self, cfg: ModelConfig, host: Mapping[str, np.ndarray] | None = None, precision: str = "fp16",
                 max_batch: int = 16, device: int = 0):
        self.cfg = cfg
        self._shapes = matrix_shapes(cfg)
        self._vectors = _vector_defaults(cfg)
        self._host = host  # optional initial host weights (uploaded at bind time)
        if host is not None:
            for k, v in host.items():
                if np.ndim(v) == 1:
                    self._vectors[k] = np.asarray(v, dtype=np.float64).copy()
        self._engine: ZoEngine | None = None
        self._cache: dict[str, np.ndarray] = {}
        self.precision = resolve_precision(precision)
        self.max_batch = max_batch
        self.device = device
        self._opt_len = 1
        self._mirror = None  # caller's host dict (as_device_params), written back by sync_host

    # Mapping protocol
    def __getitem__(self, lid: str) -> np.ndarray:
        if lid in self._vectors:
            if self._engine is not None and (self._engine.scope == "full"
                                             or self._engine.estimator == "dense_mezo"):
                # full scope: the device updates the 1-D params every step
                if lid not in self._cache:
                    self._cache[lid] = self._engine.download_vector(lid)
                return self._cache[lid]
            return self._vectors[lid]
        if lid not in self._shapes:
            raise KeyError(lid)
        if lid not in self._cache:
            self._cache[lid] = self.engine.download(lid)
        return self._cache[lid]

    def __iter__(self):
        return iter(list(self._shapes) + list(self._vectors))

    def __len__(self) -> int:
        return len(self._shapes) + len(self._vectors)

    def shape_of(self, lid: str) -> tuple[int, ...]:
        return self._shapes[lid] if lid in self._shapes else self._vectors[lid].shape

    def invalidate(self) -> None:
        self._cache.clear()

    @property
    def bound(self) -> bool:
        return self._engine is not None

    @property
    def engine(self) -> ZoEngine:
        if self._engine is None:
            self.bind()
        return self._engine

    def bind(self, rank: int = 2, estimator: str = "lozo_lazy", max_batch: int | None = None,
             opt_len: int = 1, scope: str = "lora_only") -> ZoEngine:
        """Create (or check) the device engine for this parameter set."""
        mb = max(max_batch or 0, self.max_batch)
        if self._engine is not None and self._engine.scope != scope:
            # the scope is fixed per engine (full scope adds the 1-D probe arenas): move the
            # current parameters into a fresh engine of the requested scope
            old = self._engine
            host = {lid: old.download(lid) for lid in old.lids}
            if old.scope == "full" or old.estimator == "dense_mezo":
                for vid in old.vids:
                    self._vectors[vid] = old.download_vector(vid)
            old.close()
            self._engine = None
            self._cache.clear()
            self._host = host
        if self._engine is not None:
            e = self._engine
            if (e.rank, e.estimator, e.opt_len) != (rank, estimator, opt_len) or e.max_batch < mb:
                if e.rank == rank and e.estimator == estimator and e.opt_len == opt_len:
                    pass  # smaller batches fit
                else:
                    raise ConfigError(
                        f"params are bound to an engine with rank={e.rank}, estimator={e.estimator}, "
                        f"opt_len={e.opt_len}; requested rank={rank}, estimator={estimator}, opt_len={opt_len}")
            return e
        c = self.cfg
        e = ZoEngine(c.vocab, c.dim, c.n_layers, c.n_heads, c.prompt_len, opt_len=opt_len, max_batch=mb,
                     rank=rank, estimator=estimator, precision=self.precision, device=self.device, scope=scope,
                     arch=c.arch, max_pos=c.max_positions)
        if self._host is None:
            e.init_params(c.init_seed, c.init_scale)
        else:
            e.upload({k: v for k, v in self._host.items()})
            self._host = None
        for k, v in self._vectors.items():
            e.upload({k: v})
        self._engine = e
        return e

    def sync_host(self, matrices: bool = True, vectors: bool = True) -> None:
        """Write the device values back into the host dict this replica was made from
        (in place, like the reference's mutations); no-op for device-born params."""
        mirror = getattr(self, "_mirror", None)
        if mirror is None or self._engine is None:
            return
        self.invalidate()
        for k in list(mirror):
            if (np.ndim(mirror[k]) == 2 and matrices) or (np.ndim(mirror[k]) == 1 and vectors):
                mirror[k][...] = self[k]

    def to_host(self) -> dict[str, np.ndarray]:
        return {k: np.array(self[k]) for k in self}


def init_params(cfg: ModelConfig, precision: str = "fp16", max_batch: int = 16, device: int = 0) -> DeviceParams:
    """Fresh parameters (model.py:84-108), regenerated on the device: matrices
    = init_scale * N(0,1) from Role.INIT streams (bit-exact float64), layer
    norms at identity."""
    return DeviceParams(cfg, precision=precision, max_batch=max_batch, device=device)


# the last plain host dict a step function saw and its device replica: the reference's
# params are a caller-owned dict mutated in place (runtime.py:242-250, zo_engine.py:449-450),
# so a dict keeps ONE replica across calls and mutating entry points write back into it
_HOST_BINDING: list = [None, None]


def as_device_params(params, cfg: ModelConfig) -> DeviceParams:
    """``params`` as a device replica.  A :class:`DeviceParams` is used as is.  A plain
    mapping (the reference's dict) is uploaded once and the replica cached by identity;
    the device copy is authoritative from then on, and the step functions that mutate
    parameters (folds, factorized / dense updates, full-scope vector updates) write
    the new values back into the caller's arrays in place (``sync_host``).  Use
    ``DeviceParams`` directly at scale: the write-back downloads every matrix."""
    if isinstance(params, DeviceParams):
        return params
    if isinstance(params, Mapping):
        dp = _HOST_BINDING[1]
        if _HOST_BINDING[0] is params and dp is not None and dp.cfg == cfg:
            return dp
        dp = DeviceParams(cfg, host=params)
        dp._mirror = params
        _HOST_BINDING[0], _HOST_BINDING[1] = params, dp
        return dp
    raise InputError("params must be a mapping of layer id -> array")


def params_digest(params: Mapping[str, np.ndarray]) -> str:
    """Chained digest over sorted layer ids and float64 weights (model.py:111-117)."""
    h = digest_text("params")
    for lid in sorted(params):
        h = digest_text(lid, h)
        h = digest_array(params[lid], h)
    return digest_hex(h)


def matrix_ids(params) -> list[str]:
    if isinstance(params, DeviceParams):
        return sorted(params._shapes)
    return sorted(k for k, v in params.items() if np.ndim(v) == 2)


def vector_ids(params) -> list[str]:
    if isinstance(params, DeviceParams):
        return sorted(params._vectors)
    return sorted(k for k, v in params.items() if np.ndim(v) == 1)


def pos_encoding(length: int, dim: int) -> np.ndarray:
    """Sinusoidal table (model.py:128-136); the device keeps an fp32 copy."""
    t = np.arange(length, dtype=np.float64)[:, None]
    j = np.arange(dim)[None, :]
    ang = t / np.power(10000.0, (2.0 * (j // 2)) / dim)
    return np.where(j % 2 == 0, np.sin(ang), np.cos(ang))


# --------------------------------------------------------------------------- task
@dataclass(frozen=True)
class TaskConfig:
    """Synthetic marker-detection task (model.py:312-336)."""
    seed: int = 11
    vocab: int = 64
    prompt_len: int = 16
    train_size: int = 256
    dev_size: int = 64
    val_size: int = 128
    marker_token: int = 3

    def __post_init__(self) -> None:
        if self.vocab < 8:
            raise ConfigError("task vocab too small for markers and options")
        if min(self.train_size, self.dev_size, self.val_size) < 2:
            raise ConfigError("split sizes must be >= 2")

    @property
    def options(self) -> tuple[tuple[int, ...], ...]:
        return ((self.vocab - 2,), (self.vocab - 1,))

    @property
    def alphabet(self) -> tuple[int, int]:
        return (4, self.vocab - 2)


@dataclass
class TaskData:
    config: TaskConfig
    splits: dict[str, tuple[np.ndarray, np.ndarray]] = field(default_factory=dict)

    def digest(self) -> str:  # model.py:339-352
        h = digest_text("task")
        h = digest_text(json.dumps(self.config.__dict__, sort_keys=True), h)
        for name in sorted(self.splits):
            p, g = self.splits[name]
            h = digest_text(name, h)
            h = digest_bytes(p.astype("<i8").tobytes(), h)
            h = digest_bytes(g.astype("<i8").tobytes(), h)
        return digest_hex(h)


def _make_split(cfg: TaskConfig, name: str, size: int):
    rng = StreamKey(cfg.seed, 0, f"task.{name}", Role.INIT).generator()
    lo, hi = cfg.alphabet
    prompts = rng.integers(lo, hi, size=(size, cfg.prompt_len), dtype=np.int64)
    labels = np.zeros(size, dtype=np.int64)
    labels[: size // 2] = 1
    labels = labels[rng.permutation(size)]
    pos = rng.integers(0, cfg.prompt_len, size=size)
    rows = np.nonzero(labels == 1)[0]
    prompts[rows, pos[rows]] = cfg.marker_token
    return prompts, labels


def generate_task(cfg: TaskConfig) -> TaskData:
    """Balanced train/dev/val splits (model.py:355-378); gold option = label."""
    data = TaskData(config=cfg)
    for name, size in (("train", cfg.train_size), ("dev", cfg.dev_size), ("val", cfg.val_size)):
        data.splits[name] = _make_split(cfg, name, size)
    return data


def save_task(data: TaskData, path: str) -> None:
    doc = {"config": data.config.__dict__,
           "splits": {n: {"prompts": p.tolist(), "golds": g.tolist()} for n, (p, g) in sorted(data.splits.items())}}
    with open(path, "w") as f:
        json.dump(doc, f, sort_keys=True)


def load_task(path: str) -> TaskData:
    with open(path) as f:
        doc = json.load(f)
    data = TaskData(config=TaskConfig(**doc["config"]))
    for n, s in doc["splits"].items():
        data.splits[n] = (np.asarray(s["prompts"], dtype=np.int64), np.asarray(s["golds"], dtype=np.int64))
    return data


@dataclass
class Minibatch:
    """Examples of one scoring call (model.py:406-427)."""
    prompts: np.ndarray
    golds: np.ndarray
    options: tuple[tuple[int, ...], ...]
    indices: np.ndarray

    def __post_init__(self) -> None:
        if len({len(o) for o in self.options}) != 1:
            raise InputError("candidate options must share one token length")
        if self.golds.min() < 0 or self.golds.max() >= len(self.options):
            raise InputError("gold option index out of range")

    def option_array(self) -> np.ndarray:
        return np.asarray(self.options, dtype=np.int64)

    @property
    def batch_id(self) -> str:
        return digest_hex(digest_bytes(self.indices.astype("<i8").tobytes()))

    def sequences(self) -> tuple[np.ndarray, np.ndarray]:
        """(prompt || gold option tokens [B, T], gold option tokens [B, L]) (model.py:238-240)."""
        gold = self.option_array()[self.golds]
        return np.concatenate([self.prompts, gold], axis=1), gold


def sample_minibatch(data: TaskData, split: str, seed: int, step: int, batch_size: int) -> Minibatch:
    """With-replacement draw from the (seed, step) MINIBATCH stream (model.py:463-475)."""
    prompts, golds = data.splits[split]
    if batch_size < 1 or batch_size > prompts.shape[0]:
        raise DimensionError(f"batch_size {batch_size} not in [1, {prompts.shape[0]}]")
    idx = sample_indices(StreamKey(seed, step, f"task.{split}", Role.MINIBATCH), batch_size, prompts.shape[0])
    return Minibatch(prompts=prompts[idx], golds=golds[idx], options=data.config.options, indices=idx)


@dataclass
class EvalPoint:
    step: int
    wall_ms: float
    loss: float
    acc: float

    def to_dict(self) -> dict:
        return {"step": self.step, "wall_ms": self.wall_ms, "loss": self.loss, "acc": self.acc}


# --------------------------------------------------------------------------- scoring
def _check_tokens(tokens: np.ndarray, vocab: int) -> None:
    if tokens.min() < 0 or tokens.max() >= vocab:
        raise InputError(f"token id outside [0, {vocab})")


def _view_state(view):
    """The AdapterState behind a view (our views carry it; None = bare base)."""
    if view is None:
        return None
    st = getattr(view, "state", None)
    if st is None:
        raise ConfigError("forward_score on the B200 engine needs a view from AdapterState.view()")
    return st


def forward_nll(params, cfg: ModelConfig, prompts: np.ndarray, option_tokens: np.ndarray, view=None,
                precision: str = "real64") -> np.ndarray:
    """Per-example option NLL (model.py:202-215) for one composition, chunked
    over the engine's batch capacity.  option_tokens: [B, L]."""
    dp = as_device_params(params, cfg)
    eng = dp.engine if dp.bound else dp.bind(opt_len=option_tokens.shape[1])
    st = _view_state(view)
    sign = 0 if st is None else st.perturb_sign
    seq = np.concatenate([prompts, option_tokens], axis=1)
    _check_tokens(seq, cfg.vocab)
    if st is not None:
        st._sync_to_engine(eng)
    eng.prepare_probe(st.epsilon if st is not None else 0.0, 1 if (st is None or sign == 0 or not st._probe_on) else 0)
    out = np.empty(seq.shape[0])
    for s in range(0, seq.shape[0], eng.max_batch):
        tk, gd = seq[s: s + eng.max_batch], option_tokens[s: s + eng.max_batch]
        if sign == 0 or st is None or not st._probe_on:
            out[s: s + len(tk)] = eng.score(tk, gd, nsign=1)[0]
        else:
            nll = eng.score(tk, np.stack([gd, gd]), nsign=2)
            out[s: s + len(tk)] = nll[0] if sign > 0 else nll[1]
    return out


def forward_score(params, cfg: ModelConfig, batch: Minibatch, view=None, precision: str = "real64") -> float:
    """Mean gold-option NLL under the composed weights (model.py:223-244):
    per-example scores on the tensor-core path, float64 canonical mean."""
    resolve_precision(precision)
    prompts, gold = batch.prompts, batch.option_array()[batch.golds]
    return canonical_mean(forward_nll(params, cfg, prompts, gold, view, precision))


def eval_accuracy(params, cfg: ModelConfig, prompts: np.ndarray, golds: np.ndarray,
                  options: tuple[tuple[int, ...], ...], view=None, precision: str = "real64") -> float:
    """Fraction whose gold option scores highest; ties -> lowest index (model.py:247-269).
    score_j = -(NLL of option j), computed per option as the reference does."""
    B = prompts.shape[0]
    scores = np.zeros((B, len(options)))
    for j, opt in enumerate(options):
        toks = np.tile(np.asarray(opt, dtype=np.int64), (B, 1))
        scores[:, j] = -forward_nll(params, cfg, prompts, toks, view, precision)
    return float(np.mean(np.argmax(scores, axis=1) == np.asarray(golds)))


def _one_forward_options(params, cfg: ModelConfig, prompts: np.ndarray, opts: np.ndarray, view):
    """Every single-token option's NLL [n_opt, B] from ONE sign-0 forward per batch chunk
    (zob200.h zo_score_options): the scored row never sees the option token, so its
    logits serve all options.  None when the configuration needs a forward per option
    (multi-token options, a +-eps probe view, high rank, real32)."""
    if opts.shape[1] != 1:
        return None
    dp = as_device_params(params, cfg)
    eng = dp.engine if dp.bound else dp.bind(opt_len=1)
    st = _view_state(view)
    if (st is not None and st.perturb_sign != 0 and st._probe_on) or eng.rank > 8 or eng.precision == "real32":
        return None
    if st is not None:
        st._sync_to_engine(eng)
    eng.prepare_probe(st.epsilon if st is not None else 0.0, 1)
    seq = np.concatenate([prompts, np.tile(opts[0], (prompts.shape[0], 1))], axis=1)
    _check_tokens(seq, cfg.vocab)
    out = np.empty((opts.shape[0], seq.shape[0]))
    for s in range(0, seq.shape[0], eng.max_batch):
        tk = seq[s: s + eng.max_batch]
        out[:, s: s + len(tk)] = eng.score_options(tk, opts[:, 0])
    return out


def evaluate_split(params, cfg: ModelConfig, data: TaskData, split: str = "dev", view=None,
                   precision: str = "real64") -> tuple[float, float]:
    """(loss, accuracy) over a whole split (model.py:444-460).  Single-token options
    (the SST-2 shape) are all scored from one forward (_one_forward_options); otherwise
    one forward per option, as the reference does."""
    prompts, golds = data.splits[split]
    opts = np.asarray(data.config.options, dtype=np.int64)
    one = _one_forward_options(params, cfg, prompts, opts, view)
    per_opt = list(one) if one is not None else [
        forward_nll(params, cfg, prompts, np.tile(opts[j], (prompts.shape[0], 1)), view, precision)
        for j in range(len(opts))]
    nll_gold = np.choose(golds, per_opt)
    loss = canonical_mean(nll_gold)
    scores = -np.stack(per_opt, axis=1)
    acc = float(np.mean(np.argmax(scores, axis=1) == golds))
    return loss, acc
