"""LoRA-slot algebra of ``zoserve.adapter`` (adapter.py:33-47) over the device engine.

On the B200 engine a slot is never materialised: the window slot (A, V_win)
and the probe (U, V_win) become one rank-r K-extension of every projection
GEMM, x . W_eff = [x | x (A +- eps U)] . [W ; V^T]  (csrc/zob200.cu), and the
tied embedding gets the same rank-r term on its gather and LM-head sides.

``AdapterState`` keeps the reference's public surface (epsilon, perturb_sign,
slot_cap, entries, set_sign, set_probe, clear_probes, view).  When bound to an
engine the device arenas are authoritative and ``entries`` returns host
snapshots; host-side edits (set_probe / window slots assigned by a caller) are
uploaded before the next scoring call.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, DimensionError

__all__ = ["LoraSlot", "AdapterEntry", "AdapterState", "compose_probe", "merge_slots", "accumulate_on_U",
           "fold_window"]


@dataclass
class LoraSlot:
    """contribution = scale * A @ B.T, A (m, k), B (n, k) (adapter.py:53-88)."""
    A: np.ndarray
    B: np.ndarray
    scale: float = 1.0

    def __post_init__(self) -> None:
        if self.A.ndim != 2 or self.B.ndim != 2:
            raise DimensionError("slot factors must be 2-D")
        if self.A.shape[1] != self.B.shape[1]:
            raise DimensionError(f"slot rank mismatch: A has {self.A.shape[1]} columns, B has {self.B.shape[1]}")

    @property
    def rank(self) -> int:
        return self.A.shape[1]

    @property
    def out_shape(self) -> tuple[int, int]:
        return (self.A.shape[0], self.B.shape[0])

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.out_shape)
        for k in range(self.rank):  # canonical k-ascending order (numerics.py:207-212)
            out += self.scale * np.multiply.outer(self.A[:, k], self.B[:, k])
        return out

    def copy(self) -> "LoraSlot":
        return LoraSlot(self.A.copy(), self.B.copy(), self.scale)


@dataclass
class AdapterEntry:
    m: int
    n: int
    update_slots: list[LoraSlot] = field(default_factory=list)
    window_slot: LoraSlot | None = None
    perturb_slot: LoraSlot | None = None

    def active_slots(self) -> list[LoraSlot]:
        return list(self.update_slots) + ([self.window_slot] if self.window_slot is not None else [])


class AdapterState:
    """Adapter entries + the shared probe switch (adapter.py:131-197)."""

    def __init__(self, epsilon: float, perturb_sign: int = 0, slot_cap: int = 4, entries=None):
        if epsilon < 0:
            raise ConfigError("epsilon must be >= 0")
        if slot_cap < 1:
            raise ConfigError("slot_cap must be >= 1")
        self.epsilon = epsilon
        self.perturb_sign = perturb_sign
        self.slot_cap = slot_cap
        self._host_entries: dict[str, AdapterEntry] = dict(entries or {})
        self._host_dirty = bool(entries)
        self._engine = None
        self._probe_on = False
        self._version = 0

    @property
    def version(self) -> int:
        """Mutation counter: bumped by every slot edit (entries, probes, frozen
        slots) and by every device update of the window A.  Scorers that cache
        L- between the +1 and -1 calls key the cache on it."""
        return self._version

    def _touch(self) -> None:
        self._version += 1

    # ---- reference surface
    @property
    def entries(self) -> dict[str, AdapterEntry]:
        if self._engine is None or self._host_dirty:
            return self._host_entries
        eng = self._engine
        A = eng.split(2, eng.get_slot(2))
        Vw = eng.split(1, eng.get_slot(1))
        Up = eng.split(0, eng.get_slot(0)) if self._probe_on else None
        out = {}
        for lid in eng.lids:
            m, n = eng.shapes[lid]
            e = AdapterEntry(m, n, window_slot=LoraSlot(A[lid], Vw[lid], 1.0))
            if Up is not None:
                e.perturb_slot = LoraSlot(Up[lid], Vw[lid], eng_probe_scale(eng))
            out[lid] = e
        return out

    def ensure_entry(self, layer_id: str, m: int, n: int) -> AdapterEntry:
        e = self._host_entries.get(layer_id)
        if e is None:
            e = AdapterEntry(m=m, n=n)
            self._host_entries[layer_id] = e
        elif (e.m, e.n) != (m, n):
            raise DimensionError(f"entry {layer_id} registered as {e.m}x{e.n}")
        self._host_dirty = True
        self._touch()
        return e

    def set_sign(self, sign: int) -> None:
        if sign not in (-1, 0, 1):
            raise ConfigError(f"perturb_sign must be -1, 0, or +1, got {sign}")
        self.perturb_sign = sign

    def set_probe(self, layer_id: str, left: np.ndarray, right: np.ndarray) -> None:
        e = self.ensure_entry(layer_id, left.shape[0], right.shape[0])
        e.perturb_slot = LoraSlot(left, right, 1.0)
        self._probe_on = True
        self._touch()

    def clear_probes(self) -> None:
        for e in self._host_entries.values():
            e.perturb_slot = None
        self._probe_on = False
        self._touch()

    def view(self):
        return _StateView(self)

    def add_frozen_slot(self, layer_id: str, slot: LoraSlot) -> None:
        e = self._host_entries[layer_id]
        e.update_slots.append(slot)
        if len(e.update_slots) > self.slot_cap:
            e.update_slots = [merge_slots(e.update_slots)]
        self._host_dirty = True
        self._touch()

    # ---- engine binding
    def _bind(self, engine) -> None:
        if self._engine is not None and self._engine is not engine:
            raise ConfigError("AdapterState is already bound to another engine")
        self._engine = engine

    def _sync_to_engine(self, eng) -> None:
        """Upload host-side slot edits: window A, window/probe V (shared), probe U."""
        self._bind(eng)
        if not self._host_dirty:
            return
        r = eng.rank
        A = {l: np.zeros((eng.shapes[l][0], r)) for l in eng.lids}
        Vw = eng.split(1, eng.get_slot(1))
        Up = {l: np.zeros((eng.shapes[l][0], r)) for l in eng.lids}
        for lid, e in self._host_entries.items():
            if e.update_slots and any(s.rank for s in e.update_slots):
                raise ConfigError("frozen update slots must be folded before device scoring")
            B = None
            if e.window_slot is not None and e.window_slot.rank:
                if e.window_slot.rank != r or e.window_slot.scale != 1.0:
                    raise ConfigError("window slot rank/scale must match the engine")
                A[lid] = e.window_slot.A
                B = e.window_slot.B
            if e.perturb_slot is not None:
                if e.perturb_slot.rank != r:
                    raise ConfigError("probe rank must match the engine")
                Up[lid] = e.perturb_slot.A
                if B is not None and not np.array_equal(B, e.perturb_slot.B):
                    raise ConfigError("window slot and probe must share V (one rank-r extension)")
                B = e.perturb_slot.B
            if B is not None:
                Vw[lid] = B
        eng.set_slot(1, eng.join(1, Vw))
        eng.set_slot(2, eng.join(2, A))
        eng.set_slot(0, eng.join(0, Up))
        # a host V has no window key unless the caller knows it (load_checkpoint); without
        # one the next step folds the uploaded A with this V and resamples V
        hint = getattr(self, "_window_hint", None)
        if hint is not None:
            eng.set_window(hint)
        self._window = hint
        self._window_hint = None
        self._host_dirty = False


def eng_probe_scale(eng) -> float:
    return 1.0 if eng.estimator == "lozo_lazy" else 1.0 / np.sqrt(eng.rank)


class _StateView:
    """WeightView stand-in: scoring reads the state (and its engine) directly."""

    def __init__(self, state: AdapterState):
        self.state = state

    def __call__(self, layer_id: str, base: np.ndarray) -> np.ndarray:
        """Host materialisation of the composed weight (debug/inspection only)."""
        e = self.state.entries.get(layer_id)
        return compose_probe(base, e, self.state.perturb_sign, self.state.epsilon)


def compose_probe(base: np.ndarray, entry: AdapterEntry | None, sign: int = 0, epsilon: float = 0.0) -> np.ndarray:
    """Host composition base + slots + sign*eps*probe (adapter.py:200-234).
    The engine never calls this -- it scores the K-extension instead."""
    if sign not in (-1, 0, 1):
        raise ConfigError(f"perturb_sign must be -1, 0, or +1, got {sign}")
    if entry is None:
        return base
    contrib = np.zeros(base.shape)
    for s in entry.active_slots():
        if s.rank:
            contrib += s.to_dense()
    p = entry.perturb_slot
    if sign != 0 and p is not None and p.rank:
        for k in range(p.rank):
            contrib += ((sign * epsilon) * p.scale) * np.multiply.outer(p.A[:, k], p.B[:, k])
    return base + contrib


def merge_slots(slots: list[LoraSlot]) -> LoraSlot:
    content = [s for s in slots if s.rank > 0]
    if not content:
        return LoraSlot(np.zeros((0, 0)), np.zeros((0, 0)), 1.0)
    return LoraSlot(np.hstack([s.scale * s.A for s in content]), np.hstack([s.B for s in content]), 1.0)


def accumulate_on_U(slot: LoraSlot, eta: float, c: float, g: np.ndarray) -> None:
    """Host form of the device update K8: A <- A + (-(eta*c)) * g (adapter.py:252-257)."""
    if g.shape != slot.A.shape:
        raise DimensionError(f"update shape {g.shape} != slot A shape {slot.A.shape}")
    slot.A += (-(eta * c)) * g


def fold_window(slot: LoraSlot, target: np.ndarray) -> None:
    """Host form of the device fold K9 (adapter.py:260-271)."""
    if slot.rank == 0:
        return
    for k in range(slot.rank):
        target += slot.scale * np.multiply.outer(slot.A[:, k], slot.B[:, k])
    slot.A[...] = 0.0
