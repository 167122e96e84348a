"""ZOAD adapter files and manifests -- ``zoserve.adapter`` serialization
(adapter.py:279-415), byte-compatible with the reference's writer/reader.

The wire format is fixed by the reference (little-endian); it is declared once
here as a record table and every reader / writer / digest walks that table:

    header  ZOAD magic | u32 version=1 | f64 epsilon | i8 perturb_sign | u32 n_entries
    entry   u16 id length | utf-8 layer id | u32 m | u32 n | u32 n_slots   (sorted ids)
    slot    u8 kind (0 frozen, 1 window, 2 probe) | u32 rank | f64 scale
            | A (m x rank f64) | B (n x rank f64)

plus a sidecar ``<path>.manifest.json`` with per-layer and whole-state FNV digests
and the file digest.  A bound ``AdapterState`` serializes its device arenas
(window A, window V and -- while a probe is installed -- the probe U), so a device
run checkpoints into the same file the reference writes.
"""
from __future__ import annotations

import json
import struct
from collections.abc import Iterator

import numpy as np

from .adapter import AdapterState, LoraSlot
from .errors import InputError
from .numerics import FNV_OFFSET_BASIS, digest_array, digest_bytes, digest_hex, digest_text

__all__ = ["save_adapter", "load_adapter", "state_digest", "adapter_manifest"]

MAGIC = b"ZOAD"
VERSION = 1
# record table of the ZOAD layout: record -> struct format of its fixed-size fields
RECORDS = {
    "header": "<IdbI",     # version, epsilon, perturb_sign, n_entries
    "id_len": "<H",
    "entry": "<III",       # m, n, n_slots
    "slot_kind": "<B",
    "slot": "<Id",         # rank, scale
}
KINDS = ("frozen", "window", "probe")


class _Cursor:
    """Sequential reader over the file bytes; every short read is an InputError."""

    def __init__(self, data: bytes):
        self.buf = memoryview(data)
        self.pos = 0

    def record(self, name: str) -> tuple:
        fmt = RECORDS[name]
        try:
            out = struct.unpack_from(fmt, self.buf, self.pos)
        except struct.error as e:
            raise InputError(f"truncated adapter file ({name}): {e}") from None
        self.pos += struct.calcsize(fmt)
        return out

    def raw(self, n: int) -> bytes:
        if self.pos + n > len(self.buf):
            raise InputError("truncated adapter file (layer id)")
        out = bytes(self.buf[self.pos:self.pos + n])
        self.pos += n
        return out

    def matrix(self, rows: int, cols: int) -> np.ndarray:
        n = rows * cols
        if self.pos + 8 * n > len(self.buf):
            raise InputError("truncated adapter file (slot factor)")
        out = np.frombuffer(self.buf, dtype="<f8", count=n, offset=self.pos).reshape(rows, cols).copy()
        self.pos += 8 * n
        return out


def _slots(entries) -> Iterator[tuple[str, object, list[tuple[int, LoraSlot]]]]:
    """(layer id, entry, [(kind, slot)]) in file order: sorted ids; frozen slots, then the
    window slot, then the probe (adapter.py:295-302)."""
    for lid in sorted(entries):
        e = entries[lid]
        seq = [(0, s) for s in e.update_slots]
        seq += [(k, s) for k, s in ((1, e.window_slot), (2, e.perturb_slot)) if s is not None]
        yield lid, e, seq


def _slot_bytes(slot: LoraSlot) -> bytes:
    return (struct.pack(RECORDS["slot"], slot.rank, slot.scale) + np.ascontiguousarray(slot.A, "<f8").tobytes()
            + np.ascontiguousarray(slot.B, "<f8").tobytes())


def _encode(state: AdapterState, entries) -> bytes:
    parts = [MAGIC, struct.pack(RECORDS["header"], VERSION, state.epsilon, state.perturb_sign, len(entries))]
    for lid, e, seq in _slots(entries):
        name = lid.encode("utf-8")
        parts += [struct.pack(RECORDS["id_len"], len(name)), name,
                  struct.pack(RECORDS["entry"], e.m, e.n, len(seq))]
        for kind, slot in seq:
            parts += [struct.pack(RECORDS["slot_kind"], kind), _slot_bytes(slot)]
    return b"".join(parts)


def _decode(data: bytes) -> AdapterState:
    if data[:4] != MAGIC:
        raise InputError("not an adapter file (bad magic)")
    cur = _Cursor(data)
    cur.pos = len(MAGIC)
    version, epsilon, sign, n_entries = cur.record("header")
    if version != VERSION:
        raise InputError(f"unsupported adapter file version {version}")
    state = AdapterState(epsilon=float(epsilon), perturb_sign=int(sign))
    for _ in range(n_entries):
        (n_id,) = cur.record("id_len")
        try:
            lid = cur.raw(n_id).decode("utf-8")
        except UnicodeDecodeError as e:
            raise InputError(f"corrupt layer id: {e}") from None
        m, n, n_slots = cur.record("entry")
        entry = state.ensure_entry(lid, m, n)
        for _ in range(n_slots):
            (kind,) = cur.record("slot_kind")
            if kind >= len(KINDS):
                raise InputError(f"unknown slot kind {kind}")
            rank, scale = cur.record("slot")
            slot = LoraSlot(cur.matrix(m, rank), cur.matrix(n, rank), float(scale))
            if kind == 0:
                entry.update_slots.append(slot)
            elif kind == 1:
                entry.window_slot = slot
            else:
                entry.perturb_slot = slot
    state._probe_on = any(e.perturb_slot is not None for e in state._host_entries.values())
    return state


def _fold_slot_digest(h: int, kind: int, slot: LoraSlot) -> int:
    """kind byte, (rank, scale) record, A, B -- the per-slot digest chain (adapter.py:371-389)."""
    h = digest_bytes(bytes([kind]), h)
    h = digest_bytes(struct.pack(RECORDS["slot"], slot.rank, slot.scale), h)
    return digest_array(slot.B, digest_array(slot.A, h))


def state_digest(state: AdapterState, entries: dict | None = None) -> str:
    """Whole-state fingerprint: slots, probes, sign and epsilon (adapter.py:378-389)."""
    entries = state.entries if entries is None else entries
    h = digest_bytes(struct.pack("<db", state.epsilon, state.perturb_sign), digest_text("adapter"))
    for lid, _e, seq in _slots(entries):
        h = digest_text(lid, h)
        for kind, slot in seq:
            h = _fold_slot_digest(h, kind, slot)
    return digest_hex(h)


def adapter_manifest(state: AdapterState, entries: dict | None = None) -> dict:
    """Per-layer shape / slot count / digest plus the state digest (adapter.py:392-415)."""
    entries = state.entries if entries is None else entries
    layers = {}
    for lid, e, seq in _slots(entries):
        h = FNV_OFFSET_BASIS
        for kind, slot in seq:
            h = _fold_slot_digest(h, kind, slot)
        layers[lid] = {"shape": [e.m, e.n], "slots": len(seq), "digest": digest_hex(h)}
    return {"version": VERSION, "epsilon": state.epsilon, "perturb_sign": state.perturb_sign,
            "state_digest": state_digest(state, entries), "layers": layers}


def save_adapter(state: AdapterState, path: str) -> dict:
    """Versioned binary file + ``<path>.manifest.json`` (adapter.py:305-328)."""
    entries = state.entries
    data = _encode(state, entries)
    with open(path, "wb") as f:
        f.write(data)
    manifest = adapter_manifest(state, entries)
    manifest["file_digest"] = digest_hex(digest_bytes(data))
    with open(path + ".manifest.json", "w") as f:
        json.dump(manifest, f, indent=2, sort_keys=True)
    return manifest


def load_adapter(path: str, check_manifest: bool = True) -> AdapterState:
    """Digest-checked read (adapter.py:331-368); InputError on corruption, bad magic
    or an unsupported version."""
    with open(path, "rb") as f:
        data = f.read()
    if check_manifest:
        try:
            with open(path + ".manifest.json") as f:
                expected = json.load(f).get("file_digest")
        except FileNotFoundError:
            expected = None
        got = digest_hex(digest_bytes(data))
        if expected is not None and expected != got:
            raise InputError(f"adapter file digest {got} does not match manifest")
    return _decode(data)
