"""ZOAD adapter files and manifests -- ``zoserve.adapter`` serialization
(adapter.py:279-415), byte-compatible with the reference's writer/reader.

Wire format (little-endian), restated from adapter.py:305-368:

    b"ZOAD" | u32 version=1 | f64 epsilon | i8 perturb_sign | u32 n_entries
    per entry (sorted layer ids):
        u16 len | utf-8 layer id | u32 m | u32 n | u32 n_slots
        per slot: u8 kind (0 frozen, 1 window, 2 probe) | u32 rank | f64 scale
                  | A (m x rank f64) | B (n x rank f64)

plus a sidecar ``<path>.manifest.json`` with per-layer and whole-state FNV
digests and the file digest (adapter.py:370-415).  A bound ``AdapterState``
serializes its device arenas (window A, window V and -- while a probe is
installed -- the probe U), so a device run checkpoints into the same file the
reference writes.
"""
from __future__ import annotations

import json
import struct

import numpy as np

from .adapter import AdapterEntry, AdapterState, LoraSlot
from .errors import InputError
from .numerics import FNV_OFFSET_BASIS, digest_array, digest_bytes, digest_hex, digest_text

__all__ = ["save_adapter", "load_adapter", "state_digest", "adapter_manifest"]

_MAGIC = b"ZOAD"
_VERSION = 1
_HEAD = "<IdbI"
_SLOT = "<Id"


def _pack_slot(slot: LoraSlot) -> bytes:  # adapter.py:279-281
    return (struct.pack(_SLOT, slot.rank, slot.scale) + np.ascontiguousarray(slot.A, "<f8").tobytes()
            + np.ascontiguousarray(slot.B, "<f8").tobytes())


def _unpack_slot(buf: memoryview, off: int, m: int, n: int) -> tuple[LoraSlot, int]:  # adapter.py:284-292
    k, scale = struct.unpack_from(_SLOT, buf, off)
    off += struct.calcsize(_SLOT)
    a = np.frombuffer(buf, dtype="<f8", count=m * k, offset=off).reshape(m, k).copy()
    off += m * k * 8
    b = np.frombuffer(buf, dtype="<f8", count=n * k, offset=off).reshape(n, k).copy()
    off += n * k * 8
    return LoraSlot(a, b, float(scale)), off


def _entry_slots(entry: AdapterEntry) -> list[tuple[int, LoraSlot]]:  # adapter.py:295-302
    out = [(0, s) for s in entry.update_slots]
    if entry.window_slot is not None:
        out.append((1, entry.window_slot))
    if entry.perturb_slot is not None:
        out.append((2, entry.perturb_slot))
    return out


def save_adapter(state: AdapterState, path: str) -> dict:
    """adapter.py:305-328: versioned binary file + ``<path>.manifest.json``."""
    entries = state.entries
    blob = bytearray(_MAGIC)
    blob += struct.pack(_HEAD, _VERSION, state.epsilon, state.perturb_sign, len(entries))
    for lid in sorted(entries):
        entry = entries[lid]
        lb = lid.encode("utf-8")
        slots = _entry_slots(entry)
        blob += struct.pack("<H", len(lb)) + lb
        blob += struct.pack("<III", entry.m, entry.n, len(slots))
        for kind, slot in slots:
            blob += struct.pack("<B", kind) + _pack_slot(slot)
    data = bytes(blob)
    with open(path, "wb") as f:
        f.write(data)
    manifest = adapter_manifest(state, entries)
    manifest["file_digest"] = digest_hex(digest_bytes(data))
    with open(path + ".manifest.json", "w") as f:
        json.dump(manifest, f, indent=2, sort_keys=True)
    return manifest


def load_adapter(path: str, check_manifest: bool = True) -> AdapterState:
    """adapter.py:331-368: digest-checked read; raises InputError on corruption,
    bad magic or an unsupported version."""
    with open(path, "rb") as f:
        data = f.read()
    if check_manifest:
        try:
            with open(path + ".manifest.json") as f:
                manifest = json.load(f)
        except FileNotFoundError:
            manifest = None
        if manifest is not None:
            got = digest_hex(digest_bytes(data))
            if manifest.get("file_digest") != got:
                raise InputError(f"adapter file digest {got} does not match manifest")
    if data[:4] != _MAGIC:
        raise InputError("not an adapter file (bad magic)")
    off = 4
    try:
        version, epsilon, sign, n_entries = struct.unpack_from(_HEAD, data, off)
    except struct.error as e:
        raise InputError(f"truncated adapter file: {e}") from None
    off += struct.calcsize(_HEAD)
    if version != _VERSION:
        raise InputError(f"unsupported adapter file version {version}")
    state = AdapterState(epsilon=float(epsilon), perturb_sign=int(sign))
    buf = memoryview(data)
    try:
        for _ in range(n_entries):
            (ll,) = struct.unpack_from("<H", buf, off)
            off += 2
            lid = bytes(buf[off:off + ll]).decode("utf-8")
            off += ll
            m, n, n_slots = struct.unpack_from("<III", buf, off)
            off += struct.calcsize("<III")
            entry = state.ensure_entry(lid, m, n)
            for _ in range(n_slots):
                (kind,) = struct.unpack_from("<B", buf, off)
                off += 1
                slot, off = _unpack_slot(buf, off, m, n)
                if kind == 0:
                    entry.update_slots.append(slot)
                elif kind == 1:
                    entry.window_slot = slot
                else:
                    entry.perturb_slot = slot
    except (struct.error, ValueError) as e:
        raise InputError(f"truncated adapter file: {e}") from None
    state._probe_on = any(e.perturb_slot is not None for e in state._host_entries.values())
    return state


def _digest_slot(slot: LoraSlot, h: int) -> int:  # adapter.py:371-375
    h = digest_bytes(struct.pack(_SLOT, slot.rank, slot.scale), h)
    h = digest_array(slot.A, h)
    return digest_array(slot.B, h)


def state_digest(state: AdapterState, entries: dict | None = None) -> str:
    """adapter.py:378-389: slots, probes, sign and epsilon."""
    entries = state.entries if entries is None else entries
    h = digest_text("adapter")
    h = digest_bytes(struct.pack("<db", state.epsilon, state.perturb_sign), h)
    for lid in sorted(entries):
        h = digest_text(lid, h)
        for kind, slot in _entry_slots(entries[lid]):
            h = digest_bytes(bytes([kind]), h)
            h = _digest_slot(slot, h)
    return digest_hex(h)


def adapter_manifest(state: AdapterState, entries: dict | None = None) -> dict:
    """adapter.py:392-415."""
    entries = state.entries if entries is None else entries
    layers = {}
    for lid in sorted(entries):
        entry = entries[lid]
        h = FNV_OFFSET_BASIS
        for kind, slot in _entry_slots(entry):
            h = digest_bytes(bytes([kind]), h)
            h = _digest_slot(slot, h)
        layers[lid] = {"shape": [entry.m, entry.n], "slots": len(_entry_slots(entry)), "digest": digest_hex(h)}
    return {"version": _VERSION, "epsilon": state.epsilon, "perturb_sign": state.perturb_sign,
            "state_digest": state_digest(state, entries), "layers": layers}
