"""ZOAD adapter files (adapter.py:279-415) -- byte compatibility with the
reference's writer, pinned on tests/golden/adapter_rich.zoad (written by the
reference's save_adapter, see tests/golden/make_golden.py).  Host-only: no GPU."""
import json
import os

import numpy as np
import pytest

from paper_2605_28760_b200.adapter_io import adapter_manifest, load_adapter, save_adapter, state_digest
from paper_2605_28760_b200.errors import InputError


def _golden(golden_dir):
    p = os.path.join(golden_dir, "adapter_rich.zoad")
    with open(p + ".manifest.json") as f:
        return p, json.load(f)


def test_load_reference_file_and_digests(golden_dir):
    path, man = _golden(golden_dir)
    st = load_adapter(path)
    assert state_digest(st) == man["state_digest"]
    assert adapter_manifest(st)["layers"] == man["layers"]
    e = st.entries["blk0.qkv"]
    assert len(e.update_slots) == 1 and e.update_slots[0].scale == 0.5 and e.window_slot.rank == 2
    assert st.entries["embed"].perturb_slot.rank == 1
    assert st.epsilon == 2e-3 and st.perturb_sign == 0


def test_save_is_byte_identical_to_reference(golden_dir, tmp_path):
    path, man = _golden(golden_dir)
    st = load_adapter(path)
    out = str(tmp_path / "a.zoad")
    m2 = save_adapter(st, out)
    assert open(out, "rb").read() == open(path, "rb").read()
    assert m2 == man


def test_corruption_and_bad_magic_raise(golden_dir, tmp_path):
    path, _ = _golden(golden_dir)
    data = bytearray(open(path, "rb").read())
    bad = str(tmp_path / "bad.zoad")
    with open(bad, "wb") as f:
        f.write(bytes(data))
    with open(path + ".manifest.json") as f, open(bad + ".manifest.json", "w") as g:
        g.write(f.read())
    data[100] ^= 0xFF
    with open(bad, "wb") as f:
        f.write(bytes(data))
    with pytest.raises(InputError):
        load_adapter(bad)
    junk = str(tmp_path / "junk.bin")
    with open(junk, "wb") as f:
        f.write(b"nope" + b"\x00" * 64)
    with pytest.raises(InputError):
        load_adapter(junk, check_manifest=False)


def test_truncated_file_raises(golden_dir, tmp_path):
    path, _ = _golden(golden_dir)
    data = open(path, "rb").read()
    t = str(tmp_path / "t.zoad")
    with open(t, "wb") as f:
        f.write(data[:200])
    with pytest.raises(InputError):
        load_adapter(t, check_manifest=False)


def test_manifest_layer_digest_tracks_content(golden_dir):
    path, man = _golden(golden_dir)
    st = load_adapter(path)
    st.entries["blk1.ff_down"].window_slot.A[0, 0] += 1.0
    m2 = adapter_manifest(st)
    assert m2["layers"]["blk1.ff_down"]["digest"] != man["layers"]["blk1.ff_down"]["digest"]
    assert m2["layers"]["blk0.qkv"] == man["layers"]["blk0.qkv"]
    assert not np.isnan(st.entries["blk1.ff_down"].window_slot.A).any()
