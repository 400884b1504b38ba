"""Binary tensor containers (include/ttutv/io.hpp:10-19): the engine's header reader
(host only, no device) against the reference's read_tensor (src/io.cpp:151-161) on the same
files -- valid ones written by the reference, and every defect its checks name. The
error class, message and byte offset must agree."""
import struct

import numpy as np
import pytest

from paper_2501_07904_b200 import api
from paper_2501_07904_b200._native import ParseError


def _ten(dims, payload=None, magic=b"TTUTVTEN", version=1, order=None):
    order = len(dims) if order is None else order
    if payload is None:
        payload = np.arange(int(np.prod(dims)) if dims else 0, dtype="<f8").tobytes()
    return magic + struct.pack("<II", version, order) + b"".join(struct.pack("<Q", d) for d in dims) + payload


GOOD = _ten([3, 4, 5])
CASES = {
    "short_magic": b"TTUT",
    "bad_magic": b"TTUTVCOR" + GOOD[8:],
    "no_version": b"TTUTVTEN\x01\x00",
    "bad_version": _ten([3, 4, 5], version=2),
    "no_order": b"TTUTVTEN" + struct.pack("<I", 1) + b"\x03",
    "order_zero": _ten([], order=0),
    "order_big": b"TTUTVTEN" + struct.pack("<II", 1, 256),
    "short_dims": b"TTUTVTEN" + struct.pack("<II", 1, 3) + struct.pack("<Q", 3) + b"\x04\x00",
    "dim_zero": _ten([3, 0, 5], payload=b""),
    "dim_huge": _ten([3, 2**62, 5], payload=b""),
    "count_overflow": _ten([2**30, 2**30, 16], payload=b""),
    "short_payload": GOOD[:-8],
    "trailing": GOOD + b"\x00" * 3,
}


def test_valid_file_written_by_reference(ref, tmp_path):
    a = np.random.default_rng(3).standard_normal(2 * 3 * 4 * 5)
    p = tmp_path / "a.ttt"
    ref.write_tensor(p, a, [2, 3, 4, 5])
    assert api.tensor_file_header(p) == [2, 3, 4, 5]
    dims, payload = ref.read_tensor(p)
    assert dims == [2, 3, 4, 5]
    np.testing.assert_array_equal(payload, a)


@pytest.mark.parametrize("name", list(CASES))
def test_defects_match_reference(ref, tmp_path, name):
    p = tmp_path / f"{name}.ttt"
    p.write_bytes(CASES[name])
    with pytest.raises(ref.RefError) as r:
        ref.read_tensor(p)
    with pytest.raises(ParseError) as g:
        api.tensor_file_header(p)
    assert r.value.code == 3
    assert g.value.message == r.value.message
    assert g.value.offset == r.value.offset


def test_missing_file(ref, tmp_path):
    p = tmp_path / "nope.ttt"
    with pytest.raises(ref.RefError) as r:
        ref.read_tensor(p)
    with pytest.raises(ParseError) as g:
        api.tensor_file_header(p)
    assert (g.value.message, g.value.offset) == (r.value.message, r.value.offset)
