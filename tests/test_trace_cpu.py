"""ICET traces: the reader and writer against a trace
written by the reference's save_trace and the arrays its load_trace returns
(tests/golden/trace_small.*, made by tests/golden/make_golden.py trace);
error reporting as in the reference's tests (test_workload.py:97-125)."""

import os

import numpy as np
import pytest

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")


def test_reads_the_reference_trace():
    from paper_2604_10539_b200.trace import load_trace
    tr = load_trace(os.path.join(GOLD, "trace_small.icet"))
    z = np.load(os.path.join(GOLD, "trace_small.npz"))
    assert [tr.layers, tr.kv_heads, tr.query_heads_per_group, tr.d, tr.d_prime, tr.n_tokens] == list(z["shape"])
    assert np.array_equal(tr.keys.astype(np.float64), z["keys"])
    assert np.array_equal(tr.values.astype(np.float64), z["values"])
    assert np.array_equal(tr.queries.astype(np.float64), z["queries"])


def test_write_is_byte_identical_to_the_reference(tmp_path):
    from paper_2604_10539_b200.trace import load_trace, save_trace
    src = os.path.join(GOLD, "trace_small.icet")
    tr = load_trace(src)
    out = tmp_path / "again.icet"
    save_trace(tr.keys, tr.values, tr.queries, tr.query_heads_per_group, str(out))
    assert out.read_bytes() == open(src, "rb").read()


def test_header_layout(tmp_path):
    from paper_2604_10539_b200.trace import save_trace
    rng = np.random.default_rng(7)
    path = tmp_path / "t.icet"
    save_trace(rng.random((3, 1, 1, 2)), rng.random((3, 1, 1, 2)), rng.random((3, 1, 1, 2)), 1, str(path))
    raw = path.read_bytes()
    assert raw[:4] == b"ICET" and int.from_bytes(raw[4:8], "little") == 1
    assert [int.from_bytes(raw[8 + 4 * i:12 + 4 * i], "little") for i in range(6)] == [1, 1, 1, 2, 2, 3]
    assert len(raw) == 32 + 3 * (2 + 2 + 2) * 4


def test_malformed_traces_name_byte_offsets(tmp_path):
    from paper_2604_10539_b200.errors import TraceFormatError
    from paper_2604_10539_b200.trace import load_trace
    good = open(os.path.join(GOLD, "trace_small.icet"), "rb").read()
    path = tmp_path / "bad.icet"
    for data, where in ((b"NOPE" + good[4:], "byte offset 0"), (good[:20], "byte offset 20"),
                        (good[:4] + (2).to_bytes(4, "little") + good[8:], "byte offset 4"),
                        (good[:-3], f"byte offset {len(good) - 3}"),
                        (good[:8] + (0).to_bytes(4, "little") + good[12:], "byte offset 8")):
        path.write_bytes(data)
        with pytest.raises(TraceFormatError, match=where):
            load_trace(str(path))
