"""Trace ingestion: the native parser (bs_trace_parse) against the
live reference's load_trace on golden inputs (oracle/gen_trace_golden.py): records in
arrival order with file-order ids, or the same TraceFormatError line and message.
Host code only — runs without a GPU."""

import gzip
import io
import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN_DIR
from paper_2507_17120_b200 import TraceFormatError
from paper_2507_17120_b200 import trace as T

with gzip.open(os.path.join(GOLDEN_DIR, "traces.json.gz"), "rt") as fh:
    FIXTURES = json.load(fh)


def _check(fx, threads=1):
    fmt = T.TraceFormat(fx["fmt"])
    if fx["ok"]:
        tr = T.parse_trace(fx["text"], fmt, threads=threads)
        assert tr.id.tolist() == fx["id"]
        assert [repr(float(a)) for a in tr.arrival] == fx["arrival"]
        assert tr.input_len.tolist() == fx["input"]
        assert tr.output_len.tolist() == fx["output"]
        assert tr.cls.tolist() == fx["cls"]
    else:
        with pytest.raises(TraceFormatError) as exc:
            T.parse_trace(fx["text"], fmt, threads=threads)
        assert exc.value.line == fx["err_line"]
        assert str(exc.value) == fx["err_msg"]


@pytest.mark.parametrize("fx", FIXTURES, ids=[f["name"] for f in FIXTURES])
def test_parser_matches_reference(fx):
    _check(fx)


def test_fixture_set_covers_both_formats_and_errors():
    assert len(FIXTURES) >= 60
    assert sum(f["ok"] for f in FIXTURES) >= 20 and sum(not f["ok"] for f in FIXTURES) >= 30
    assert {f["fmt"] for f in FIXTURES} == {"csv", "jsonl"}


def _big(fmt, copies):
    src = next(f for f in FIXTURES if f["name"] == f"synthetic0_{fmt}")
    body = src["text"]
    if fmt == "csv":
        header, rest = body.split("\n", 1)
        return header + "\n" + rest * copies, src
    return body * copies, src


@pytest.mark.parametrize("fmt", ["csv", "jsonl"])
def test_multithreaded_parse_equals_single_thread(fmt):
    text, src = _big(fmt, 40)          # > 1 MiB: the parser splits it across threads
    assert len(text) > (1 << 20)
    one = T.parse_trace(text, fmt, threads=1)
    many = T.parse_trace(text, fmt, threads=8)
    for k in ("id", "arrival", "input_len", "output_len", "cls"):
        assert np.array_equal(getattr(one, k), getattr(many, k)), k
    n1 = len(src["id"])
    assert len(one) == 40 * n1
    # copy c of record j has file-order id c*n1 + j; the stable sort keeps equal arrivals in file order
    assert np.all(np.diff(one.arrival) >= 0)
    first = one.id[one.id < n1]
    assert first.tolist() == sorted(first.tolist(), key=lambda i: src["id"].index(i))


@pytest.mark.parametrize("fmt", ["csv", "jsonl"])
def test_error_line_numbers_under_chunking(fmt):
    text, _ = _big(fmt, 40)
    lines = text.split("\n")
    bad = len(lines) * 3 // 4
    lines[bad] = "1.0,oops,1,online" if fmt == "csv" else '{"arrival_s": 1.0, "input_tokens": "x", "class": "online"}'
    with pytest.raises(TraceFormatError) as exc:
        T.parse_trace("\n".join(lines), fmt, threads=8)
    assert exc.value.line == bad + 1


def test_binary_roundtrip(tmp_path):
    src = next(f for f in FIXTURES if f["name"] == "synthetic1_jsonl")
    tr = T.parse_trace(src["text"], "jsonl")
    p = tmp_path / "t.bst"
    T.save_binary(tr, p)
    back = T.load_trace_path(p)
    for k in ("id", "arrival", "input_len", "output_len", "cls"):
        assert np.array_equal(getattr(tr, k), getattr(back, k)), k
    empty = T.parse_trace("", "csv")
    T.save_binary(empty, tmp_path / "e.bst")
    assert len(T.load_binary(tmp_path / "e.bst")) == 0


def test_text_roundtrip_and_window():
    src = next(f for f in FIXTURES if f["name"] == "synthetic1_csv")
    tr = T.parse_trace(src["text"], "csv")
    buf = io.StringIO()
    T.save_trace(tr, buf, T.TraceFormat.CSV)
    again = T.parse_trace(buf.getvalue(), "csv")
    assert np.array_equal(again.arrival, tr.arrival)
    assert np.array_equal(again.input_len, tr.input_len)
    lens, cls = tr.window(max_seq_len=4096)
    assert lens.dtype == np.int32 and lens.max() <= 4095 and len(cls) == len(tr)
    reqs = tr.requests()
    assert reqs[0].id == int(tr.id[0]) and reqs[0].arrival_time == float(tr.arrival[0])
    tr.validate()


def test_format_for_path_rejects_unknown_extension():
    from paper_2507_17120_b200 import ConfigError
    with pytest.raises(ConfigError):
        T.format_for_path("trace.txt")
