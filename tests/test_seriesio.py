"""The GPU search's file front end against the reference's own io.cpp outputs
(tests/golden/io_golden.json, made by tests/golden/make_io_golden.py from the
unmodified reference): format_double (io.cpp:50-55), emit_stats
(io.cpp:57-74), load_series (io.cpp:17-42), save_series (io.cpp:44-48); plus
the binary series format's round trip and validation."""
from __future__ import annotations

import json
import os
import struct

import numpy as np
import pytest

from paper_2010_05371_b200 import seriesio
from paper_2010_05371_b200.api import BestSoFar, SearchReport

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "io_golden.json")))


def unbits(h: str) -> float:
    return struct.unpack("<d", struct.pack("<Q", int(h, 16)))[0]


def bits(v: float) -> str:
    return "0x%016x" % struct.unpack("<Q", struct.pack("<d", float(v)))[0]


def test_format_double_matches_reference():
    bad = [(s, seriesio.format_double(unbits(b))) for b, s in GOLDEN["format_double"]
           if seriesio.format_double(unbits(b)) != s]
    assert not bad, bad[:10]
    assert len(GOLDEN["format_double"]) > 300


def test_emit_stats_matches_reference(tmp_path):
    for case in GOLDEN["emit_stats"]:
        r = {k: (unbits(v) if isinstance(v, str) else v) for k, v in case["report"].items()}
        rep = SearchReport(**{k: r[k] for k in SearchReport.__dataclass_fields__ if k in r})
        best = BestSoFar(r["location"], r["distance_sq"], bool(r["found"]))
        assert seriesio.stats_json(rep, best) == case["text"]
        p = tmp_path / "stats.json"
        seriesio.emit_stats(rep, best, p)
        assert p.read_text() == case["text"]


@pytest.mark.parametrize("case", GOLDEN["load_series"], ids=lambda c: repr(c["content"])[:24])
def test_load_series_matches_reference(tmp_path, case):
    p = tmp_path / "series.txt"
    p.write_text(case["content"])
    if "values" in case:
        got = seriesio.load_series(p)
        assert [bits(v) for v in got] == case["values"]
    else:
        with pytest.raises(seriesio.SeriesFileError) as e:
            seriesio.load_series(p)
        assert str(e.value) == case["error"].replace("@PATH@", str(p))


def test_load_missing_file(tmp_path):
    p = tmp_path / "missing.txt"
    with pytest.raises(seriesio.SeriesFileError) as e:
        seriesio.load_series(p)
    assert str(e.value) == GOLDEN["load_missing_error"].replace("@PATH@", str(p))


def test_save_series_matches_reference(tmp_path):
    for case in GOLDEN["save_series"]:
        p = tmp_path / "s.txt"
        seriesio.save_series([unbits(b) for b in case["values"]], p)
        assert p.read_text() == case["text"]
        # text round trip is exact (shortest round-trip digits)
        assert [bits(v) for v in seriesio.load_series(p)] == case["values"]


@pytest.mark.parametrize("ext", [".f64", ".bin", ".npy"])
def test_binary_round_trip(tmp_path, ext):
    x = np.cumsum(np.random.default_rng(3).standard_normal(1000))
    p = tmp_path / ("ref" + ext)
    seriesio.save_series_binary(x, p)
    for mmap in (False, True):
        got = seriesio.read_series(p, mmap=mmap)
        assert np.array_equal(np.asarray(got), x)


def test_binary_validation(tmp_path):
    p = tmp_path / "e.f64"
    p.write_bytes(b"")
    with pytest.raises(seriesio.SeriesFileError, match="empty series file"):
        seriesio.load_series_binary(p)
    p.write_bytes(b"\0" * 12)
    with pytest.raises(seriesio.SeriesFileError, match="multiple of 8"):
        seriesio.load_series_binary(p)
    np.array([1.0, np.inf, 2.0]).tofile(p)
    with pytest.raises(seriesio.SeriesFileError, match="sample 2 is not finite"):
        seriesio.load_series_binary(p)
    q = tmp_path / "x.npy"
    np.save(q, np.zeros((2, 2)))
    with pytest.raises(seriesio.SeriesFileError, match="1-D float64"):
        seriesio.load_series_binary(q)
    with pytest.raises(seriesio.SeriesFileError, match="cannot open"):
        seriesio.load_series_binary(tmp_path / "nope.f64")


def test_load_series_splits_on_c_whitespace_only(tmp_path):
    """operator>> (io.cpp:24) splits on " \\t\\n\\v\\f\\r" only: a NBSP (0xA0)
    or 0x1C byte stays inside the token, which then is not a number."""
    p = tmp_path / "s.txt"
    p.write_bytes(b"1\x0b2\x0c3\r4")
    assert seriesio.load_series(p).tolist() == [1.0, 2.0, 3.0, 4.0]
    for sep in (b"\xa0", b"\x1c", b"\x85"):
        p.write_bytes(b"1" + sep + b"2")
        with pytest.raises(seriesio.SeriesFileError, match="token 1"):
            seriesio.load_series(p)


def test_module_entry_point_validation_exit_code(tmp_path):
    """python -m paper_2010_05371_b200 is the CLI (exit 2 on a validation error)."""
    import subprocess
    import sys
    root = os.path.dirname(HERE)
    r = subprocess.run([sys.executable, "-m", "paper_2010_05371_b200", "search", "--data", "x",
                        "--query", "y", "--query-len", "8", "--window-ratio", "0.6",
                        "--algo", "eap"], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2
    assert r.stderr.startswith("error: --window-ratio")
