"""File front end of the GPU search: the reference's text formats plus a binary
series format for references too large to parse as text.

Text formats follow proj/src/io.cpp exactly (pinned by
tests/golden/io_golden.json, generated from the reference by
tests/golden/make_io_golden.py):

* ``load_series`` -- whitespace-delimited ASCII, tokens parsed like
  ``std::from_chars`` (io.cpp:17-42): optional '-', decimal digits with an
  optional point and exponent; no '+', no hex, no separators; out-of-range
  values are "not a number", inf/nan are "not finite"; empty -> error.
* ``save_series`` -- one ``format_double`` value per line (io.cpp:44-48).
* ``format_double`` -- ``std::to_chars`` shortest round-trip (io.cpp:50-55):
  the shorter of fixed and scientific notation, fixed on a tie, "inf" for the
  PRUNED sentinel.
* ``stats_json`` / ``emit_stats`` -- the ordered 10-key object of
  io.cpp:57-74 as nlohmann ``dump(2)`` writes it (doubles in its grisu
  format: fixed for decimal exponents in (-4, 15], ".0" on integral values,
  ``null`` for non-finite).

The binary format (new; no reference counterpart) is raw little-endian
float64 (``.f64``/``.bin``) or a NumPy ``.npy`` file, validated with the same
rules as the text loader (non-empty, finite) so both load paths accept the
same series.
"""
from __future__ import annotations

import math
import os
import re
from decimal import Decimal

import numpy as np

# from_chars(chars_format::general) subject sequence, plus the inf/nan spellings
# it also accepts (rejected afterwards as "not finite").
_NUMBER = re.compile(r"-?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?")
_NONFINITE = re.compile(r"-?(?:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)", re.IGNORECASE)


_CSPACE = re.compile(r"[ \t\n\v\f\r]+")


class SeriesFileError(RuntimeError):
    """io.cpp's std::runtime_error for unreadable or malformed series files."""


def _shortest(v: float) -> tuple[str, int]:
    """Shortest round-trip digits of |v| > 0 and the decimal point position n
    (|v| = 0.d1d2...dk x 10^n)."""
    d = Decimal(repr(abs(v))).normalize()
    sign, digits, exp = d.as_tuple()
    s = "".join(map(str, digits))
    return s, exp + len(s)


def format_double(v: float) -> str:
    """io.cpp:50-55 (std::to_chars, plain overload)."""
    v = float(v)
    if v == math.inf:
        return "inf"
    if v == -math.inf:
        return "-inf"
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    neg = math.copysign(1.0, v) < 0
    if v == 0.0:
        return "-0" if neg else "0"
    digits, n = _shortest(v)
    k = len(digits)
    # scientific: d[.ddd]e[+-]XX
    mant = digits[0] + ("." + digits[1:] if k > 1 else "")
    e = n - 1
    sci = mant + "e" + ("-" if e < 0 else "+") + ("%02d" % abs(e))
    # fixed: libstdc++ prints integral values >= 10^k exactly
    if v == math.floor(v):
        fixed = str(int(abs(v)))
    elif n <= 0:
        fixed = "0." + "0" * (-n) + digits
    else:
        fixed = digits[:n] + "." + digits[n:]
    out = fixed if len(fixed) <= len(sci) else sci
    return ("-" if neg else "") + out


def _json_double(v: float) -> str:
    """nlohmann::json serialisation of a double (dump_float + format_buffer,
    kMinExp = -4, kMaxExp = 15)."""
    v = float(v)
    if not math.isfinite(v):
        return "null"
    neg = math.copysign(1.0, v) < 0
    if v == 0.0:
        return "-0.0" if neg else "0.0"
    digits, n = _shortest(v)
    k = len(digits)
    if k <= n <= 15:
        s = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        s = (digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + ("-" if e < 0 else "+")
             + ("%02d" % abs(e)))
    return ("-" if neg else "") + s


_STATS_KEYS = ("candidates_total", "pruned_kim", "pruned_keogh_eq", "pruned_keogh_ec",
               "dtw_calls", "dtw_abandoned", "dp_cells_evaluated")


def stats_json(report, best) -> str:
    """The text io.cpp:57-74 writes (nlohmann ordered_json, dump(2), newline)."""
    items = [(k, str(int(getattr(report, k)))) for k in _STATS_KEYS]
    items.append(("elapsed_seconds", _json_double(report.elapsed_seconds)))
    items.append(("best_location", str(int(best.location))))
    items.append(("best_distance_sq", _json_double(best.distance_sq)))
    body = ",\n".join(f'  "{k}": {v}' for k, v in items)
    return "{\n" + body + "\n}\n"


def emit_stats(report, best, path) -> None:
    """io.cpp:57-74"""
    try:
        with open(path, "w") as f:
            f.write(stats_json(report, best))
    except OSError:
        raise SeriesFileError(f"cannot write stats to '{os.fspath(path)}'") from None


def trace_csv(trace) -> str:
    """write_trace_csv (io.cpp:76-122): header, then events in order -- every
    cell, a discard point right after its cell, a row's pruning points when
    the row closes (the border row's before every cell), the abandon cell
    last; marker values are the last captured value of their cell, else inf."""
    lines = ["row,col,value,kind"]

    def value_at(ref):
        for r, c, v in reversed(trace.cells):
            if (r, c) == tuple(ref):
                return format_double(v)
        return "inf"

    def emit(r, c, value, kind):
        lines.append(f"{r},{c},{value},{kind}")

    nd = npp = 0
    dps, pps, cells = trace.discard_points, trace.pruning_points, trace.cells
    while npp < len(pps) and pps[npp][0] == 0:
        emit(pps[npp][0], pps[npp][1], "inf", "pruning_point")
        npp += 1
    for k, (r, c, v) in enumerate(cells):
        emit(r, c, format_double(v), "cell")
        if nd < len(dps) and tuple(dps[nd]) == (r, c):
            nd += 1
            emit(r, c, format_double(v), "discard_point")
        row_done = k + 1 == len(cells) or cells[k + 1][0] != r
        while row_done and npp < len(pps) and pps[npp][0] == r:
            emit(pps[npp][0], pps[npp][1], value_at(pps[npp]), "pruning_point")
            npp += 1
    if trace.abandon_cell is not None:
        a = trace.abandon_cell
        emit(a[0], a[1], value_at(a), "abandon")
    return "\n".join(lines) + "\n"


def write_trace_csv(trace, path) -> None:
    """io.cpp:76-122"""
    try:
        with open(path, "w") as f:
            f.write(trace_csv(trace))
    except OSError:
        raise SeriesFileError(f"cannot write trace to '{os.fspath(path)}'") from None


def _parse_token(tok: str) -> float | None:
    """std::from_chars on the whole token; None = 'is not a number'."""
    if _NONFINITE.fullmatch(tok):
        return math.nan
    if not _NUMBER.fullmatch(tok):
        return None
    v = float(tok)
    # from_chars reports result_out_of_range on overflow and on underflow past
    # the smallest subnormal (the value rounds to zero from a non-zero input)
    if math.isinf(v):
        return None
    if v == 0.0 and any(c in "123456789" for c in tok.split("e")[0].split("E")[0]):
        return None
    return v


def load_series(path) -> np.ndarray:
    """io.cpp:17-42 -- whitespace-delimited text -> validated float64 array."""
    p = os.fspath(path)
    try:
        with open(p, "rb") as f:
            text = f.read().decode("latin-1")
    except OSError:
        raise SeriesFileError(f"cannot open '{p}'") from None
    out = []
    # operator>> splits on the C locale's isspace set only (not on the
    # latin-1 bytes Python's str.split() also treats as whitespace)
    for index, tok in enumerate((t for t in _CSPACE.split(text) if t), start=1):
        v = _parse_token(tok)
        if v is None:
            raise SeriesFileError(f"'{p}': token {index} ('{tok}') is not a number")
        if not math.isfinite(v):
            raise SeriesFileError(f"'{p}': token {index} is not finite")
        out.append(v)
    if not out:
        raise SeriesFileError(f"'{p}': empty series file")
    return np.asarray(out, dtype=np.float64)


def save_series(s, path) -> None:
    """io.cpp:44-48"""
    p = os.fspath(path)
    try:
        with open(p, "w") as f:
            for v in np.asarray(s, dtype=np.float64).tolist():
                f.write(format_double(v) + "\n")
    except OSError:
        raise SeriesFileError(f"cannot write '{p}'") from None


def is_binary_path(path) -> bool:
    return os.fspath(path).endswith((".f64", ".bin", ".npy"))


def load_series_binary(path, *, mmap: bool = False) -> np.ndarray:
    """Raw little-endian float64 (.f64/.bin) or .npy, validated like load_series
    (non-empty, every sample finite). ``mmap`` maps the file instead of reading
    it (the search copies it to HBM once either way)."""
    p = os.fspath(path)
    try:
        if p.endswith(".npy"):
            a = np.load(p, mmap_mode="r" if mmap else None)
            if a.ndim != 1 or a.dtype != np.float64:
                raise SeriesFileError(f"'{p}': expected a 1-D float64 array")
        else:
            if os.path.getsize(p) % 8:
                raise SeriesFileError(f"'{p}': size is not a multiple of 8 bytes")
            a = (np.memmap(p, dtype="<f8", mode="r") if mmap and os.path.getsize(p)
                 else np.fromfile(p, dtype="<f8"))
    except OSError:
        raise SeriesFileError(f"cannot open '{p}'") from None
    if a.size == 0:
        raise SeriesFileError(f"'{p}': empty series file")
    bad = np.flatnonzero(~np.isfinite(a[:]))
    if bad.size:
        raise SeriesFileError(f"'{p}': sample {int(bad[0]) + 1} is not finite")
    return a


def save_series_binary(s, path) -> None:
    a = np.ascontiguousarray(s, dtype="<f8")
    if os.fspath(path).endswith(".npy"):
        np.save(path, a)
    else:
        a.tofile(path)


def read_series(path, *, mmap: bool = False) -> np.ndarray:
    """Text or binary by extension."""
    return load_series_binary(path, mmap=mmap) if is_binary_path(path) else load_series(path)
