"""CPU: the C-ABI library loads, exports every symbol include/eapdtw_b200.h
declares, and refuses to compute without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "eapdtw_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eapdtw_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_2010_05371_b200 import _capi
    syms = declared_symbols()
    assert len(syms) >= 25
    lib = C.CDLL(_capi.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes signature table covers the whole header
    assert sorted(n for n, _, _ in _capi.SIGNATURES) == syms


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2010_05371_b200 import Context, EapdtwError
    with pytest.raises(EapdtwError):
        Context(0)


def test_series_validation():
    from paper_2010_05371_b200 import Series
    with pytest.raises(ValueError):
        Series([])
    with pytest.raises(ValueError):
        Series([1.0, float("nan")])
    with pytest.raises(ValueError):
        Series([1.0, float("inf")])
    assert Series([0.0]).length() == 1
    with pytest.raises(ValueError):
        Series([1.0, 2.0]).prefix(0)


def test_window_cells_and_generators():
    from paper_2010_05371_b200 import random_walk_normal, window_cells_for
    assert window_cells_for(0.1, 128) == 12
    assert window_cells_for(0.2, 1024) == 204  # SURVEY.md section 7, hard part 6
    assert window_cells_for(205 / 1024, 1024) == 205
    assert window_cells_for(0.0, 10) == 0
    x = random_walk_normal(10000, 1)
    assert x[0] == 0.0
    d = np.diff(x)
    assert abs(d.mean()) < 0.05 and abs(d.std() - 1.0) < 0.05
    assert np.array_equal(x, random_walk_normal(10000, 1))


def test_oracle_not_imported_by_product():
    """The product package must never load the oracle."""
    import subprocess
    import sys
    code = ("import sys, paper_2010_05371_b200 as p; "
            "assert not any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules); "
            "print('ok')")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2010_05371_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text and "libeapdtw_ref" not in text, f
