"""The reference's own acceptance suite (proj/tests/acceptance.cpp, criteria
1-9 of SPEC.md:449-459), compiled unmodified against the B200 C++ shim
(include/compat/eapdtw/*.hpp -> include/eapdtw_b200.hpp) and linked with
libeapdtw_b200.so by oracle/Makefile's `acceptance` target (built where
/root/reference exists; the binary travels to the GPU box).  Every criterion
must print PASS on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "acceptance_gpu")


@pytest.mark.gpu
@pytest.mark.timeout(1200)
@pytest.mark.skipif(not os.path.exists(EXE), reason="acceptance_gpu not built (needs /root/reference)")
def test_reference_acceptance_suite_on_gpu():
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=1200)
    lines = [l for l in out.stdout.splitlines() if l.startswith("criterion")]
    print(out.stdout)
    assert len(lines) == 9, out.stdout + out.stderr
    failed = [l for l in lines if "[PASS]" not in l]
    assert not failed, "\n".join(failed)
    assert out.returncode == 0
