"""The C-ABI library loads without a GPU and exports every entry point include/snop_cuda.h
declares (no compute calls here)."""
import re
import subprocess
from pathlib import Path

import pytest

from paper_2509_01416_b200 import _capi

ROOT = Path(__file__).resolve().parents[1]


def declared():
    txt = (ROOT / "include" / "snop_cuda.h").read_text()
    rx = r"^(?:snop_status|int32_t|int64_t|const char\*|void\*)\s+(snop_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(rx, txt, flags=re.M)))


def test_header_declares_the_python_export_list():
    assert sorted(_capi.EXPORTS) == declared()


def test_library_exports_every_declared_symbol():
    if not _capi.LIB_PATH.exists():
        pytest.skip("libsnop_cuda.so not built")
    out = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared() if s not in syms]
    assert not missing, missing


def test_library_loads_and_reports_abi_without_gpu():
    if not _capi.LIB_PATH.exists():
        pytest.skip("libsnop_cuda.so not built")
    lib = _capi.load()
    assert lib.snop_abi_version() == 1
    import numpy as np
    mu = np.empty(4)
    w = np.empty(4)
    assert lib.snop_gauss_legendre(4, mu.ctypes.data, w.ctypes.data) == 0  # host-only entry point
    assert abs(w.sum() - 2.0) < 1e-14
    assert lib.snop_gauss_legendre(5, mu.ctypes.data, w.ctypes.data) == 1  # InvalidArgument


def test_host_gauss_legendre_matches_oracle():
    if not _capi.LIB_PATH.exists():
        pytest.skip("libsnop_cuda.so not built")
    from paper_2509_01416_b200 import snop
    from tests import oracle_lib as O
    for n in (2, 8, 16, 32, 64):
        q = snop.gauss_legendre(n)
        mu, w = O.gauss_legendre(n)
        assert np.max(np.abs(q.mu - mu)) < 1e-15 and np.max(np.abs(q.w - w)) < 1e-14


import numpy as np  # noqa: E402
