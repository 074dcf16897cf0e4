"""Randomised differential test of the fused solvers (K1 fixed source incl. P1 / both norms / warm
starts, K2 single- and multigroup with upscatter) and the standalone sweep against the CPU oracle:
seeded random sizes around every CTA-size boundary (1 ... 5000 cells), orders 2 ... 64, all boundary
combinations, thin cells, at fixed iteration counts so fluxes and k must agree at 1e-10
(tools/fuzz_parity.py; 3000 cases with other seeds were run clean during development)."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [11, 12])
def test_random_cases_match_the_oracle(seed):
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "fuzz_parity.py"), "150", str(seed)],
                         capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "150 cases ok" in out.stdout


@pytest.mark.gpu
def test_random_md_pnop_cases_match_the_oracle():
    """recast_fixed_point / precondition_fixed_source / cp_eigen with the exact operator on random
    small problems (statuses, counts +-1, fields) - tools/fuzz_mdpnop.py; 720 further cases run clean."""
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "fuzz_mdpnop.py"), "40", "21"],
                         capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "40 cases, 0 mismatches" in out.stdout


@pytest.mark.gpu
def test_random_operator_shapes_match_the_oracle():
    """DeepONet / FNO forwards over random shapes (the GEMM engines' tile edges): within 1e-5 of the
    output max, or - random networks whose output nearly cancels - within 5x the exact-fp32 engines'
    error on the same case (tools/fuzz_operators.py)."""
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "fuzz_operators.py"), "80", "31"],
                         capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert " 0 failures" in out.stdout
