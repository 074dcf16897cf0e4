import numpy as np, os
from paper_2509_01416_b200 import operators as OPS, snop, workloads as W
from tests import oracle_lib as O
prm = OPS.deeponet_init(2000, width=128, activation=OPS.TANH)
g = snop.Grid1D(10.0, 2000)
op = snop.SolutionOperator.deeponet(g, prm)
oo = O.OracleOperator.deeponet(10.0, 2000, (1.0, 0.5), OPS.TANH, prm.branch.sizes, prm.branch.packed(), prm.trunk.sizes, prm.trunk.packed())
s = W.config2(batch=16).source * np.random.default_rng(1).uniform(0.5, 1.5, (16, 1))
a, b = op.predict(s), oo.predict(s)
print(os.environ.get("SNOP_GEMM"), "max|ref|", np.abs(b).max(), "maxerr", np.abs(a-b).max(), "rel", np.abs(a-b).max()/np.abs(b).max())
