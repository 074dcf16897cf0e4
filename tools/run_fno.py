import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2509_01416_b200 import operators as OPS, snop, workloads as W
p5 = W.config5(batch=int(sys.argv[1]) if len(sys.argv) > 1 else 4096)
fno = snop.SolutionOperator.fno(snop.Grid1D(10.0, 1024), OPS.fno_init(), (1.0, 0.8))
src = torch.from_numpy(p5.source).cuda()
for _ in range(2):
    out = fno.predict(src)
torch.cuda.synchronize()
print("ok", float(out.abs().max()))
