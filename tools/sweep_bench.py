"""Device-resident timing of the standalone sweep (snop_sweep_batched) at the BASELINE sizes:
ms per sweep and achieved HBM GB/s (16 B per cell.angle update + 8 B per cell of Sigma_t).
Usage: python tools/sweep_bench.py [c2|c5 ...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2509_01416_b200 import snop

ctx = snop.default_context()
import os
if os.environ.get("L2_FETCH"):  # experiment: cudaLimitMaxL2FetchGranularity (0x05)
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12")
    print("cudaDeviceSetLimit ->", rt.cudaDeviceSetLimit(5, ctypes.c_size_t(int(os.environ["L2_FETCH"]))))
    v = ctypes.c_size_t()
    rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
    print("MaxL2FetchGranularity =", v.value)
for name in sys.argv[1:] or ["c2", "c5"]:
    B, Nc, N = (2048, 2000, 32) if name == "c2" else (4096, 1024, 16)
    gen = torch.Generator(device="cuda").manual_seed(1)
    st = torch.rand((B, Nc), generator=gen, device="cuda", dtype=torch.float64) + 0.5
    em = torch.rand((B, Nc, N), generator=gen, device="cuda", dtype=torch.float64)
    g = snop.Grid1D(10.0, Nc)
    ext = torch.cuda.ExternalStream(ctx.stream_ptr)
    for bc in ((0, 0), (1, 0)):
        for _ in range(3):
            snop.sweep(g, N, st, em, *bc)
        ts = []
        R = 8  # calls per timed region: the host prepares call i+1 while the device runs call i
        for _ in range(5):
            with torch.cuda.stream(ext):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                snop.sweep(g, N, st, em, *bc, sync=False)
                e0.record()
                for _ in range(R):
                    snop.sweep(g, N, st, em, *bc, sync=False)
                e1.record()
            ctx.synchronize()
            ts.append(e0.elapsed_time(e1) / R)
        ms = sorted(ts)[len(ts) // 2]
        byts = B * Nc * (16.0 * N + 8.0)
        print(f"{name} bc={bc}: {ms:.3f} ms/sweep, {B*Nc*N/ms/1e6:.1f} G updates/s, {byts/ms/1e6:.0f} GB/s", flush=True)
