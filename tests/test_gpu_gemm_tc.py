"""The tcgen05 3xTF32 GEMM engine vs the FFMA fp32 GEMM and an fp64 torch reference, across
shapes, ragged edges, transposed (MN-major) operands, batch folding and epilogues."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2509_01416_b200 import _capi
    lib = _capi.load()
    f = lib.snop_internal_gemm_test
    f.restype = C.c_int
    f.argtypes = [C.c_int] * 5 + [C.c_void_p] + [C.c_longlong] * 3 + [C.c_void_p] + [C.c_longlong] * 3 + \
                 [C.c_void_p] + [C.c_longlong] * 3 + [C.c_void_p, C.c_float, C.c_float, C.c_int, C.c_longlong]
    return f


def _run(engine, M, N, K, batch, A, sa, B, sb, Cshape, sc, bias=None, alpha=1.0, beta=0.0, act=3, C0=None,
         mfold=0):
    import torch
    Ct = (C0.clone() if C0 is not None else torch.zeros(Cshape, dtype=torch.float32, device="cuda"))
    rc = _lib()(engine, M, N, K, batch, A.data_ptr(), *sa, B.data_ptr(), *sb, Ct.data_ptr(), *sc,
                None if bias is None else bias.data_ptr(), alpha, beta, act, mfold)
    assert rc == 0
    return Ct


@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (256, 128, 128), (300, 100, 70), (4096, 32, 1024),
                                   (1000, 64, 96), (129, 17, 5)])
def test_tc_matches_fp64_reference(M, N, K):
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    ref = (A.double() @ B.double().T)
    tc = _run(1, M, N, K, 1, A, (K, 1, 0), B, (K, 1, 0), (M, N), (N, 1, 0))
    ff = _run(0, M, N, K, 1, A, (K, 1, 0), B, (K, 1, 0), (M, N), (N, 1, 0))
    scale = ref.abs().max().item()
    err_tc = (tc.double() - ref).abs().max().item() / scale
    err_ff = (ff.double() - ref).abs().max().item() / scale
    assert err_tc < 2e-6, err_tc          # 3xTF32: fp32-class
    assert err_tc < 10 * err_ff + 1e-7


def test_tc_transposed_batched_bias_act_beta():
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    Bt, M, N, K = 5, 200, 64, 48
    A = torch.randn(Bt, K, M, device="cuda", generator=g)   # MN-major A: A(b,m,k) = A[b][k][m]
    Bm = torch.randn(Bt, N, K, device="cuda", generator=g)
    bias = torch.randn(N, device="cuda", generator=g)
    C0 = torch.randn(Bt, M, N, device="cuda", generator=g)
    ref = torch.einsum("bkm,bnk->bmn", A.double(), Bm.double()) * 0.5 + 0.75 * C0.double() + bias.double()
    ref = torch.nn.functional.gelu(ref)
    out = _run(1, M, N, K, Bt, A, (1, M, K * M), Bm, (K, 1, N * K), (Bt, M, N), (N, 1, M * N), bias=bias,
               alpha=0.5, beta=0.75, act=2, C0=C0)
    assert (out.double() - ref).abs().max().item() / ref.abs().max().item() < 2e-6


def test_tc_batch_folded_into_m():
    # FNO forward DFT shape: rows = (sample, channel), A(b,c,i) = V[b][i][c]
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    Bt, n, Cc, M2 = 6, 256, 64, 32
    V = torch.randn(Bt, n, Cc, device="cuda", generator=g)
    F = torch.randn(M2, n, device="cuda", generator=g)
    ref = torch.einsum("bic,mi->bcm", V.double(), F.double())
    out = _run(1, Bt * Cc, M2, n, 1, V, (1, Cc, n * Cc), F, (n, 1, 0), (Bt, Cc, M2), (M2, 1, Cc * M2),
               mfold=Cc)
    assert (out.double() - ref).abs().max().item() / ref.abs().max().item() < 2e-6


@pytest.mark.parametrize("M,N,K,batch", [(128, 64, 32, 1), (256, 128, 128, 1), (300, 100, 64, 1), (1000, 64, 96, 1),
                                         (1024, 64, 96, 3), (131, 33, 32, 2)])
def test_tc2_matches_tc_and_fp64(M, N, K, batch):
    """The TMA-fed warp-specialised engine (K-contiguous operands, K <= 128) against the original
    tcgen05 engine and an fp64 reference, with per-sample batch strides, bias and GELU."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M + 13 * K + batch)
    A = torch.randn(batch, M, K, device="cuda", generator=g)
    B = torch.randn(batch, N, K, device="cuda", generator=g)
    bias = torch.randn(N, device="cuda", generator=g)
    sa, sb, sc = (K, 1, M * K), (K, 1, N * K), (N, 1, M * N)
    c2 = _run(2, M, N, K, batch, A, sa, B, sb, (batch, M, N), sc, bias=bias, act=2)
    c1 = _run(1, M, N, K, batch, A, sa, B, sb, (batch, M, N), sc, bias=bias, act=2)
    x = torch.einsum("bmk,bnk->bmn", A.double(), B.double()) + bias.double()
    ref = 0.5 * x * (1 + torch.erf(x / np.sqrt(2.0)))
    scale = ref.abs().max().item()
    assert (c2.double() - ref).abs().max().item() / scale < 2e-6
    assert (c2 - c1).abs().max().item() / scale < 1e-6
