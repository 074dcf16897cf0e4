"""Seeded random-init neural-operator parameters (BASELINE C2/C5) and their
packed fp32 layouts for the C-ABI (include/snop_cuda.h).

Init conventions: Xavier-uniform weights W ~ U(-a, a),
a = sqrt(6/(fan_in + fan_out)), zero biases; FNO complex spectral weights
R = (1/(C_in C_out)) * U[0,1) for real then imaginary parts. Draw order: layer by layer, W row-major
[out][in]; DeepONet branch before trunk; FNO lift, then per layer (R_re, R_im, W), then projection.
All draws from ``Rng(seed)`` (rng.hpp restatement).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rng import Rng

RELU, TANH, GELU = 0, 1, 2


def _xavier(r: Rng, n_in: int, n_out: int) -> np.ndarray:
    a = np.sqrt(6.0 / (n_in + n_out))
    return r.uniform_array(n_in * n_out, -a, a).reshape(n_out, n_in).astype(np.float32)


@dataclass
class DenseParams:
    sizes: list
    weights: list  # [n_out][n_in] fp32
    biases: list   # [n_out] fp32

    def packed(self) -> np.ndarray:
        parts = []
        for W, b in zip(self.weights, self.biases):
            parts += [W.ravel(), b.ravel()]
        return np.concatenate(parts).astype(np.float32)


def dense_init(r: Rng, sizes) -> DenseParams:
    Ws, bs = [], []
    for i in range(len(sizes) - 1):
        Ws.append(_xavier(r, sizes[i], sizes[i + 1]))
        bs.append(np.zeros(sizes[i + 1], dtype=np.float32))
    return DenseParams(list(sizes), Ws, bs)


@dataclass
class DeepONetParams:
    """SPEC.md:300-304 (BASELINE C2: branch Nc->128x4, trunk 1->128x4, p=128, tanh)."""
    branch: DenseParams
    trunk: DenseParams
    activation: int = TANH
    bias0: float | None = None


def deeponet_init(n_cells: int, width: int = 128, depth: int = 4, activation: int = TANH,
                  seed: int = 7) -> DeepONetParams:
    r = Rng(seed)
    branch = dense_init(r, [n_cells] + [width] * depth)
    trunk = dense_init(r, [1] + [width] * depth)
    return DeepONetParams(branch, trunk, activation)


@dataclass
class FNOParams:
    """SPEC.md:306-311 (BASELINE C5: 4 layers, width 64, 16 modes, lift 2->64, proj 64->128->1, GELU)."""
    width: int
    modes: int
    layers: int
    hidden: int
    activation: int
    lift_W: np.ndarray
    lift_b: np.ndarray
    R_re: list
    R_im: list
    W: list
    b: list
    P1_W: np.ndarray
    P1_b: np.ndarray
    P2_W: np.ndarray
    P2_b: np.ndarray

    def packed(self) -> np.ndarray:
        parts = [self.lift_W.ravel(), self.lift_b]
        for l in range(self.layers):
            parts += [self.R_re[l].ravel(), self.R_im[l].ravel(), self.W[l].ravel(), self.b[l]]
        parts += [self.P1_W.ravel(), self.P1_b, self.P2_W.ravel(), self.P2_b]
        return np.concatenate(parts).astype(np.float32)


def fno_init(width: int = 64, modes: int = 16, layers: int = 4, hidden: int = 128, activation: int = GELU,
             seed: int = 11) -> FNOParams:
    r = Rng(seed)
    lift_W = _xavier(r, 2, width)
    lift_b = np.zeros(width, np.float32)
    scale = 1.0 / (width * width)
    R_re, R_im, W, b = [], [], [], []
    for _ in range(layers):
        R_re.append((scale * r.uniform_array(modes * width * width)).reshape(modes, width, width).astype(np.float32))
        R_im.append((scale * r.uniform_array(modes * width * width)).reshape(modes, width, width).astype(np.float32))
        W.append(_xavier(r, width, width))
        b.append(np.zeros(width, np.float32))
    P1_W = _xavier(r, width, hidden)
    P2_W = _xavier(r, hidden, 1)
    return FNOParams(width, modes, layers, hidden, activation, lift_W, lift_b, R_re, R_im, W, b, P1_W,
                     np.zeros(hidden, np.float32), P2_W.reshape(-1), np.zeros(1, np.float32))


def dense_from_packed(sizes, flat) -> DenseParams:
    """Inverse of DenseParams.packed(): per layer W[n_out][n_in] then b[n_out]."""
    flat = np.asarray(flat, dtype=np.float32)
    Ws, bs, off = [], [], 0
    for i in range(len(sizes) - 1):
        n_in, n_out = int(sizes[i]), int(sizes[i + 1])
        Ws.append(flat[off:off + n_in * n_out].reshape(n_out, n_in).copy())
        off += n_in * n_out
        bs.append(flat[off:off + n_out].copy())
        off += n_out
    if off != flat.size:
        raise ValueError("parameter vector length does not match the layer sizes")
    return DenseParams(list(int(s) for s in sizes), Ws, bs)


def fno_from_packed(width, modes, layers, hidden, activation, flat) -> FNOParams:
    """Inverse of FNOParams.packed()."""
    flat = np.asarray(flat, dtype=np.float32)
    C, M, H = int(width), int(modes), int(hidden)
    off = 0

    def take(n, shape=None):
        nonlocal off
        v = flat[off:off + n].copy()
        off += n
        return v.reshape(shape) if shape else v

    lift_W = take(2 * C, (C, 2))
    lift_b = take(C)
    R_re, R_im, W, b = [], [], [], []
    for _ in range(int(layers)):
        R_re.append(take(M * C * C, (M, C, C)))
        R_im.append(take(M * C * C, (M, C, C)))
        W.append(take(C * C, (C, C)))
        b.append(take(C))
    P1_W = take(H * C, (H, C))
    P1_b = take(H)
    P2_W = take(H)
    P2_b = take(1)
    if off != flat.size:
        raise ValueError("parameter vector length does not match the FNO architecture")
    return FNOParams(C, M, int(layers), H, int(activation), lift_W, lift_b, R_re, R_im, W, b, P1_W, P1_b, P2_W, P2_b)
