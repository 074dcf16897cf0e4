"""Seeded synthetic workloads C1-C5 (repo BASELINE.json ``configs``, made concrete in SURVEY.md
§8d / §9). Generated once on the host with the reference's RNG stream (rng.py restating
rng.hpp:17-49), one stream per instance ``Rng(seed_base + b)`` (stream split as SPEC.md:263),
and passed identically to the CUDA path and to the CPU oracle.

The paper's own profiles (§5.1 Case 3 sinusoids, §5.2 Case 3 from Nease et al.) exist only as
figures; these seeded parametric profiles stand in for them.
Arrays are row-major fp64: per-cell ``[B][Nc]``, multigroup ``[B][G][Nc]``, scattering
``[B][G][G][Nc]`` with entry ``[b][g'][g][i] = Sigma_s0^{g'->g}``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .rng import Rng

L_CM = 10.0  # slab width for C2-C5


@dataclass
class FixedSourceProblem:
    name: str
    length: float
    n_cells: int
    order: int
    sigma_t: np.ndarray
    sigma_s0: np.ndarray
    source: np.ndarray
    sigma_s1: np.ndarray | None = None
    bc_left: int = 0
    bc_right: int = 0
    tolerance: float = 1e-8
    max_inner: int = 10000
    ref_params: tuple[float, float] = (1.0, 0.5)  # p* = (Sigma_t*, Sigma_s0*)

    @property
    def batch(self) -> int:
        return self.sigma_t.shape[0]

    def subset(self, idx) -> "FixedSourceProblem":
        idx = np.asarray(idx)
        return FixedSourceProblem(
            self.name, self.length, self.n_cells, self.order, self.sigma_t[idx].copy(),
            self.sigma_s0[idx].copy(), self.source[idx].copy(),
            None if self.sigma_s1 is None else self.sigma_s1[idx].copy(),
            self.bc_left, self.bc_right, self.tolerance, self.max_inner, self.ref_params)


@dataclass
class EigenProblem:
    name: str
    length: float
    n_cells: int
    order: int
    n_groups: int
    sigma_t: np.ndarray       # [B][G][Nc]
    sigma_s0: np.ndarray      # [B][G][G][Nc]
    nu_sigma_f: np.ndarray    # [B][G][Nc]
    chi: np.ndarray           # [B][G]
    sigma_s1: np.ndarray | None = None
    bc_left: int = 0
    bc_right: int = 0
    tolerance_k: float = 1e-8
    tolerance_phi: float = 1e-7
    tolerance_inner: float = 1e-7
    max_inner: int = 10000
    max_outer: int = 5000

    @property
    def batch(self) -> int:
        return self.sigma_t.shape[0]

    def subset(self, idx) -> "EigenProblem":
        idx = np.asarray(idx)
        return EigenProblem(
            self.name, self.length, self.n_cells, self.order, self.n_groups, self.sigma_t[idx].copy(),
            self.sigma_s0[idx].copy(), self.nu_sigma_f[idx].copy(), self.chi[idx].copy(),
            None if self.sigma_s1 is None else self.sigma_s1[idx].copy(), self.bc_left, self.bc_right,
            self.tolerance_k, self.tolerance_phi, self.tolerance_inner, self.max_inner, self.max_outer)


def centers(length: float, n_cells: int) -> np.ndarray:
    dx = length / n_cells
    return (np.arange(n_cells) + 0.5) * dx


def _sinusoid_sigma_t(rng: Rng, x: np.ndarray, length: float) -> np.ndarray:
    a = rng.uniform(0.8, 1.5)
    b = rng.uniform(0.0, 0.5)
    f = 1 + int(math.floor(4.0 * rng.uniform()))
    return a * (1.0 + b * np.sin(2.0 * math.pi * f * x / length))


def _regions(rng: Rng, x: np.ndarray, length: float) -> np.ndarray:
    """4 sorted U(0,L) interfaces -> region index (0..4) of every cell centre."""
    cuts = np.sort(np.array([rng.uniform(0.0, length) for _ in range(4)]))
    return np.searchsorted(cuts, x, side="left")


def config1() -> FixedSourceProblem:
    """C1: 1 x 1000 cells, S16, St=1, Ss=0.5, q=1, vacuum, tol 1e-8 (BASELINE configs[0])."""
    n = 1000
    return FixedSourceProblem("C1", 10.0, n, 16, np.full((1, n), 1.0), np.full((1, n), 0.5),
                              np.full((1, n), 1.0), tolerance=1e-8)


def config2(batch: int = 2048, n_cells: int = 2000, seed: int = 2000) -> FixedSourceProblem:
    """C2: batched parametric sinusoidal St(x)=a(1+b sin(2 pi f x/L)), Ss=c St, q=1, S32, vacuum.
    Draw order per instance: a~U[0.8,1.5], b~U[0,0.5], f=1+floor(4u), c~U[0.5,0.95]."""
    x = centers(L_CM, n_cells)
    st = np.empty((batch, n_cells))
    ss = np.empty((batch, n_cells))
    for b in range(batch):
        r = Rng(seed + b)
        st[b] = _sinusoid_sigma_t(r, x, L_CM)
        ss[b] = r.uniform(0.5, 0.95) * st[b]
    return FixedSourceProblem("C2", L_CM, n_cells, 32, st, ss, np.ones((batch, n_cells)),
                              tolerance=1e-8, ref_params=(1.0, 0.5))


def config3(batch: int = 512, n_cells: int = 4096, seed: int = 3000) -> EigenProblem:
    """C3: single-group k-eigenvalue, 5 seeded regions; per region St~U[0.5,2], c~U[0.3,0.9],
    fissile flag u<1/2 with nuSf~U[0,0.3] (>=1 fissile forced); S32;
    reflective left / vacuum right; tol_k 1e-8, tol_phi = inner tol = 1e-7.
    Draw order: 4 interfaces; per region (St, c, flag-u, nuSf-u); if none fissile: region floor(5u)."""
    x = centers(L_CM, n_cells)
    st = np.empty((batch, 1, n_cells))
    ss = np.empty((batch, 1, 1, n_cells))
    nsf = np.empty((batch, 1, n_cells))
    for b in range(batch):
        r = Rng(seed + b)
        reg = _regions(r, x, L_CM)
        rst, rc, rnf, fis = [], [], [], []
        for _ in range(5):
            rst.append(r.uniform(0.5, 2.0))
            rc.append(r.uniform(0.3, 0.9))
            fis.append(r.uniform() < 0.5)
            rnf.append(r.uniform(0.0, 0.3))
        if not any(fis):
            fis[int(math.floor(5.0 * r.uniform()))] = True
        rst, rc = np.array(rst), np.array(rc)
        rnf = np.array([v if f else 0.0 for v, f in zip(rnf, fis)])
        st[b, 0] = rst[reg]
        ss[b, 0, 0] = (rc * rst)[reg]
        nsf[b, 0] = rnf[reg]
    return EigenProblem("C3", L_CM, n_cells, 32, 1, st, ss, nsf, np.ones((batch, 1)),
                        bc_left=1, bc_right=0, tolerance_k=1e-8, tolerance_phi=1e-7, tolerance_inner=1e-7)


THERMAL = (4, 5, 6)  # groups 5-7 (0-based) carry upscatter in C4


def config4(batch: int = 128, n_cells: int = 2000, groups: int = 7, seed: int = 4000) -> EigenProblem:
    """C4: G=7 coupled k-eigenvalue, S16, vacuum. Per instance & group constants:
    St,g~U[0.2,2]; per source group g a scattering ratio rho_g~U[0.5,0.95] split over allowed
    destinations (down-scatter g'>=g, plus up-scatter inside the thermal groups 5-7) with U[0,1]
    weights, so row sums = rho_g St,g < St,g; nuSf,g~U[0,0.2]; chi on groups 1-3, sum 1.
    Draw order: St[0..G-1]; per g: rho_g then weights for allowed g' ascending; nuSf[0..G-1];
    chi raw[0..2]."""
    G = groups
    st = np.empty((batch, G, n_cells))
    ss = np.zeros((batch, G, G, n_cells))
    nsf = np.empty((batch, G, n_cells))
    chi = np.zeros((batch, G))
    for b in range(batch):
        r = Rng(seed + b)
        sig_t = np.array([r.uniform(0.2, 2.0) for _ in range(G)])
        mat = np.zeros((G, G))
        for g in range(G):
            rho = r.uniform(0.5, 0.95)
            dest = [gp for gp in range(G) if gp >= g or (g in THERMAL and gp in THERMAL)]
            w = np.array([r.uniform() for _ in dest])
            if w.sum() <= 0.0:
                w[:] = 1.0
            mat[g, dest] = rho * sig_t[g] * w / w.sum()
        nu = np.array([r.uniform(0.0, 0.2) for _ in range(G)])
        c = np.array([r.uniform() for _ in range(3)])
        if c.sum() <= 0.0:
            c[:] = 1.0
        chi[b, :3] = c / c.sum()
        st[b] = sig_t[:, None]
        ss[b] = mat[:, :, None]
        nsf[b] = nu[:, None]
    return EigenProblem("C4", L_CM, n_cells, 16, G, st, np.broadcast_to(ss, ss.shape).copy(), nsf, chi,
                        bc_left=0, bc_right=0, tolerance_k=1e-8, tolerance_phi=1e-7, tolerance_inner=1e-7)


def config5(batch: int = 4096, n_cells: int = 1024, seed: int = 5000) -> FixedSourceProblem:
    """C5: MD-PNOP warm start, S16, q=1, c=0.8, p*=(1.0, 0.8); even instances sinusoidal St (as
    C2: a, b, f draws), odd instances 5-region step St (4 interfaces + 5 St~U[0.5,2])."""
    x = centers(L_CM, n_cells)
    st = np.empty((batch, n_cells))
    for b in range(batch):
        r = Rng(seed + b)
        if b % 2 == 0:
            st[b] = _sinusoid_sigma_t(r, x, L_CM)
        else:
            reg = _regions(r, x, L_CM)
            st[b] = np.array([r.uniform(0.5, 2.0) for _ in range(5)])[reg]
    return FixedSourceProblem("C5", L_CM, n_cells, 16, st, 0.8 * st, np.ones((batch, n_cells)),
                              tolerance=1e-8, ref_params=(1.0, 0.8))


def three_group_table9(n_cells: int = 100, length: float = 10.0, bc: int = 0) -> EigenProblem:
    """Paper Tables 7-8: 3-group constants. Table 7 rows = source g,
    columns = destination g', i.e. exactly our [g'->g] storage order."""
    G = 3
    table7 = np.array([[0.024, 0.171, 0.033], [0.000, 0.600, 0.275], [0.000, 0.000, 2.000]])
    nu = np.array([3.0, 2.5, 2.0])
    sig_t = np.array([0.240, 0.975, 3.000])
    sig_f = np.array([0.006, 0.060, 0.900])
    chi = np.array([0.96, 0.04, 0.00])
    st = np.broadcast_to(sig_t[None, :, None], (1, G, n_cells)).copy()
    ss = np.broadcast_to(table7[None, :, :, None], (1, G, G, n_cells)).copy()
    nsf = np.broadcast_to((nu * sig_f)[None, :, None], (1, G, n_cells)).copy()
    return EigenProblem("T9", length, n_cells, 32, G, st, ss, nsf, chi[None, :].copy(), bc_left=bc,
                        bc_right=bc, tolerance_k=1e-8, tolerance_phi=1e-7, tolerance_inner=1e-7)
