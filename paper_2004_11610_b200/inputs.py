"""Seeded synthetic inputs shared by the tests, the oracle and bench.py.

This module holds none of the method's arithmetic: only the workload shapes of
BASELINE.json's configs and numpy PCG64 draws.
Gauss nodes are NOT generated here: the tests take them from the oracle, the
product computes its own (``xc.gauss_rule``).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KIND_COS, KIND_JACOBI, KIND_LAGUERRE, KIND_EXP, KIND_LAGSPEC, KIND_LAG2D = 1, 2, 3, 4, 5, 6


@dataclass(frozen=True)
class Config:
    name: str
    kind: int
    N: int
    B: int
    eps: float
    seed: int
    alpha: float = 0.0
    beta: float = 0.0
    dirs: tuple = ("A",)
    eps2: float = 1e-2
    M: int = 0          # degrees (rows) when != N (complex kinds); 0 = square
    eta: float = 0.0    # LAGSPEC: Laguerre scale eta
    T: float = 0.0      # LAGSPEC: Fourier period, frequencies k_j = 2 pi j / T


CONFIGS = {
    # BASELINE.json configs[0..4]; see DESIGN.md for the readings (R2 for c2, C-15 for c4)
    "c1": Config("c1_legendre_512", KIND_JACOBI, 512, 1, 1e-12, 0),
    "c2": Config("c2_noncos_4096", KIND_COS, 4096, 64, 1e-10, 1),
    "c3": Config("c3_jacobi_16384", KIND_JACOBI, 16384, 256, 1e-12, 2, alpha=0.5, beta=-0.3),
    "c4": Config("c4_laguerre_8192", KIND_LAGUERRE, 8192, 256, 1e-11, 3, dirs=("A", "WAT")),
    "c5": Config("c5_legendre_65536", KIND_JACOBI, 65536, 4096, 1e-12, 4),
    # NEXT-3: the complex exponential kind, non-uniform DFT e^{i pi j t_k}, t_k in [0,2);
    # not a BASELINE config -- a parity / measurement case of the widened path
    "c6": Config("c6_nonexp_4096", KIND_EXP, 4096, 64, 1e-10, 6),
    # NEXT-3 second half: the spectral Laguerre forward V = C^T F at the sizes of the paper's
    # Fig. lag_row: C^T is 649 x 501, eta = 2500, k_j = 2 pi j / T, T = 4 s
    "c7": Config("c7_lagspec_649x501", KIND_LAGSPEC, 501, 64, 1e-10, 7, M=649, eta=2500.0, T=4.0),
    # NEXT-1: the time-domain Laguerre series sum D c, D[i,j] = l_j(eta t_i), t_i = 12 i / (N-1)
    # (P:528), by the 2D block method; eps2 = 0.1 (R-23: errors pass two window divisions)
    "c8": Config("c8_lag2d_4096", KIND_LAG2D, 4096, 256, 1e-10, 8, eps2=0.1, eta=100.0),
    # off the configured lengths (c5's kind and batch at half and twice N): the generic C2R
    # passes, no length-specialised kernel -- a check for performance cliffs (not BASELINE configs)
    "c5n32k": Config("legendre_32768", KIND_JACOBI, 32768, 4096, 1e-12, 12),
    "c5n128k": Config("legendre_131072", KIND_JACOBI, 131072, 4096, 1e-12, 13),
}


def cos_nodes(N: int, seed: int) -> np.ndarray:
    """Non-uniform cosine nodes t_k = sort(U[0,1]) (first draw of the seed; c2 reading R2)."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.random(N))


def exp_nodes(N: int, seed: int) -> np.ndarray:
    """Non-uniform DFT nodes t_k = sort(U[0,2)) (theta_k = pi t_k on the whole circle)."""
    rng = np.random.default_rng(seed)
    return 2.0 * np.sort(rng.random(N))


def lagspec_freqs(N: int, T: float) -> np.ndarray:
    """Fourier frequencies k_j = 2 pi j / T, j = 0..N-1 (Fig. lag_row caption); no draw."""
    return 2.0 * np.pi * np.arange(N, dtype=np.float64) / T


def lag2d_grid(N: int, eta: float) -> np.ndarray:
    """x_i = eta t_i, t_i = 12 i / (N - 1), i = 1..N; no draw."""
    return eta * 12.0 * np.arange(1, N + 1, dtype=np.float64) / (N - 1)


def complex_rhs(N: int, B: int, seed: int, skip_nodes: bool = True) -> np.ndarray:
    """X = N(0,1) + i N(0,1) (complex128, N x B); the node draw first when skip_nodes."""
    rng = np.random.default_rng(seed)
    if skip_nodes:
        rng.random(N)
    re = rng.standard_normal((N, B))
    return re + 1j * rng.standard_normal((N, B))


def rhs(N: int, B: int, seed: int, skip_cos_nodes: bool = False) -> np.ndarray:
    """X ~ N(0,1), row-major N x B (RHS fastest).  For the cos config the node
    draw comes first from the same stream (skip_cos_nodes=True)."""
    rng = np.random.default_rng(seed)
    if skip_cos_nodes:
        rng.random(N)
    return rng.standard_normal((N, B))


def laguerre_coeffs(N: int, B: int, seed: int) -> np.ndarray:
    """C[j,b] = N(0,1) / (1+j)^2 (BASELINE.json configs[3])."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((N, B)) / (1.0 + np.arange(N, dtype=np.float64))[:, None] ** 2


def config_rhs(cfg: Config, B: int | None = None) -> np.ndarray:
    B = cfg.B if B is None else B
    if cfg.kind == KIND_EXP:
        return complex_rhs(cfg.N, B, cfg.seed)
    if cfg.kind == KIND_LAGSPEC:  # Fourier coefficients F~ (no node draw: the k_j are a grid)
        return complex_rhs(cfg.N, B, cfg.seed, skip_nodes=False)
    if cfg.kind == KIND_COS:
        return rhs(cfg.N, B, cfg.seed, skip_cos_nodes=True)
    if cfg.kind == KIND_LAGUERRE:
        return laguerre_coeffs(cfg.N, B, cfg.seed)
    return rhs(cfg.N, B, cfg.seed)
