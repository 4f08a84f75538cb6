"""Seeded synthetic inputs shared by the product tests, the bench and the oracle checks.

This module holds NO arithmetic of the REXI method: it only samples the paper's
initial conditions on the grid and draws seeded random fields. Both the CUDA
path and the oracle consume its arrays; neither side's numbers come from the
other.

Grid: x_j = j / D, y_m = m / D on the bi-periodic unit square;
arrays are indexed [y, x] (x fastest), float64.
"""
from __future__ import annotations

import numpy as np

PARITY_SEED = 2008116070   # PCG64 seed + field index


def grid(D):
    x = np.arange(D, dtype=np.float64) / D
    Y, X = np.meshgrid(x, x, indexing="ij")
    return X, Y


def gaussian_scenario(D):
    """eq:GAUSSIANSCENARIO."""
    X, Y = grid(D)
    eta = np.exp(-100.0 * ((X - 0.5) ** 2 + (Y - 0.5) ** 2))
    u = 0.1 * np.sin(64.0 * np.pi * X) * np.sin(16.0 * np.pi * Y)
    v = 0.1 * np.sin(32.0 * np.pi * X) * np.sin(32.0 * np.pi * Y)
    return eta, u, v


def wave_scenario_1(D):
    """eq:WAVESCENARIO1."""
    X, Y = grid(D)
    p = np.pi
    eta = np.sin(4 * p * X) * np.cos(2 * p * Y) - 0.2 * np.cos(4 * p * X) * np.sin(4 * p * Y)
    u = np.cos(8 * p * X) * np.cos(2 * p * Y)
    v = np.cos(4 * p * X) * np.cos(4 * p * Y)
    return eta, u, v


def wave_scenario_2(D):
    """eq:WAVESCENARIO2."""
    X, Y = grid(D)
    p = np.pi
    eta = np.sin(32 * p * X) * np.cos(16 * p * Y) - 0.2 * np.cos(32 * p * X) * np.sin(32 * p * Y)
    u = np.cos(64 * p * X) * np.cos(16 * p * Y)
    v = np.cos(32 * p * X) * np.cos(32 * p * Y)
    return eta, u, v


def white_noise(D, seed=PARITY_SEED):
    """i.i.d. N(0,1) real eta, u, v (PCG64, seed + field index): excites every mode."""
    return tuple(np.random.Generator(np.random.PCG64(seed + i)).standard_normal((D, D))
                 for i in range(3))


def spectral_white(D, seed=PARITY_SEED):
    """Seeded complex N(0,1) spectra (3, D, D) — input for the spectral pole-sum call,
    which is linear per mode and needs no Hermitian symmetry."""
    g = np.random.Generator(np.random.PCG64(seed + 7))
    z = g.standard_normal((3, D, D, 2))
    return z[..., 0] + 1j * z[..., 1]


def sample_modes(D, n, seed=PARITY_SEED):
    """Deterministic sample of n distinct (l, k) mode indices, always including the
    degenerate K = 0 modes (0,0), (0,D/2), (D/2,0), (D/2,D/2), the highest |k| corner
    and a few on the Nyquist row/column."""
    D2 = D // 2
    must = [(0, 0), (0, D2), (D2, 0), (D2, D2), (D2 - 1, D2 - 1), (D2 + 1, D2 + 1),
            (0, 1), (1, 0), (D2, 3 % D), (5 % D, D2), (D - 1, D - 1)]
    g = np.random.Generator(np.random.PCG64(seed + 99))
    total = D * D
    n = min(n, total)
    pick = set(l * D + k for l, k in must)
    if n >= total:
        flat = np.arange(total)
    else:
        while len(pick) < n:
            for x in g.integers(0, total, size=n):
                pick.add(int(x))
                if len(pick) >= n:
                    break
        flat = np.array(sorted(pick))
    return (flat // D).astype(np.int32), (flat % D).astype(np.int32)


def spectral_hermitian(D, seed=PARITY_SEED):
    """Seeded Hermitian spectra (3, D, D): F(K) = (Z(K) + conj Z(-K)) / 2 for the complex white
    spectra Z of spectral_white, so F(-K) = conj F(K) exactly (the spectrum of real fields,
    input of rexi_poles_real) — without a transform (no O(D^3) DFT at large D)."""
    Z = spectral_white(D, seed)
    j = (-np.arange(D)) % D
    return 0.5 * (Z + np.conj(Z[:, j][:, :, j]))
