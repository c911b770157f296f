"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds input generators only -- none of the method's arithmetic.
Both the CPU oracle (``oracle/``) and the CUDA product path consume what it
produces; neither imports the other.

Recipe:
* Taylor-Green lattice (reading Z26): x = lo + (i + 1/2) h, h = L/n, one
  particle per lattice node, alpha = omega_TG(x) h^3, sigma = overlap * h.
  The paper's workload is a uniform particle lattice carrying vorticity
  (P:212 reinitialisation to the same positions; P:243 256^3 per process).
* Tiled Taylor-Green (reading Z27): P_x x P_y x P_z copies of the 2 pi cube,
  one copy per GPU for weak scaling (C5).
* Random clouds: uniform positions (seeds 1106 and 5273 by convention),
  alpha ~ N(0, 1) h^3, used for stress and brute-force cases.
All arrays are float32, the boundary's precision.
"""
from __future__ import annotations

import numpy as np

TWO_PI = 2.0 * np.pi


def omega_tg(x):
    """Vorticity of u_TG = (sin x cos y cos z, -cos x sin y cos z, 0) (Z26)."""
    x = np.asarray(x, dtype=np.float64)
    X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
    return np.stack([-np.cos(X) * np.sin(Y) * np.sin(Z),
                     -np.sin(X) * np.cos(Y) * np.sin(Z),
                     2.0 * np.sin(X) * np.sin(Y) * np.cos(Z)], axis=-1)


def lattice(n: int, lo=-np.pi, L=TWO_PI, tiles=(1, 1, 1)):
    """Cell-centred lattice of n^3 points per tile; tiles extend along +x,+y,+z.

    Ordering: x fastest, then y, then z, then tile (x-fastest)."""
    h = L / n
    c = lo + (np.arange(n, dtype=np.float64) + 0.5) * h
    Z, Y, X = np.meshgrid(c, c, c, indexing="ij")
    base = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=-1)
    out = []
    for tz in range(tiles[2]):
        for ty in range(tiles[1]):
            for tx in range(tiles[0]):
                out.append(base + np.array([tx * L, ty * L, tz * L]))
    return np.concatenate(out, axis=0), h


def taylor_green(n: int, overlap: float = 1.0, lo=-np.pi, L=TWO_PI, tiles=(1, 1, 1)):
    """Taylor-Green vortex particles on an n^3 lattice per tile.

    Returns (x, alpha, sigma) float32 arrays of shapes [N,3], [N,3], [N]."""
    x, h = lattice(n, lo, L, tiles)
    alpha = omega_tg(x) * h ** 3
    sigma = np.full(x.shape[0], overlap * h)
    return (x.astype(np.float32), alpha.astype(np.float32), sigma.astype(np.float32))


def random_cloud(n: int, seed: int = 1106, lo=-np.pi, L=TWO_PI, sigma=None, h=None):
    """Uniform random positions in [lo, lo+L)^3 with alpha ~ N(0,1) h^3."""
    rng = np.random.default_rng(seed)
    x = lo + L * rng.random((n, 3))
    if h is None:
        h = L / max(1.0, round(n ** (1.0 / 3.0)))
    alpha = rng.standard_normal((n, 3)) * h ** 3
    sig = np.full(n, h if sigma is None else sigma)
    return x.astype(np.float32), alpha.astype(np.float32), sig.astype(np.float32)


def jittered_lattice(n: int, seed: int = 5273, lo=-np.pi, L=TWO_PI, overlap=1.0, amp=0.25):
    """Taylor-Green lattice with positions jittered uniformly by +-amp*h
    (amp = 1/4 keeps every particle in its lattice cell; amp = 1 moves
    particles across leaf boundaries, so leaf counts vary and the tree adapts)."""
    x, a, s = taylor_green(n, overlap, lo, L)
    h = L / n
    rng = np.random.default_rng(seed)
    xj = x.astype(np.float64) + (rng.random(x.shape) - 0.5) * 2.0 * amp * h
    xj = np.clip(xj, lo, np.nextafter(np.float32(lo + L), np.float32(lo)))
    return xj.astype(np.float32), a, s


# ----------------------------------------------------------------- multi-GPU --
RANK_LATTICE = {1: (1, 1, 1), 2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}


def taylor_green_rank(n: int, nranks: int, rank: int, lo=-np.pi, L=TWO_PI):
    """Weak-scaling workload: the Taylor-Green field in
    the fixed periodic cube [lo, lo+L)^3 sampled on a global lattice of
    n*(mx, my, mz) points, (mx, my, mz) = RANK_LATTICE[nranks], so every rank
    holds n^3 particles: those of its top-level Morton octants
    [8 rank / P, 8 (rank+1) / P) (x-fastest octant bits).  P = 8 is the
    isotropic 2n^3 lattice (C4 for n = 256); sigma = the largest spacing.

    Returns (x, alpha, sigma) float32 for this rank, in x-fastest order."""
    m = RANK_LATTICE[nranks]
    o = 8 * rank // nranks
    bits = (o & 1, (o >> 1) & 1, (o >> 2) & 1)
    h = [L / (m[d] * n) for d in range(3)]
    axes = []
    for d in range(3):
        i0 = bits[d] * n if m[d] == 2 else 0
        axes.append(lo + (np.arange(i0, i0 + n, dtype=np.float64) + 0.5) * h[d])
    Z, Y, X = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    x = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=-1)
    alpha = omega_tg(x) * (h[0] * h[1] * h[2])
    sigma = np.full(x.shape[0], max(h))
    return x.astype(np.float32), alpha.astype(np.float32), sigma.astype(np.float32)


RANK_TILES = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}


def taylor_green_tile(n: int, nranks: int, rank: int, lo=-np.pi, L=TWO_PI):
    """Weak-scaling workload of reading Z27: the periodic domain is
    RANK_TILES[nranks] copies of the 2 pi cube and rank r holds the n^3
    Taylor-Green lattice of tile r (tile index = the bits of r, x fastest),
    i.e. top-level octant r of the root cube.  Per-GPU work equals the
    single-GPU periodic run."""
    t = (rank & 1, (rank >> 1) & 1, (rank >> 2) & 1)
    x, a, s = taylor_green(n, 1.0, lo, L)
    x = x.astype(np.float64) + np.array([t[0] * L, t[1] * L, t[2] * L])
    return x.astype(np.float32), a, s


def taylor_green_octants(n: int, nranks: int, rank: int, lo=-np.pi, L=TWO_PI):
    """Strong-scaling workload (C4: n^3 in the fixed periodic cube): rank r
    holds the lattice points of top-level Morton octants [8r/P, 8(r+1)/P)
    (z halves for P = 2, y-z quarters for P = 4, octants for P = 8)."""
    x, a, s = taylor_green(n, 1.0, lo, L)
    mid = lo + 0.5 * L
    o = ((x[:, 0] >= mid).astype(int) | ((x[:, 1] >= mid).astype(int) << 1) | ((x[:, 2] >= mid).astype(int) << 2))
    keep = (o >= 8 * rank // nranks) & (o < 8 * (rank + 1) // nranks)
    return x[keep], a[keep], s[keep]


def clustered_cloud(n: int, seed: int = 1106, lo=-np.pi, L=TWO_PI, sigma=None):
    """Non-uniform workload for the balanced partition (NEXT-3): half the
    particles uniform in the periodic cube, half in a Gaussian cluster of
    width L/16 (wrapped), alpha ~ N(0,1) h^3 with h = L / n^(1/3), sigma = h
    (or the given sigma)."""
    rng = np.random.default_rng(seed)
    h = L / round(n ** (1.0 / 3.0))
    m = n // 2
    xu = rng.uniform(lo, lo + L, size=(n - m, 3))
    xc = lo + np.mod(0.3 * L + rng.normal(0.0, L / 16, size=(m, 3)), L)
    x = np.concatenate([xu, xc]).astype(np.float32)
    a = (rng.standard_normal((n, 3)) * h ** 3).astype(np.float32)
    s = np.full(n, h if sigma is None else sigma, dtype=np.float32)
    return x, a, s


def scatter_to_ranks(n: int, nranks: int, rank: int, seed: int = 5273):
    """Indices of the particles rank `rank` passes in the balanced-partition
    tests: a seeded random assignment (every rank holds an arbitrary subset)."""
    owner = np.random.default_rng(seed).integers(0, nranks, size=n)
    return np.nonzero(owner == rank)[0]
