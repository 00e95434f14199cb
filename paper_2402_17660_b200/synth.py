"""Seeded synthetic workloads of BASELINE.json.

Positions are rounded through float32 so the GPU (float32 in, exact float64 internally) and
the float64 CPU oracle see identical bits.  Returns plain numpy arrays:
(species int64 [N], positions float64 [N,3] (float32-representable), batch int64 [N], box 3x3 or None).
"""

from __future__ import annotations

import numpy as np

WATER_DENSITY = 0.1003  # atoms / A^3


def _thin_cloud(rng, n, edge, min_sep):
    """Uniform cloud with a minimum-separation rejection pass, vectorised with a cell hash."""
    pos = rng.uniform(0.0, edge, (n, 3))
    if min_sep <= 0:
        return pos
    m = max(int(np.floor(edge / min_sep)), 1)
    for _ in range(200):
        cells = np.minimum((pos / edge * m).astype(np.int64), m - 1)
        bad = np.zeros(n, dtype=bool)
        key = (cells[:, 0] * m + cells[:, 1]) * m + cells[:, 2]
        order = np.argsort(key, kind="stable")
        skey = key[order]
        start = np.searchsorted(skey, np.arange(m**3), side="left")
        end = np.searchsorted(skey, np.arange(m**3), side="right")
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    nb = ((cells[:, 0] + dx) % m * m + (cells[:, 1] + dy) % m) * m + (cells[:, 2] + dz) % m
                    s, e = start[nb], end[nb]
                    width = int((e - s).max()) if n else 0
                    for t in range(width):
                        idx = s + t
                        ok = idx < e
                        j = order[np.where(ok, idx, 0)]
                        d = pos - pos[j]
                        d -= edge * np.rint(d / edge)
                        close = ok & (j < np.arange(n)) & ((d * d).sum(1) < min_sep * min_sep)
                        bad |= close
        if not bad.any():
            return pos
        pos[bad] = rng.uniform(0.0, edge, (int(bad.sum()), 3))
    return pos


def _f32(pos):
    return pos.astype(np.float32).astype(np.float64)


def config_a_molecule(seed: int = 0):
    """A: 22 atoms, open, alanine-dipeptide composition C6 H12 N2 O2, min separation 0.9 A."""
    rng = np.random.default_rng(seed)
    pts = []
    while len(pts) < 22:
        p = rng.uniform(0.0, 6.0, 3)
        if all(np.linalg.norm(p - q) >= 0.9 for q in pts):
            pts.append(p)
    species = np.array([6] * 6 + [1] * 12 + [7] * 2 + [8] * 2, dtype=np.int64)
    rng.shuffle(species)
    return species, _f32(np.array(pts)), np.zeros(22, dtype=np.int64), None


def config_b_cloud(n: int, seed: int = 0):
    """B: uniform cloud at water density in a periodic cube (neighbor-list sweep)."""
    edge = (n / WATER_DENSITY) ** (1.0 / 3.0)
    rng = np.random.default_rng(seed)
    pos = _f32(rng.uniform(0.0, edge, (n, 3)))
    edge32 = float(np.float32(edge))
    pos = np.minimum(pos, np.nextafter(np.float32(edge32), np.float32(0)).astype(np.float64))
    return np.ones(n, dtype=np.int64), pos, np.zeros(n, dtype=np.int64), np.eye(3) * edge32


def config_c_box(n: int = 23558, edge: float = 62.23, seed: int = 1, min_sep: float = 0.8):
    """C: DHFR-sized periodic cubic box, water-like species mix, 0.8 A minimum separation."""
    rng = np.random.default_rng(seed)
    pos = _thin_cloud(rng, n, edge, min_sep)
    species = rng.choice([1, 6, 7, 8], size=n, p=[0.66, 0.14, 0.06, 0.14]).astype(np.int64)
    edge32 = float(np.float32(edge))
    return species, _f32(pos), np.zeros(n, dtype=np.int64), np.eye(3) * edge32


def config_d_molecules(n_molecules: int = 8192, seed: int = 2):
    """D: QM9-sized molecules (12..24 atoms) grown by random-walk bonding, open boundaries."""
    rng = np.random.default_rng(seed)
    sizes = rng.integers(12, 25, n_molecules)
    pos, species, batch = [], [], []
    for m, k in enumerate(sizes):
        pts = [np.zeros(3)]
        while len(pts) < k:
            base = pts[rng.integers(len(pts))]
            step = rng.standard_normal(3)
            cand = base + step / np.linalg.norm(step) * rng.uniform(1.1, 1.5)
            if all(np.linalg.norm(cand - q) >= 0.9 for q in pts):
                pts.append(cand)
        pos.append(np.array(pts))
        species.append(rng.choice([1, 6, 7, 8, 9], size=k, p=[0.5, 0.3, 0.07, 0.1, 0.03]))
        batch.append(np.full(k, m, dtype=np.int64))
    return (np.concatenate(species).astype(np.int64), _f32(np.concatenate(pos)),
            np.concatenate(batch), None)


def config_e_triclinic(n: int = 100_000, seed: int = 3, min_sep: float = 0.0):
    """E: triclinic periodic box at water density; rows a=(L,0,0), b=(0.3L,L,0), c=(0.2L,-0.25L,L)."""
    rng = np.random.default_rng(seed)
    L = float(np.float32((n / WATER_DENSITY) ** (1.0 / 3.0)))
    box = np.array([[L, 0.0, 0.0], [0.3 * L, L, 0.0], [0.2 * L, -0.25 * L, L]])
    box = box.astype(np.float32).astype(np.float64)
    pos = rng.uniform(0.0, 1.0, (n, 3)) @ box
    species = rng.choice([1, 8], size=n, p=[2 / 3, 1 / 3]).astype(np.int64)
    return species, _f32(pos), np.zeros(n, dtype=np.int64), box


from .sharding import shard_by_molecule  # noqa: E402,F401  (kept importable from here)
