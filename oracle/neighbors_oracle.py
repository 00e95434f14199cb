"""CPU oracle for the neighbor-search half of the hot path.

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / reference arm
may import this module; the product package never does.

This is a float64 restatement of the reference's neighbor engine
(``/root/reference/pkg/src/nnpkit``):

* grid construction           ``neighbors.py:103-124``
* cell sort                   ``neighbors.py:127-133``   (C: ``nlo_sort_cells``)
* the four pair kernels       ``_neighbor_kernels.py:24-233`` (C: ``nl_oracle.c``)
* build / overflow / mirror / loops / lexsort   ``neighbors.py:136-235``
* canonical form              ``neighbors.py:250-260``
* half/full views             ``neighbors.py:263-320``
* distance pullback           ``neighbors.py:323-355``
* box widths                  ``system.py:93-106``
* radial functions            ``radial.py:11-73``
* segment_sum / silu          ``_ops.py:6-37``

Parity status: PINNED.  ``tests/golden/make_golden.py`` runs the reference
itself (imported from ``/root/reference``) on seeded inputs and stores its
outputs; ``tests/test_oracle_neighbors.py`` checks this module against those
vectors bit for bit, and against the reference's own known-answer cases
(``tests/test_neighbors.py:42-108``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

AUTO_STRATEGY_THRESHOLD = 10_000  # neighbors.py:24


class OracleCapacityError(Exception):
    def __init__(self, required: int, capacity: int):
        super().__init__(f"overflow: required {required}, capacity {capacity}")
        self.required = int(required)
        self.capacity = int(capacity)


class OracleValidationError(Exception):
    pass


class OracleNumericError(Exception):
    pass


def build_library(force: bool = False) -> str:
    """Compile nl_oracle.c with the committed Makefile recipe."""
    so = os.path.join(_HERE, "libnl_oracle.so")
    src = os.path.join(_HERE, "nl_oracle.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-s", "libnl_oracle.so"], check=True)
    return so


def _lib():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(build_library())
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        f64 = ctypes.c_double
        lib.nlo_brute_half.restype = i64
        lib.nlo_brute_half.argtypes = [p, p, i64, p, f64, f64, i64, p, p, p]
        lib.nlo_cell_half.restype = i64
        lib.nlo_cell_half.argtypes = [p, p, i64, p, ctypes.c_int, f64, f64, p, p, p, p, i64, p, p, p]
        lib.nlo_sort_cells.restype = None
        lib.nlo_sort_cells.argtypes = [p, p, i64, p, p]
        _LIB = lib
    return _LIB


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------- box

def perpendicular_widths(vectors: np.ndarray) -> np.ndarray:
    """Face-to-face distances V / |b x c| etc. (system.py:93-103)."""
    a, b, c = np.asarray(vectors, dtype=np.float64)
    vol = abs(np.linalg.det(np.asarray(vectors, dtype=np.float64)))
    return np.array(
        [
            vol / np.linalg.norm(np.cross(b, c)),
            vol / np.linalg.norm(np.cross(a, c)),
            vol / np.linalg.norm(np.cross(a, b)),
        ]
    )


def periodic_grid(positions, vectors, cutoff):
    """Fractional-space cells; None when an axis holds fewer than 3 (neighbors.py:103-113)."""
    widths = perpendicular_widths(vectors)
    dims = np.floor(widths / cutoff).astype(np.int64)
    if np.any(dims < 3):
        return None
    frac = positions @ np.linalg.inv(vectors)
    frac = frac - np.floor(frac)
    coords = np.floor(frac * dims).astype(np.int64) % dims
    return coords, dims


def open_grid(positions, cutoff):
    """Bounding-box cells inflated by half a cutoff per side (neighbors.py:116-124)."""
    low = positions.min(axis=0) - 0.5 * cutoff
    extent = positions.max(axis=0) - low + 0.5 * cutoff
    dims = np.maximum(np.floor(extent / cutoff).astype(np.int64), 1)
    edge = extent / dims
    coords = np.clip(np.floor((positions - low) / edge).astype(np.int64), 0, dims - 1)
    return coords, dims


def sort_cells(coords, dims):
    n = coords.shape[0]
    coords = np.ascontiguousarray(coords, dtype=np.int64)
    dims = np.ascontiguousarray(dims, dtype=np.int64)
    ncell = int(dims[0] * dims[1] * dims[2])
    order = np.empty(n, dtype=np.int64)
    start = np.empty(ncell + 1, dtype=np.int64)
    _lib().nlo_sort_cells(_ptr(coords), _ptr(dims), n, _ptr(order), _ptr(start))
    return order, start


# ------------------------------------------------------------------------- build

@dataclass
class OracleList:
    pairs: np.ndarray       # [capacity, 2] int64, -1 sentinels
    deltas: np.ndarray      # [capacity, 3] float64, r_i - r_j minimum image
    distances: np.ndarray   # [capacity] float64
    count: int
    n_atoms: int
    full_list: bool
    deterministic: bool
    cutoff_lower: float
    cutoff_upper: float
    notes: tuple = ()

    @property
    def capacity(self) -> int:
        return self.pairs.shape[0]

    def valid(self):
        c = self.count
        return self.pairs[:c], self.deltas[:c], self.distances[:c]


def build_neighbor_list(
    positions,
    batch,
    box_vectors,           # 3x3 rows a,b,c (lower triangular) or None for open systems
    cutoff_upper: float,
    capacity: int,
    cutoff_lower: float = 0.0,
    strategy: str = "auto",
    include_self_loops: bool = False,
    full_list: bool = False,
    deterministic: bool = True,
) -> OracleList:
    """Restatement of neighbors.py:136-235 (same dispatch, errors and ordering)."""
    positions = np.ascontiguousarray(positions, dtype=np.float64)
    n = positions.shape[0]
    batch = np.ascontiguousarray(
        np.zeros(n, dtype=np.int64) if batch is None else batch, dtype=np.int64
    )
    if not 0.0 <= cutoff_lower < cutoff_upper:
        raise OracleValidationError("cutoffs must satisfy 0 <= lower < upper")
    if capacity < 1:
        raise OracleValidationError("capacity must be >= 1")
    box9 = None
    if box_vectors is not None:
        box9 = np.ascontiguousarray(box_vectors, dtype=np.float64).reshape(3, 3)
        half = perpendicular_widths(box9).min() / 2.0
        if cutoff_upper > half:
            raise OracleValidationError(
                f"cutoff too large for box: {cutoff_upper} exceeds half the minimum "
                f"perpendicular width {half}"
            )
    if strategy == "auto":
        strategy = "brute" if n < AUTO_STRATEGY_THRESHOLD else "cell"
    notes = []
    grid = None
    if strategy == "cell":
        grid = (
            periodic_grid(positions, box9, cutoff_upper)
            if box9 is not None
            else open_grid(positions, cutoff_upper)
        )
        if grid is None:
            notes.append(
                "cell strategy needs at least 3 cells per periodic dimension; "
                "fell back to brute force"
            )
            strategy = "brute"
    elif strategy != "brute":
        raise OracleValidationError(f"unknown strategy {strategy!r}")

    pairs = np.full((capacity, 2), -1, dtype=np.int64)
    deltas = np.zeros((capacity, 3), dtype=np.float64)
    dists = np.zeros(capacity, dtype=np.float64)
    lib = _lib()
    if strategy == "brute":
        found = lib.nlo_brute_half(
            _ptr(positions), _ptr(batch), n, _ptr(box9), cutoff_lower, cutoff_upper,
            capacity, _ptr(pairs), _ptr(deltas), _ptr(dists),
        )
    else:
        coords, dims = grid
        coords = np.ascontiguousarray(coords, dtype=np.int64)
        dims = np.ascontiguousarray(dims, dtype=np.int64)
        order, start = sort_cells(coords, dims)
        found = lib.nlo_cell_half(
            _ptr(positions), _ptr(batch), n, _ptr(box9), int(box9 is not None),
            cutoff_lower, cutoff_upper, _ptr(coords), _ptr(dims), _ptr(order), _ptr(start),
            capacity, _ptr(pairs), _ptr(deltas), _ptr(dists),
        )
    found = int(found)
    n_loops = n if include_self_loops else 0
    total = (2 * found if full_list else found) + n_loops
    if total > capacity:
        raise OracleCapacityError(required=total, capacity=capacity)
    if full_list and found:
        pairs[found : 2 * found] = pairs[:found, ::-1]
        deltas[found : 2 * found] = -deltas[:found]
        dists[found : 2 * found] = dists[:found]
    if n_loops:
        base = total - n_loops
        pairs[base:total, 0] = np.arange(n)
        pairs[base:total, 1] = np.arange(n)
        deltas[base:total] = 0.0
        dists[base:total] = 0.0
    if deterministic and total > 1:
        key = np.lexsort((pairs[:total, 1], pairs[:total, 0]))
        pairs[:total] = pairs[:total][key]
        deltas[:total] = deltas[:total][key]
        dists[:total] = dists[:total][key]
    return OracleList(
        pairs, deltas, dists, total, n, full_list, deterministic,
        float(cutoff_lower), float(cutoff_upper), tuple(notes),
    )


def build_with_auto_capacity(positions, batch, box_vectors, cutoff_upper, capacity, **kw):
    """neighbors.py:238-247."""
    for _ in range(32):
        try:
            return build_neighbor_list(positions, batch, box_vectors, cutoff_upper, capacity, **kw)
        except OracleCapacityError as err:
            capacity = max(err.required, 2 * capacity)
    raise OracleCapacityError(required=2 * capacity, capacity=capacity)


def canonicalize(pairs, distances, count):
    """Unordered sorted unique (i<j) rows + first-occurrence distance (neighbors.py:250-260)."""
    p = np.sort(np.asarray(pairs)[:count], axis=1)
    unique, first = np.unique(p, axis=0, return_index=True)
    return unique, np.asarray(distances)[:count][first]


def as_full_list(nl: OracleList) -> OracleList:
    """Directed view (neighbors.py:263-294); capacity doubles."""
    if nl.full_list:
        return nl
    pairs, deltas, dists = nl.valid()
    nonloop = pairs[:, 0] != pairs[:, 1]
    p = np.concatenate([pairs, pairs[nonloop][:, ::-1]], axis=0)
    d = np.concatenate([deltas, -deltas[nonloop]], axis=0)
    r = np.concatenate([dists, dists[nonloop]], axis=0)
    if nl.deterministic and p.shape[0] > 1:
        key = np.lexsort((p[:, 1], p[:, 0]))
        p, d, r = p[key], d[key], r[key]
    cap = 2 * nl.capacity
    total = p.shape[0]
    op = np.full((cap, 2), -1, dtype=np.int64)
    od = np.zeros((cap, 3))
    orr = np.zeros(cap)
    op[:total], od[:total], orr[:total] = p, d, r
    return OracleList(op, od, orr, total, nl.n_atoms, True, nl.deterministic,
                      nl.cutoff_lower, nl.cutoff_upper, nl.notes)


def as_half_list(nl: OracleList) -> OracleList:
    """Undirected view keeping i <= j rows (neighbors.py:297-320)."""
    if not nl.full_list:
        return nl
    pairs, deltas, dists = nl.valid()
    keep = pairs[:, 0] <= pairs[:, 1]
    cap = nl.capacity
    total = int(keep.sum())
    op = np.full((cap, 2), -1, dtype=np.int64)
    od = np.zeros((cap, 3))
    orr = np.zeros(cap)
    op[:total], od[:total], orr[:total] = pairs[keep], deltas[keep], dists[keep]
    return OracleList(op, od, orr, total, nl.n_atoms, False, nl.deterministic,
                      nl.cutoff_lower, nl.cutoff_upper, nl.notes)


def distance_pullback(pairs, deltas, distances, count, n_atoms, d_grad):
    """d(sum_k g_k d_k)/d(positions): +g*u at i, -g*u at j; loops zero (neighbors.py:323-355)."""
    pairs = np.asarray(pairs)[:count]
    deltas = np.asarray(deltas, dtype=np.float64)[:count]
    dists = np.asarray(distances, dtype=np.float64)[:count]
    g = np.asarray(d_grad, dtype=np.float64)[:count]
    loops = pairs[:, 0] == pairs[:, 1]
    bad = ~loops & (dists == 0.0)
    if np.any(bad):
        i, j = pairs[bad][0]
        raise OracleNumericError(f"zero-distance pair ({i}, {j}) has no defined distance direction")
    safe = np.where(loops, 1.0, dists)
    unit = deltas / safe[:, None]
    unit[loops] = 0.0
    contrib = g[:, None] * unit
    return segment_sum(contrib, pairs[:, 0], n_atoms) - segment_sum(contrib, pairs[:, 1], n_atoms)


def distance_pullback_second(pairs, deltas, distances, count, n_atoms, capacity, d_grad, position_tangent):
    """Directional derivative of distance_pullback along a position tangent with the analytic pair
    Hessian (I - u u^T)/d; also the distance tangents u . (t_i - t_j), zero on loops and in sentinel
    slots (neighbors.py:358-380, same operation order)."""
    pairs = np.asarray(pairs)[:count]
    deltas = np.asarray(deltas, dtype=np.float64)[:count]
    dists = np.asarray(distances, dtype=np.float64)[:count]
    g = np.asarray(d_grad, dtype=np.float64)[:count]
    tangent = np.asarray(position_tangent, dtype=np.float64)
    loops = pairs[:, 0] == pairs[:, 1]
    bad = ~loops & (dists == 0.0)
    if np.any(bad):
        i, j = pairs[bad][0]
        raise OracleNumericError(f"zero-distance pair ({i}, {j}) has no defined distance direction")
    safe = np.where(loops, 1.0, dists)
    unit = deltas / safe[:, None]
    unit[loops] = 0.0
    tdiff = tangent[pairs[:, 0]] - tangent[pairs[:, 1]]
    ddot = np.einsum("ij,ij->i", unit, tdiff)
    hvp = g[:, None] * (tdiff - unit * ddot[:, None]) / safe[:, None]
    hvp[loops] = 0.0
    grad = segment_sum(hvp, pairs[:, 0], n_atoms) - segment_sum(hvp, pairs[:, 1], n_atoms)
    distance_tangent = np.zeros(capacity)
    distance_tangent[:count] = np.where(loops, 0.0, ddot)
    return grad, distance_tangent


# ------------------------------------------------------- independent O(N^2) oracle

_IMAGE_SHIFTS = np.array(
    [(i, j, k) for i in (-1, 0, 1) for j in (-1, 0, 1) for k in (-1, 0, 1)], dtype=np.float64
)


def exhaustive_pair_set(positions, batch, box_vectors, r_lower, r_upper):
    """All-pairs with the exhaustive 27-image minimum: the independent ground truth
    the reference's tests use (tests/conftest.py:57-76)."""
    positions = np.asarray(positions, dtype=np.float64)
    d = positions[:, None, :] - positions[None, :, :]
    if box_vectors is None:
        dist = np.linalg.norm(d, axis=-1)
    else:
        shifts = _IMAGE_SHIFTS @ np.asarray(box_vectors, dtype=np.float64)
        dist = np.sqrt(((d[None] + shifts[:, None, None, :]) ** 2).sum(-1)).min(axis=0)
    n = positions.shape[0]
    iu, ju = np.triu_indices(n, k=1)
    batch = np.zeros(n, dtype=np.int64) if batch is None else np.asarray(batch)
    keep = (batch[iu] == batch[ju]) & (dist[iu, ju] > r_lower) & (dist[iu, ju] <= r_upper)
    return np.stack([iu[keep], ju[keep]], axis=1), dist[iu[keep], ju[keep]]


# ------------------------------------------------------------------ radial / ops

def cosine_cutoff(d, cutoff_lower, cutoff_upper):
    """radial.py:11-27."""
    d = np.asarray(d, dtype=np.float64)
    if cutoff_lower == 0.0:
        val = 0.5 * (np.cos(np.pi * d / cutoff_upper) + 1.0)
        return np.where(d <= cutoff_upper, val, 0.0)
    t = 2.0 * (d - cutoff_lower) / (cutoff_upper - cutoff_lower) + 1.0
    val = 0.5 * (np.cos(np.pi * t) + 1.0)
    return np.where((d >= cutoff_lower) & (d <= cutoff_upper), val, 0.0)


def cosine_cutoff_grad(d, cutoff_lower, cutoff_upper):
    """radial.py:30-39."""
    d = np.asarray(d, dtype=np.float64)
    if cutoff_lower == 0.0:
        val = -0.5 * np.pi / cutoff_upper * np.sin(np.pi * d / cutoff_upper)
        return np.where(d <= cutoff_upper, val, 0.0)
    span = cutoff_upper - cutoff_lower
    t = 2.0 * (d - cutoff_lower) / span + 1.0
    val = -np.pi / span * np.sin(np.pi * t)
    return np.where((d >= cutoff_lower) & (d <= cutoff_upper), val, 0.0)


def expnorm_initial_params(num_rbf, cutoff_lower, cutoff_upper):
    """radial.py:42-50."""
    start = np.exp(-(cutoff_upper - cutoff_lower))
    means = np.linspace(start, 1.0, num_rbf)
    betas = np.full(num_rbf, (2.0 / num_rbf * (1.0 - start)) ** -2)
    return means, betas


def rbf_expnorm(d, means, betas, cutoff_lower):
    """radial.py:53-59."""
    u = np.exp(cutoff_lower - np.asarray(d, dtype=np.float64))[..., None]
    return np.exp(-betas * (u - means) ** 2)


def rbf_expnorm_dd(d, means, betas, cutoff_lower):
    """df/dd of the basis (radial.py:62-73)."""
    u = np.exp(cutoff_lower - np.asarray(d, dtype=np.float64))[..., None]
    diff = u - means
    return np.exp(-betas * diff**2) * 2.0 * betas * diff * u


def segment_sum(values, index, n_segments):
    """Row-order scatter-add (_ops.py:6-19)."""
    values = np.asarray(values, dtype=np.float64)
    index = np.asarray(index, dtype=np.int64)
    if values.ndim == 1:
        return np.bincount(index, weights=values, minlength=n_segments)
    cols = values.shape[1]
    flat = (index[:, None] * cols + np.arange(cols)[None, :]).ravel()
    return np.bincount(flat, weights=values.ravel(), minlength=n_segments * cols).reshape(
        n_segments, cols
    )


def sigmoid(x):
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def silu(x):
    return x * sigmoid(x)


def silu_grad(x):
    s = sigmoid(x)
    return s * (1.0 + x * (1.0 - s))
