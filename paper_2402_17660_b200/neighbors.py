"""Batched cutoff neighbor search on the GPU behind the reference's Python API.

``build_neighbor_list(system, spec) -> NeighborList`` keeps the signature and semantics of
``nnpkit/neighbors.py:136-235`` (NeighborSpec :30-57, NeighborList :61-84): rows [0, count) are
valid, the rest hold -1 / 0 sentinels; ``deltas = r_i - r_j`` minimum image; window
``cutoff_lower < d <= cutoff_upper``; same-batch pairs only; half list (i < j) unless
``full_list``; self loops bypass the window; rows are in lexicographic (i, j) order; a periodic
cell grid with fewer than 3 cells per axis falls back to brute force with a note; a cutoff above
half the minimum perpendicular width raises ``ValidationError``; overflow raises
``CapacityError(required, capacity)``.

Departure: the arrays of the returned list are CUDA tensors (int32 pairs, float64
deltas/distances -- computed in float64 with the reference's operation order, so they are
bit-identical to the reference's); ``NeighborList.as_reference()`` gives the numpy
int64/float64 form.  All compute happens in ``libnnp_b200.so``; there is no CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import _lib
from .errors import CapacityError, NumericError, ValidationError
from .system import Box, System

#: Atom count at which strategy "auto" switches from brute force to cells (neighbors.py:24).
AUTO_STRATEGY_THRESHOLD = 10_000
_STRATEGIES = ("brute", "cell", "auto")
#: Hard ceiling on the cells of an open-boundary grid (device clamps to the workspace size).
_MAX_OPEN_CELLS = 1 << 22


@dataclass(frozen=True)
class NeighborSpec:
    """Construction parameters of a neighbor list (neighbors.py:30-57)."""

    cutoff_upper: float
    capacity: int
    cutoff_lower: float = 0.0
    strategy: str = "auto"
    include_self_loops: bool = False
    full_list: bool = False
    deterministic: bool = True

    def __post_init__(self):
        if not 0.0 <= self.cutoff_lower < self.cutoff_upper:
            raise ValidationError(
                "cutoffs must satisfy 0 <= cutoff_lower < cutoff_upper, got "
                f"{self.cutoff_lower} and {self.cutoff_upper}"
            )
        if self.capacity < 1:
            raise ValidationError("capacity must be >= 1")
        if self.strategy not in _STRATEGIES:
            raise ValidationError(
                f"unknown strategy {self.strategy!r}, expected one of {_STRATEGIES}"
            )


@dataclass(frozen=True)
class NeighborList:
    """Padded pair set; rows [0, count) are valid (neighbors.py:61-84).

    ``pairs``/``deltas``/``distances`` are CUDA tensors when the list comes from
    ``build_neighbor_list`` and numpy arrays after ``as_reference()``.  ``row_ptr`` (CSR offsets
    per atom, device lists only) is extra information the reference does not carry.
    """

    pairs: object
    deltas: object
    distances: object
    count: int
    n_atoms: int
    spec: NeighborSpec
    notes: tuple = ()
    row_ptr: object = None

    @property
    def capacity(self) -> int:
        return int(self.pairs.shape[0])

    @property
    def on_device(self) -> bool:
        return not isinstance(self.pairs, np.ndarray)

    def valid(self):
        c = self.count
        return self.pairs[:c], self.deltas[:c], self.distances[:c]

    def as_reference(self) -> "NeighborList":
        """Host copy in the reference's dtypes: int64 pairs, float64 deltas/distances."""
        if not self.on_device:
            return self
        return NeighborList(
            pairs=self.pairs.cpu().numpy().astype(np.int64),
            deltas=self.deltas.cpu().numpy().astype(np.float64),
            distances=self.distances.cpu().numpy().astype(np.float64),
            count=self.count, n_atoms=self.n_atoms, spec=self.spec, notes=self.notes,
        )


def capacity_heuristic(n_atoms: int, max_num_neighbors: int) -> int:
    """atoms x max-neighbors pair budget (neighbors.py:87-89)."""
    return max(1, int(n_atoms) * int(max_num_neighbors))


# --------------------------------------------------------------------------- host planning

def check_cutoff_against_box(box: Optional[Box], cutoff_upper: float) -> None:
    """cutoff <= half the minimum perpendicular width (neighbors.py:146-152)."""
    if box is not None and box.periodic:
        half = box.min_width() / 2.0
        if cutoff_upper > half:
            raise ValidationError(
                f"cutoff too large for box: {cutoff_upper} exceeds half the "
                f"minimum perpendicular width {half}"
            )


def plan_strategy(n_atoms: int, box: Optional[Box], cutoff_upper: float, strategy: str):
    """Resolve "auto" and the periodic grid on the host (neighbors.py:155-170).

    Returns (strategy_code, grid_dims, max_cells, notes)."""
    notes = []
    if strategy == "auto":
        strategy = "brute" if n_atoms < AUTO_STRATEGY_THRESHOLD else "cell"
    dims = (0, 0, 0)
    max_cells = 1
    if strategy == "cell":
        if box is not None and box.periodic:
            d = np.floor(box.perpendicular_widths() / cutoff_upper).astype(np.int64)
            if np.any(d < 3):
                notes.append(
                    "cell strategy needs at least 3 cells per periodic dimension; "
                    "fell back to brute force"
                )
                strategy = "brute"
            else:
                # more cells than atoms only adds empty cells to scan; coarsen (cells stay >= cutoff)
                while int(d[0] * d[1] * d[2]) > max(8 * n_atoms, 27) and np.any(d > 3):
                    k = int(np.argmax(d))
                    d[k] = max(3, (d[k] + 1) // 2)
                dims = tuple(int(x) for x in d)
                max_cells = int(d[0] * d[1] * d[2])
        else:
            max_cells = int(min(max(2 * n_atoms, 64), _MAX_OPEN_CELLS))
    code = _lib.STRATEGY_CELL if strategy == "cell" else _lib.STRATEGY_BRUTE
    return code, dims, max_cells, tuple(notes)


class NeighborEngine:
    """Device buffers + one enqueue call for a fixed (n_atoms, capacity, flags, box) shape.

    Used by ``build_neighbor_list`` and, with RENUMBER | F32_OUT | NO_PAD, by the TensorNet
    step.  ``build`` only enqueues kernels on the current stream (CUDA-graph capturable); the
    caller reads ``counts`` after synchronising to detect overflow.
    """

    def __init__(self, n_atoms: int, n_samples: int, capacity: int, box: Optional[Box],
                 cutoff_lower: float, cutoff_upper: float, strategy_code: int, grid_dims,
                 max_cells: int, flags: int, device=None, want_row_ptr: bool = True,
                 want_order: bool = False):
        torch = _lib.require_cuda()
        self.lib = _lib.load()
        self.device = torch.device(device if device is not None else "cuda")
        self.n_atoms, self.n_samples, self.capacity, self.flags = n_atoms, n_samples, capacity, flags
        p = _lib.NlParams()
        p.n_atoms, p.n_samples, p.capacity = n_atoms, n_samples, capacity
        p.box_kind = _lib.BOX_KIND[box.kind] if box is not None else 0
        p.strategy, p.flags, p.max_cells = strategy_code, flags, max_cells
        p.grid_dims[:] = list(grid_dims)
        p.cutoff_lower, p.cutoff_upper = float(cutoff_lower), float(cutoff_upper)
        if box is not None and box.periodic:
            p.box[:] = list(np.asarray(box.vectors, dtype=np.float64).ravel())
            p.inv_box[:] = list(np.linalg.inv(np.asarray(box.vectors, dtype=np.float64)).ravel())
        self.params = p
        need = ctypes.c_size_t(0)
        _lib.check(self.lib.nnp_nl_workspace_bytes(ctypes.byref(p), ctypes.byref(need)),
                   "nnp_nl_workspace_bytes")
        real = torch.float32 if flags & _lib.NL_F32_OUT else torch.float64
        dev = self.device
        self.workspace = torch.empty(need.value, dtype=torch.uint8, device=dev)
        self.pairs = torch.empty((capacity, 2), dtype=torch.int32, device=dev)
        self.deltas = torch.empty((capacity, 3), dtype=real, device=dev)
        self.dists = torch.empty(capacity, dtype=real, device=dev)
        self.row_ptr = torch.empty(n_atoms + 1, dtype=torch.int32, device=dev) if want_row_ptr else None
        self.order = torch.empty(n_atoms, dtype=torch.int32, device=dev) if want_order else None
        self.counts = torch.zeros(4, dtype=torch.int32, device=dev)

    def build(self, pos64, batch32) -> None:
        rc = self.lib.nnp_nl_build(
            ctypes.byref(self.params), _lib.ptr(pos64), _lib.ptr(batch32), _lib.ptr(self.pairs),
            _lib.ptr(self.deltas), _lib.ptr(self.dists), _lib.ptr(self.row_ptr),
            _lib.ptr(self.order), _lib.ptr(self.counts), _lib.ptr(self.workspace),
            self.workspace.numel(), _lib.current_stream(),
        )
        _lib.check(rc, "nnp_nl_build")


def build_neighbor_list(system: System, spec: NeighborSpec) -> NeighborList:
    """Enumerate all in-batch pairs inside the distance window on the GPU.

    Drop-in for ``nnpkit.build_neighbor_list`` (neighbors.py:136-235).  With
    ``deterministic=False`` rows are still grouped by ``i`` but the order inside a group is the
    order of discovery (the reference promises no order then, neighbors.py:221); the in-row
    ranking pass is skipped.
    """
    torch = _lib.require_cuda()
    n = system.n_atoms
    box = system.box
    check_cutoff_against_box(box, spec.cutoff_upper)
    code, dims, max_cells, notes = plan_strategy(n, box, spec.cutoff_upper, spec.strategy)
    flags = (_lib.NL_FULL_LIST if spec.full_list else 0) | (
        _lib.NL_SELF_LOOPS if spec.include_self_loops else 0) | (
        0 if spec.deterministic else _lib.NL_UNSORTED)
    eng = NeighborEngine(n, system.n_samples, spec.capacity, box, spec.cutoff_lower,
                         spec.cutoff_upper, code, dims, max_cells, flags)
    pos = torch.from_numpy(np.array(system.positions, dtype=np.float64, order="C")).to(eng.device)
    batch = torch.from_numpy(np.array(system.batch, dtype=np.int32, order="C")).to(eng.device)
    eng.build(pos, batch)
    counts = eng.counts.cpu().numpy()          # synchronises the stream
    total = int(counts[0])
    if total > spec.capacity:
        raise CapacityError(required=total, capacity=spec.capacity)
    return NeighborList(pairs=eng.pairs, deltas=eng.deltas, distances=eng.dists, count=total,
                        n_atoms=n, spec=spec, notes=notes, row_ptr=eng.row_ptr)


def build_with_auto_capacity(system: System, spec: NeighborSpec, max_doublings: int = 32) -> NeighborList:
    """Build, growing capacity to max(required, 2x) on overflow (neighbors.py:238-247)."""
    for _ in range(max_doublings):
        try:
            return build_neighbor_list(system, spec)
        except CapacityError as err:
            spec = replace(spec, capacity=max(err.required, 2 * spec.capacity))
    raise CapacityError(required=spec.capacity * 2, capacity=spec.capacity)


# ------------------------------------------------------------------------------ list views

def canonicalize(nlist: NeighborList):
    """Unordered pairs as sorted unique (i, j) rows with their distances (neighbors.py:250-260)."""
    ref = nlist.as_reference()
    pairs, _, dists = ref.valid()
    swapped = np.sort(pairs, axis=1)
    unique, first = np.unique(swapped, axis=0, return_index=True)
    return unique, dists[first]


def _host_list(pairs, deltas, dists, capacity, n_atoms, spec, notes) -> NeighborList:
    total = pairs.shape[0]
    op = np.full((capacity, 2), -1, dtype=np.int64)
    od = np.zeros((capacity, 3))
    orr = np.zeros(capacity)
    op[:total], od[:total], orr[:total] = pairs, deltas, dists
    return NeighborList(op, od, orr, total, n_atoms, spec, notes)


def as_full_list(nlist: NeighborList) -> NeighborList:
    """Directed view; capacity doubles on upgrade (neighbors.py:263-294).  A host-side
    conversion helper: lists for the model are built directed on the device in the first place."""
    if nlist.spec.full_list:
        return nlist
    ref = nlist.as_reference()
    pairs, deltas, dists = ref.valid()
    nonloop = pairs[:, 0] != pairs[:, 1]
    p = np.concatenate([pairs, pairs[nonloop][:, ::-1]], axis=0)
    d = np.concatenate([deltas, -deltas[nonloop]], axis=0)
    r = np.concatenate([dists, dists[nonloop]], axis=0)
    if nlist.spec.deterministic and p.shape[0] > 1:
        key = np.lexsort((p[:, 1], p[:, 0]))
        p, d, r = p[key], d[key], r[key]
    cap = 2 * nlist.capacity
    return _host_list(p, d, r, cap, nlist.n_atoms,
                      replace(nlist.spec, full_list=True, capacity=cap), nlist.notes)


def as_half_list(nlist: NeighborList) -> NeighborList:
    """Undirected view keeping rows with i <= j (neighbors.py:297-320)."""
    if not nlist.spec.full_list:
        return nlist
    ref = nlist.as_reference()
    pairs, deltas, dists = ref.valid()
    keep = pairs[:, 0] <= pairs[:, 1]
    return _host_list(pairs[keep], deltas[keep], dists[keep], nlist.capacity, nlist.n_atoms,
                      replace(nlist.spec, full_list=False), nlist.notes)


def distance_pullback(nlist: NeighborList, d_grad) -> np.ndarray:
    """d(sum_k g_k d_k)/d(positions) on the GPU: +g*u at i, -g*u at j, loops contribute
    nothing, sentinel slots ignored; a zero-distance non-loop pair raises NumericError
    (neighbors.py:323-355).  Returns a numpy float64 [n_atoms, 3] array like the reference."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    d_grad = np.asarray(d_grad, dtype=np.float64)
    if d_grad.shape not in ((nlist.capacity,), (nlist.count,)):
        raise ValidationError(
            f"d_grad must have capacity ({nlist.capacity}) or count "
            f"({nlist.count}) entries, got {d_grad.shape}"
        )
    dev = torch.device("cuda")

    def to_dev(a, dtype):
        if isinstance(a, np.ndarray):
            return torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)
        return a.to(dtype=dtype).contiguous()

    pairs = to_dev(nlist.pairs, torch.int32)
    deltas = to_dev(nlist.deltas, torch.float64)
    dists = to_dev(nlist.distances, torch.float64)
    g = torch.as_tensor(np.ascontiguousarray(d_grad[: nlist.count])).to(dev)
    grad = torch.empty((nlist.n_atoms, 3), dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    rc = lib.nnp_distance_pullback(_lib.ptr(pairs), _lib.ptr(deltas), _lib.ptr(dists), _lib.ptr(g),
                                   nlist.count, nlist.n_atoms, _lib.ptr(grad), _lib.ptr(flag),
                                   _lib.current_stream())
    _lib.check(rc, "nnp_distance_pullback")
    bad = int(flag.item())
    if bad != 0x7F7F7F7F:
        i, j = (int(x) for x in pairs[bad - 1].tolist())
        raise NumericError(f"zero-distance pair ({i}, {j}) has no defined distance direction")
    return grad.cpu().numpy()


def distance_pullback_second(nlist: NeighborList, d_grad, position_tangent):
    """Directional derivative of ``distance_pullback`` along a position tangent, on the GPU
    (neighbors.py:358-380): the analytic pair Hessian (I - u u^T)/d per edge.  Returns
    ``(grad [n_atoms, 3], distance_tangent [capacity])`` as numpy float64 arrays; the distance
    tangents u . (t_i - t_j) are zero on loops and in sentinel slots."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    position_tangent = np.asarray(position_tangent, dtype=np.float64)
    if position_tangent.shape != (nlist.n_atoms, 3):
        raise ValidationError(f"position tangent must have shape ({nlist.n_atoms}, 3)")
    d_grad = np.asarray(d_grad, dtype=np.float64)
    if d_grad.shape not in ((nlist.capacity,), (nlist.count,)):
        raise ValidationError(
            f"d_grad must have capacity ({nlist.capacity}) or count "
            f"({nlist.count}) entries, got {d_grad.shape}"
        )
    dev = torch.device("cuda")

    def to_dev(a, dtype):
        if isinstance(a, np.ndarray):
            return torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)
        return a.to(dtype=dtype).contiguous()

    pairs = to_dev(nlist.pairs, torch.int32)
    deltas = to_dev(nlist.deltas, torch.float64)
    dists = to_dev(nlist.distances, torch.float64)
    g = torch.as_tensor(np.ascontiguousarray(d_grad[: nlist.count])).to(dev)
    tangent = torch.as_tensor(np.ascontiguousarray(position_tangent)).to(dev)
    grad = torch.empty((nlist.n_atoms, 3), dtype=torch.float64, device=dev)
    dtan = torch.empty(nlist.capacity, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    rc = lib.nnp_distance_pullback_second(
        _lib.ptr(pairs), _lib.ptr(deltas), _lib.ptr(dists), _lib.ptr(g), _lib.ptr(tangent), nlist.count,
        nlist.capacity, nlist.n_atoms, _lib.ptr(grad), _lib.ptr(dtan), _lib.ptr(flag), _lib.current_stream())
    _lib.check(rc, "nnp_distance_pullback_second")
    bad = int(flag.item())
    if bad != 0x7F7F7F7F:
        i, j = (int(x) for x in pairs[bad - 1].tolist())
        raise NumericError(f"zero-distance pair ({i}, {j}) has no defined distance direction")
    return grad.cpu().numpy(), dtan.cpu().numpy()

