"""TensorNet energy-and-forces model behind the reference's call shapes.

Two call shapes over one implementation:

* ``TensorNet.forward(z, pos, batch=None, box=None) -> (energy[n_samples], forces[N, 3])``
  -- the upstream call shown in PAPER.md:143-150; tensors in, CUDA tensors out;
* ``TensorNet.evaluate(system, neighbors=None, forces=True) -> EnergyForces`` -- the in-package
  analogue of ``GraphPotential.evaluate`` (graphnet.py:567-580).

Constructor arguments use the ``GNConfig`` names (graphnet.py:56-83).  The arithmetic is the
TensorNet of SURVEY.md Appendix A; every kernel lives in ``libnnp_b200.so`` (csrc/tn_kernels.cu).
One step = neighbor search + forward + analytic force sweep, enqueued without host
synchronisation and replayed as one CUDA graph per input shape.  Overflow of the fixed-capacity
neighbor structure is detected after the step and answered like ``build_with_auto_capacity``
(neighbors.py:238-247): grow to max(required, 2x) and run again.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, replace
from typing import Dict, Optional

import numpy as np

from . import _lib
from .errors import CapacityError, NumericError, ValidationError
from .neighbors import (
    NeighborEngine, NeighborList, capacity_heuristic, check_cutoff_against_box, plan_strategy,
)
from .radial import expnorm_initial_params, rbf_expnorm_of_u
from .system import Box, EnergyForces, System

_SUPPORTED_CHANNELS = (32, 64, 128)


@dataclass(frozen=True)
class TNConfig:
    """Hyper-parameters; field names follow GNConfig (graphnet.py:59-69)."""

    embedding_dimension: int = 128
    num_layers: int = 2
    num_rbf: int = 32
    cutoff_lower: float = 0.0
    cutoff_upper: float = 5.0
    max_z: int = 100
    activation: str = "silu"
    trainable_rbf: bool = False
    static_shapes: bool = True
    mean: float = 0.0
    std: float = 1.0
    max_num_neighbors: int = 64
    num_knots: int = 512

    def __post_init__(self):
        if self.embedding_dimension not in _SUPPORTED_CHANNELS:
            raise ValidationError(
                f"embedding_dimension must be one of {_SUPPORTED_CHANNELS} for the CUDA kernels"
            )
        if self.num_rbf < 1:
            raise ValidationError("embedding_dimension and num_rbf must be >= 1")
        if not 0 <= self.num_layers <= _lib.TN_MAX_LAYERS:
            raise ValidationError(f"num_layers must be in [0, {_lib.TN_MAX_LAYERS}]")
        if not 0.0 <= self.cutoff_lower < self.cutoff_upper:
            raise ValidationError("cutoffs must satisfy 0 <= lower < upper")
        if self.max_z < 1:
            raise ValidationError("max_z must be >= 1")
        if self.activation != "silu":
            raise ValidationError(f"unsupported activation {self.activation!r}")
        if self.std <= 0:
            raise ValidationError("std must be positive")
        if self.num_knots < 16:
            raise ValidationError("num_knots must be >= 16")


def init_params(config: TNConfig, seed: int = 0) -> Dict[str, np.ndarray]:
    """Deterministic random weights in the style of graphnet.py:175-222: ``default_rng(seed)``,
    linears U(+-1/sqrt(fan_in)), embedding N(0, 1), LayerNorm gamma = 1, beta = 0."""
    rng = np.random.default_rng(seed)
    C, K, L = config.embedding_dimension, config.num_rbf, config.num_layers
    H = max(C // 2, 1)

    def lin(out_f, in_f, bias=True):
        bound = 1.0 / np.sqrt(in_f)
        w = rng.uniform(-bound, bound, (out_f, in_f))
        return (w, rng.uniform(-bound, bound, out_f)) if bias else w

    p: Dict[str, np.ndarray] = {}
    p["emb"] = rng.standard_normal((config.max_z, C))
    p["emb2_w"], p["emb2_b"] = lin(C, 2 * C)
    dp = [lin(C, K) for _ in range(3)]
    p["dp_w"] = np.stack([w for w, _ in dp])
    p["dp_b"] = np.stack([b for _, b in dp])
    p["init_norm_g"], p["init_norm_b"] = np.ones(C), np.zeros(C)
    p["es0_w"], p["es0_b"] = lin(2 * C, C)
    p["es1_w"], p["es1_b"] = lin(3 * C, 2 * C)
    p["et_w"] = np.stack([lin(C, C, bias=False) for _ in range(3)])
    for l in range(L):
        p[f"l{l}_s0_w"], p[f"l{l}_s0_b"] = lin(C, K)
        p[f"l{l}_s1_w"], p[f"l{l}_s1_b"] = lin(2 * C, C)
        p[f"l{l}_s2_w"], p[f"l{l}_s2_b"] = lin(3 * C, 2 * C)
        p[f"l{l}_t_w"] = np.stack([lin(C, C, bias=False) for _ in range(6)])
    p["out_norm_g"], p["out_norm_b"] = np.ones(3 * C), np.zeros(3 * C)
    p["lin_w"], p["lin_b"] = lin(C, 3 * C)
    p["h1_w"], p["h1_b"] = lin(H, C)
    bound = 1.0 / np.sqrt(H)
    p["h2_w"] = rng.uniform(-bound, bound, H)
    p["h2_b"] = np.array(rng.uniform(-bound, bound))
    p["rbf_means"], p["rbf_betas"] = expnorm_initial_params(K, config.cutoff_lower, config.cutoff_upper)
    return p


def _silu(x):
    return x / (1.0 + np.exp(-x))


def _silu_grad(x):
    s = 1.0 / (1.0 + np.exp(-x))
    return s * (1.0 + x * (1.0 - s))


def build_radial_tables(params: Dict[str, np.ndarray], config: TNConfig):
    """Tabulate every distance-only function of the model on knots in u = exp(r_l - d).

    The distance projections of the embedding and the radial MLP of each interaction layer
    depend on the edge only through d, so they are 1-D functions R -> R^{3C}; the expnorm basis
    is a set of equal-width Gaussians in u, which makes u the natural abscissa (uniform knots
    resolve every basis function equally).  Values and u-derivatives are computed in float64
    (derivative by forward mode through the MLP); the device evaluates the cubic Hermite
    interpolant of a knot interval from the data of its two knots:
    ``tables[t, k, p, j, c]`` = value (p = 0) or slope times the knot spacing (p = 1) at knot k of
    output j of channel c.  Returns (tables float32, u_min, u_step, max interpolation error measured at the
    interval midpoints relative to the largest table value).
    """
    C, K, L, nk = config.embedding_dimension, config.num_rbf, config.num_layers, config.num_knots
    u_min = float(np.exp(config.cutoff_lower - config.cutoff_upper))
    u_step = (1.0 - u_min) / (nk - 1)
    means, betas = params["rbf_means"], params["rbf_betas"]

    def evaluate(u):
        rho, drho = rbf_expnorm_of_u(u, means, betas)                   # [n, K]
        out = []
        vals = np.stack([rho @ params["dp_w"][j].T + params["dp_b"][j] for j in range(3)], 1)
        ders = np.stack([drho @ params["dp_w"][j].T for j in range(3)], 1)
        out.append((vals, ders))                                        # [n, 3, C]
        for l in range(L):
            a0 = rho @ params[f"l{l}_s0_w"].T + params[f"l{l}_s0_b"]
            a1 = _silu(a0) @ params[f"l{l}_s1_w"].T + params[f"l{l}_s1_b"]
            a2 = _silu(a1) @ params[f"l{l}_s2_w"].T + params[f"l{l}_s2_b"]
            t = drho @ params[f"l{l}_s0_w"].T
            t = (t * _silu_grad(a0)) @ params[f"l{l}_s1_w"].T
            t = (t * _silu_grad(a1)) @ params[f"l{l}_s2_w"].T
            f = _silu(a2).reshape(-1, C, 3).transpose(0, 2, 1)          # [n, 3, C]
            df = (t * _silu_grad(a2)).reshape(-1, C, 3).transpose(0, 2, 1)
            out.append((f, df))
        return out

    knots = u_min + u_step * np.arange(nk)
    at_knots = evaluate(knots)
    tables = np.empty((L + 1, nk, 2, 3, C), dtype=np.float64)
    for t, (f, df) in enumerate(at_knots):
        tables[t, :, 0] = f
        tables[t, :, 1] = df * u_step
    # interpolation error at the interval midpoints (Hermite weights at x = 1/2)
    mid = evaluate(knots[:-1] + 0.5 * u_step)
    err = 0.0
    for t, (f, _) in enumerate(mid):
        c = tables[t]
        interp = 0.5 * (c[:-1, 0] + c[1:, 0]) + 0.125 * (c[:-1, 1] - c[1:, 1])
        err = max(err, float(np.max(np.abs(interp - f)) / max(np.max(np.abs(c[:, 0])), 1e-30)))
    return tables.astype(np.float32), u_min, u_step, err


def monomial_tables(tables: np.ndarray) -> np.ndarray:
    """Knot data [T, nk, 2, 3, C] -> per-interval monomial coefficients [T, nk-1, 4, 3, C] of the
    same cubic Hermite interpolants (expanded in float64)."""
    t = tables.astype(np.float64)
    f0, f1, m0, m1 = t[:, :-1, 0], t[:, 1:, 0], t[:, :-1, 1], t[:, 1:, 1]
    mono = np.stack([f0, m0, 3.0 * (f1 - f0) - 2.0 * m0 - m1, 2.0 * (f0 - f1) + m0 + m1], axis=2)
    return mono.astype(np.float32)


class _Plan:
    """Everything that is fixed for one input shape: buffers, neighbor engine, graph."""

    __slots__ = ("key", "n", "n_samples", "capacity", "engine", "workspace", "z", "batch", "pos32",
                 "pos64", "energy", "forces", "per_atom", "graph", "notes", "box", "batch_is_zero", "proj",
                 "io")


class TensorNet:
    """TensorNet potential on one B200.  See the module docstring for the call shapes."""

    def __init__(self, config: Optional[TNConfig] = None, params: Optional[Dict[str, np.ndarray]] = None,
                 seed: int = 0, device="cuda", use_graph: bool = True, strategy: str = "auto",
                 embed_projection: Optional[bool] = None, gemm_mode: int = 0, **config_kwargs):
        torch = _lib.require_cuda()
        self._torch = torch
        self.lib = _lib.load()
        if config is None:
            config = TNConfig(**config_kwargs)
        elif config_kwargs:
            config = replace(config, **config_kwargs)
        self.config = config
        self.params = params if params is not None else init_params(config, seed)
        self.device = torch.device(device)
        self.use_graph = use_graph
        self.strategy = strategy
        self.embed_projection = embed_projection
        if gemm_mode not in (0, 1, 3, 5, 8):
            raise ValidationError("gemm_mode must be 0 (library default), 5, 3, 1 or 8 (FFMA)")
        self.gemm_mode = gemm_mode      # per model, so concurrent models do not share a switch
        self._plans: Dict[tuple, _Plan] = {}
        self._last_plan: Optional[_Plan] = None
        self._z_key, self._z_proj = None, False
        self._b_key = None
        self._capacity_hint: Dict[tuple, int] = {}
        self._upload()

    # ------------------------------------------------------------------ weights
    def _upload(self) -> None:
        torch, cfg, P = self._torch, self.config, self.params
        C = cfg.embedding_dimension
        tables, u_min, u_step, err = build_radial_tables(P, cfg)
        self.table_error = err
        keep = {}

        def dev(name, a):
            t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).to(self.device)
            keep[name] = t
            return t.data_ptr()

        m = _lib.TnModel()
        m.channels, m.num_rbf, m.num_layers = C, cfg.num_rbf, cfg.num_layers
        m.max_z, m.num_knots = cfg.max_z, cfg.num_knots
        m.cutoff_lower, m.cutoff_upper = cfg.cutoff_lower, cfg.cutoff_upper
        m.u_min, m.u_step = u_min, u_step
        m.mean, m.std, m.h2_b = cfg.mean, cfg.std, float(P["h2_b"])
        # Z_e = emb2([emb[z_i] | emb[z_j]]) hoisted into two species tables (App. A, last bullet)
        Wa, Wb = P["emb2_w"][:, :C], P["emb2_w"][:, C:]
        m.z_recv = dev("z_recv", P["emb"] @ Wa.T)
        m.z_send = dev("z_send", P["emb"] @ Wb.T + P["emb2_b"])
        m.tables = dev("tables", tables)
        m.tables_mono = dev("tables_mono", monomial_tables(tables))
        m.init_norm_g, m.init_norm_b = dev("ing", P["init_norm_g"]), dev("inb", P["init_norm_b"])

        def gemm_weight(slot, name, w):
            slot.w = dev(name, w)

        gemm_weight(m.es0_w, "es0_w", P["es0_w"])
        gemm_weight(m.es0_wT, "es0_wT", P["es0_w"].T)
        gemm_weight(m.es1_w, "es1_w", P["es1_w"])
        gemm_weight(m.es1_wT, "es1_wT", P["es1_w"].T)
        m.es0_b, m.es1_b = dev("es0_b", P["es0_b"]), dev("es1_b", P["es1_b"])
        for k in range(3):
            gemm_weight(m.et_w[k], f"et_w{k}", P["et_w"][k])
            gemm_weight(m.et_wT[k], f"et_wT{k}", P["et_w"][k].T)
        for l in range(cfg.num_layers):
            for k in range(6):
                gemm_weight(m.layer_t_w[l][k], f"t_w{l}_{k}", P[f"l{l}_t_w"][k])
                gemm_weight(m.layer_t_wT[l][k], f"t_wT{l}_{k}", P[f"l{l}_t_w"][k].T)
        m.out_norm_g, m.out_norm_b = dev("ong", P["out_norm_g"]), dev("onb", P["out_norm_b"])
        gemm_weight(m.lin_w, "lin_w", P["lin_w"])
        gemm_weight(m.lin_wT, "lin_wT", P["lin_w"].T)
        gemm_weight(m.h1_w, "h1_w", P["h1_w"])
        gemm_weight(m.h1_wT, "h1_wT", P["h1_w"].T)
        m.lin_b, m.h1_b = dev("lin_b", P["lin_b"]), dev("h1_b", P["h1_b"])
        m.h2_w = dev("h2_w", P["h2_w"])
        # embedding reverse by node-level projection (written for 128 channels and 32 basis functions;
        # other shapes keep the per-channel edge kernel)
        self._proj_capable = (C == 128 and cfg.num_rbf == 32 and self.embed_projection is not False
                              and os.environ.get("NNP_EMBED_PROJ", "1") != "0")
        if self.embed_projection and not self._proj_capable:
            raise ValidationError("embed_projection needs embedding_dimension=128 and num_rbf=32")
        m.embed_projection = 0          # set per step from the plan (see _use_projection)
        m.gemm_mode = self.gemm_mode
        m.dp_wT = dev("dp_wT", np.transpose(P["dp_w"], (0, 2, 1)))      # [3][K][C]
        m.dp_b = dev("dp_b", P["dp_b"])
        m.rbf_means, m.rbf_betas = dev("rbf_means", P["rbf_means"]), dev("rbf_betas", P["rbf_betas"])
        self._model = m
        self._weights = keep

    # ---------------------------------------------------------------- weights on disk
    def save(self, path) -> None:
        """Write config and weights (structio.save_weights)."""
        from .structio import save_weights

        save_weights(path, self.config, self.params)

    @classmethod
    def load(cls, path, **kwargs) -> "TensorNet":
        """A model from a file written by ``save``."""
        from .structio import load_weights

        config, params = load_weights(path)
        return cls(config=config, params=params, **kwargs)

    # -------------------------------------------------------------------- plans
    def neighbor_capacity(self, n_atoms: int) -> int:
        """Directed rows incl. self loops: 2*N*max_num_neighbors, as compose.py:59-71 sizes a
        full list (capacity_heuristic doubled)."""
        return 2 * capacity_heuristic(n_atoms, self.config.max_num_neighbors)

    def _choose_strategy(self, n: int, n_samples: int, box: Optional[Box]) -> str:
        if self.strategy != "auto":
            return self.strategy
        # small samples: all-pairs inside each sample; otherwise the cell list
        return "brute" if n / max(n_samples, 1) < 1024 else "cell"

    PROJECTION_MIN_ATOMS = 1024   # measured (tools/proj_threshold.py): even at 1 000 atoms, 6 % faster at 2 489; slower at 22
    PROJECTION_MAX_SPECIES = 4

    def _use_projection(self, species, n: int, count: bool = True) -> bool:
        """Whether a step over these species runs the node-projected embedding reverse: forced on
        by ``embed_projection=True``; otherwise for systems of at least PROJECTION_MIN_ATOMS atoms
        with at most four distinct species (the device falls back by itself if a projected plan is
        ever fed more, so this is a cost decision, not a correctness one)."""
        if not self._proj_capable:
            return False
        if self.embed_projection:
            return True
        if n < self.PROJECTION_MIN_ATOMS:
            return False
        if not count:
            return True
        torch = self._torch
        if isinstance(species, torch.Tensor):
            if species.is_cuda:
                return int(torch.unique(species).numel()) <= self.PROJECTION_MAX_SPECIES
            species = species.numpy()
        present = np.bincount(np.asarray(species).astype(np.int64, copy=False).ravel(), minlength=1)
        return int(np.count_nonzero(present)) <= self.PROJECTION_MAX_SPECIES

    def _species_checked(self, z_t, n: int, check: bool, remember: bool = False) -> bool:
        """Range check of the species codes (on whichever side they live: host tensors cost no
        device reduction and no synchronisation) and the projection decision.  Both depend on the
        codes only, so the answer is remembered for a tensor that has not been written since
        (same storage and version counter), as in an MD loop; arrays that torch cannot track
        (numpy inputs) are checked every time."""
        key = (z_t.data_ptr(), z_t._version, n, str(z_t.device), check) if remember else None
        if key is not None and key == self._z_key:
            return self._z_proj
        if check:
            z_min, z_max = (int(v) for v in self._torch.aminmax(z_t))
            if z_min < 0:
                raise ValidationError(f"species codes must be >= 0, got {z_min}")
            if z_max >= self.config.max_z:
                raise ValidationError(
                    f"species code {z_max} is out of range for max_z={self.config.max_z}")
        proj = self._use_projection(z_t, n, count=check)
        self._z_key, self._z_proj = key, proj
        return proj

    def _batch_checked(self, batch_t, n: int, n_samples: int, remember: bool = False) -> None:
        """Sample codes must start at 0, never decrease, and stay below ``n_samples`` (what
        ``build_system`` enforces in the reference, system.py): ``k_prep_nodes`` writes
        ``sample_ptr[code]`` and the per-sample search bisects the codes.  Empty samples (gaps in
        the codes) are allowed, as ``segment_sum`` allows them.  Remembered per unmodified tensor."""
        key = (batch_t.data_ptr(), batch_t._version, n, n_samples, str(batch_t.device)) if remember else None
        if key is not None and key == self._b_key:
            return
        torch = self._torch
        if batch_t.dtype.is_floating_point or batch_t.dtype == torch.bool:
            raise ValidationError("batch codes must be integers")
        first, last = int(batch_t[0]), int(batch_t[-1])
        if first < 0 or last >= n_samples:
            raise ValidationError(
                f"batch codes must lie in [0, n_samples): got first {first}, last {last}, n_samples {n_samples}")
        if n > 1 and bool((batch_t[1:] < batch_t[:-1]).any()):
            raise ValidationError("batch codes must be non-decreasing (atoms of one sample contiguous)")
        self._b_key = key

    def _plan(self, n: int, n_samples: int, box: Optional[Box], capacity: int, pos_is_f32: bool,
              proj: bool = False) -> _Plan:
        torch, cfg = self._torch, self.config
        box_key = None if box is None else (box.kind, box.vectors.tobytes())
        key = (n, n_samples, capacity, box_key, pos_is_f32, proj)
        plan = self._plans.get(key)
        if plan is not None:
            return plan
        check_cutoff_against_box(box, cfg.cutoff_upper)
        code, dims, max_cells, notes = plan_strategy(
            n, box, cfg.cutoff_upper, self._choose_strategy(n, n_samples, box))
        flags = (_lib.NL_FULL_LIST | _lib.NL_SELF_LOOPS | _lib.NL_F32_OUT | _lib.NL_NO_PAD
                 | (_lib.NL_RENUMBER if code == _lib.STRATEGY_CELL else 0))
        plan = _Plan()
        plan.key, plan.n, plan.n_samples, plan.capacity, plan.box = key, n, n_samples, capacity, box
        plan.notes = notes
        plan.proj = proj
        plan.engine = NeighborEngine(n, n_samples, capacity, box, cfg.cutoff_lower, cfg.cutoff_upper,
                                     code, dims, max_cells, flags, device=self.device,
                                     want_row_ptr=True, want_order=True)
        need = ctypes.c_size_t(0)
        self._model.embed_projection = int(proj)
        _lib.check(self.lib.nnp_tn_workspace_bytes(ctypes.byref(self._model), n, capacity, n_samples,
                                                   ctypes.byref(need)), "nnp_tn_workspace_bytes")
        dev = self.device
        plan.workspace = torch.empty(need.value, dtype=torch.uint8, device=dev)
        plan.z = torch.zeros(n, dtype=torch.int32, device=dev)
        plan.batch = torch.zeros(n, dtype=torch.int32, device=dev)
        plan.batch_is_zero = True
        plan.pos32 = torch.zeros((n, 3), dtype=torch.float32, device=dev) if pos_is_f32 else None
        plan.pos64 = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        plan.energy = torch.zeros(n_samples, dtype=torch.float32, device=dev)
        plan.forces = torch.zeros((n, 3), dtype=torch.float32, device=dev)
        plan.per_atom = torch.zeros(n, dtype=torch.float32, device=dev)
        plan.graph = None
        plan.io = None
        self._plans[key] = plan
        return plan

    def _enqueue(self, plan: _Plan, want_forces: bool = True) -> None:
        """Enqueue one whole step on the current stream; no allocation, no synchronisation."""
        stream = _lib.current_stream()
        if plan.pos32 is not None:
            _lib.check(self.lib.nnp_f32_to_f64(_lib.ptr(plan.pos32), _lib.ptr(plan.pos64),
                                               3 * plan.n, stream), "nnp_f32_to_f64")
        eng = plan.engine
        eng.build(plan.pos64, plan.batch)
        self._model.embed_projection = int(plan.proj)
        rc = self.lib.nnp_tn_energy_forces(
            ctypes.byref(self._model), plan.n, plan.n_samples, plan.capacity, _lib.ptr(plan.z),
            _lib.ptr(plan.batch), _lib.ptr(eng.order), _lib.ptr(eng.row_ptr), _lib.ptr(eng.pairs),
            _lib.ptr(eng.deltas), _lib.ptr(eng.dists), _lib.ptr(eng.counts), _lib.ptr(plan.energy),
            _lib.ptr(plan.forces) if want_forces else None, _lib.ptr(plan.per_atom),
            _lib.ptr(plan.workspace), plan.workspace.numel(), stream,
        )
        _lib.check(rc, "nnp_tn_energy_forces")

    def _launch(self, plan: _Plan) -> None:
        torch = self._torch
        if not self.use_graph:
            self._enqueue(plan)
            return
        if plan.graph is None:
            self._enqueue(plan)                      # warm-up outside capture
            torch.cuda.synchronize(self.device)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                self._enqueue(plan)
            plan.graph = graph
        plan.graph.replay()

    # ------------------------------------------------------------------ call shapes
    def _as_box(self, box) -> Optional[Box]:
        if box is None or isinstance(box, Box):
            return box if (box is None or box.periodic) else None
        if hasattr(box, "detach"):
            box = box.detach().cpu().numpy()
        return Box.from_matrix(box)

    def forward(self, z, pos, batch=None, box=None, *, n_samples: Optional[int] = None,
                check: bool = True, clone: bool = True):
        """Energies [n_samples] and forces [N, 3] (float32 CUDA tensors).

        ``z`` species codes [N], ``pos`` positions [N, 3] (float32, or float64), ``batch``
        non-decreasing sample codes [N] (default: one sample), ``box`` None or a 3x3 matrix
        with rows a, b, c (lower triangular, system.py:34-38) or a ``Box``.
        ``check=False`` skips the post-step overflow test (and its synchronisation).
        """
        torch = self._torch
        dev = self.device
        pos_t = torch.as_tensor(np.array(pos) if isinstance(pos, np.ndarray) and not pos.flags.writeable else pos)
        if pos_t.dim() != 2 or pos_t.shape[1] != 3:
            raise ValidationError("positions must have shape (N, 3)")
        n = pos_t.shape[0]
        if n < 1:
            raise ValidationError("system must contain at least one atom")
        if pos_t.dtype not in (torch.float32, torch.float64):
            pos_t = pos_t.to(torch.float32)
        z_t = torch.as_tensor(np.array(z) if isinstance(z, np.ndarray) and not z.flags.writeable else z)
        if z_t.shape != (n,):
            raise ValidationError(f"length mismatch: {n} positions but {tuple(z_t.shape)} species")
        if batch is None:
            batch_t, n_samples = None, 1
        else:
            batch_t = torch.as_tensor(np.array(batch) if isinstance(batch, np.ndarray) and not batch.flags.writeable else batch)
            if batch_t.shape != (n,):
                raise ValidationError(f"length mismatch: {n} positions but {tuple(batch_t.shape)} batch codes")
            if n_samples is None:
                n_samples = int(batch_t[-1]) + 1
            if check:
                self._batch_checked(batch_t, n, n_samples, remember=isinstance(batch, torch.Tensor))
        box_obj = self._as_box(box)
        capacity = self._capacity_hint.get((n, n_samples), self.neighbor_capacity(n))
        proj = self._species_checked(z_t, n, check, remember=isinstance(z, torch.Tensor))
        for _ in range(32):
            plan = self._plan(n, n_samples, box_obj, capacity, pos_t.dtype == torch.float32, proj)
            self._last_plan = plan
            # straight into the plan's buffers: one host-to-device copy per input (a dtype change,
            # if any, is made on the way), no intermediate device tensors
            plan.z.copy_(z_t, non_blocking=True)
            if batch_t is not None:
                plan.batch.copy_(batch_t, non_blocking=True)
                plan.batch_is_zero = False
            elif not plan.batch_is_zero:
                plan.batch.zero_()
                plan.batch_is_zero = True
            (plan.pos32 if plan.pos32 is not None else plan.pos64).copy_(pos_t, non_blocking=True)
            self._launch(plan)
            if not check:
                break
            required = int(plan.engine.counts[0].item())      # synchronises
            if required <= plan.capacity:
                break
            capacity = max(required, 2 * plan.capacity)
            self._capacity_hint[(n, n_samples)] = capacity
        else:
            raise CapacityError(required=capacity * 2, capacity=capacity)
        if clone:
            return plan.energy.clone(), plan.forces.clone()
        return plan.energy, plan.forces

    __call__ = forward

    # ------------------------------------------------- host in, host out: one graph, one synchronisation
    def _host_io(self, plan: _Plan, with_batch: bool):
        """Pinned staging buffers of a plan and ONE captured graph that copies the inputs up, runs the
        whole step and copies energies, forces, per-atom energies and the overflow counter down."""
        torch = self._torch
        io = plan.io
        if io is not None and io["with_batch"] == with_batch:
            return io
        pos_dev = plan.pos32 if plan.pos32 is not None else plan.pos64
        pin = lambda t: torch.empty(t.shape, dtype=t.dtype).pin_memory()
        io = {"with_batch": with_batch, "z": pin(plan.z), "batch": pin(plan.batch), "pos": pin(pos_dev),
              "energy": pin(plan.energy), "forces": pin(plan.forces), "per_atom": pin(plan.per_atom),
              "counts": pin(plan.engine.counts)}

        def enqueue():
            plan.z.copy_(io["z"], non_blocking=True)
            if with_batch:
                plan.batch.copy_(io["batch"], non_blocking=True)
            pos_dev.copy_(io["pos"], non_blocking=True)
            self._enqueue(plan)
            io["energy"].copy_(plan.energy, non_blocking=True)
            io["forces"].copy_(plan.forces, non_blocking=True)
            io["per_atom"].copy_(plan.per_atom, non_blocking=True)
            io["counts"].copy_(plan.engine.counts, non_blocking=True)

        io["z"].zero_()
        io["batch"].zero_()
        io["pos"].copy_(pos_dev)                 # a valid configuration for the warm-up run
        io["z"].copy_(plan.z)
        io["batch"].copy_(plan.batch)
        if self.use_graph:
            enqueue()
            torch.cuda.synchronize(self.device)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                enqueue()
            io["run"] = graph.replay
        else:
            io["run"] = enqueue
        plan.io = io
        return io

    def forward_host(self, z, pos, batch=None, box=None, *, n_samples: Optional[int] = None,
                     check: bool = True, copy: bool = True):
        """``forward`` for callers whose data lives on the host (the reference's own call shape:
        numpy in, numpy out): returns ``(energy [n_samples], forces [N, 3])`` as numpy float32 arrays.

        The inputs are written into pinned staging buffers and ONE captured graph does the rest
        (host-to-device copies, neighbor search, forward and force sweep, device-to-host copies of
        the results and of the overflow counter), followed by one stream synchronisation - instead
        of two copies up, a graph, a synchronising counter read and two copies down.
        ``copy=False`` returns views of the pinned result buffers (valid until the next call)."""
        torch = self._torch
        pos_t = torch.as_tensor(np.array(pos) if isinstance(pos, np.ndarray) and not pos.flags.writeable else pos)
        z_t = torch.as_tensor(np.array(z) if isinstance(z, np.ndarray) and not z.flags.writeable else z)
        if pos_t.is_cuda or z_t.is_cuda:
            raise ValidationError("forward_host takes host arrays; use forward() for device tensors")
        if pos_t.dim() != 2 or pos_t.shape[1] != 3:
            raise ValidationError("positions must have shape (N, 3)")
        n = pos_t.shape[0]
        if z_t.shape != (n,):
            raise ValidationError(f"length mismatch: {n} positions but {tuple(z_t.shape)} species")
        if pos_t.dtype not in (torch.float32, torch.float64):
            pos_t = pos_t.to(torch.float32)
        batch_t = None if batch is None else torch.as_tensor(
            np.array(batch) if isinstance(batch, np.ndarray) and not batch.flags.writeable else batch)
        if batch_t is None:
            n_samples = 1
        else:
            if batch_t.shape != (n,):
                raise ValidationError(f"length mismatch: {n} positions but {tuple(batch_t.shape)} batch codes")
            if n_samples is None:
                n_samples = int(batch_t[-1]) + 1
            if check:
                self._batch_checked(batch_t, n, n_samples, remember=isinstance(batch, torch.Tensor))
        box_obj = self._as_box(box)
        proj = self._species_checked(z_t, n, check, remember=isinstance(z, torch.Tensor))
        capacity = self._capacity_hint.get((n, n_samples), self.neighbor_capacity(n))
        plan = self._plan(n, n_samples, box_obj, capacity, pos_t.dtype == torch.float32, proj)
        if plan.graph is None and self.use_graph:
            # first use of this shape: the ordinary path creates (and, on overflow, regrows) the plan
            self.forward(z_t, pos_t, batch_t, box_obj, n_samples=n_samples, check=True, clone=False)
            plan = self._last_plan
        self._last_plan = plan
        io = self._host_io(plan, batch_t is not None)
        io["z"].copy_(z_t)
        if batch_t is not None:
            io["batch"].copy_(batch_t)
            plan.batch_is_zero = False
        elif not plan.batch_is_zero:
            plan.batch.zero_()
            plan.batch_is_zero = True
        io["pos"].copy_(pos_t)
        io["run"]()
        torch.cuda.current_stream().synchronize()
        if check and int(io["counts"][0]) > plan.capacity:
            # overflow: let forward() grow the capacity (it re-runs the step), then answer from the new plan
            self.forward(z_t, pos_t, batch_t, box_obj, n_samples=n_samples, check=True, clone=False)
            return self.forward_host(z, pos, batch, box, n_samples=n_samples, check=check, copy=copy)
        e, f = io["energy"].numpy(), io["forces"].numpy()
        return (e.copy(), f.copy()) if copy else (e, f)

    # ---------------------------------------------------------- resident replay (benchmarks, MD)
    def prepare(self, z, pos, batch=None, box=None, *, n_samples: Optional[int] = None):
        """Run one checked step and return the plan, whose inputs now live in HBM and whose
        graph is captured; ``replay(plan)`` re-runs the whole step (neighbor search included)
        on the resident inputs without touching the host."""
        self.forward(z, pos, batch, box, n_samples=n_samples, check=True, clone=False)
        return self._last_plan

    def replay(self, plan: "_Plan") -> None:
        if plan.graph is not None:
            plan.graph.replay()
        else:
            self._enqueue(plan)

    def enqueue_eager(self, plan: "_Plan") -> None:
        """The same step as ``replay`` but launched kernel by kernel (profiling, launch counts)."""
        self._enqueue(plan)

    def last_per_atom_energy(self, n: int, n_samples: int = 1):
        last = self._last_plan
        if last is not None and last.n == n and last.n_samples == n_samples:
            return last.per_atom
        for key, plan in self._plans.items():
            if key[0] == n and key[1] == n_samples:
                return plan.per_atom
        return None

    def evaluate(self, system: System, neighbors: Optional[NeighborList] = None,
                 forces: bool = True) -> EnergyForces:
        """``GraphPotential.evaluate``-shaped call (graphnet.py:567-580): numpy float64 in and
        out.  With ``neighbors`` (a device list built with ``full_list=True`` and
        ``include_self_loops=True``) the step runs on that list; otherwise it builds its own."""
        torch = self._torch
        if int(system.species.max()) >= self.config.max_z:
            raise ValidationError(
                f"species code {int(system.species.max())} is out of range for "
                f"max_z={self.config.max_z}")
        if neighbors is None:
            e, f = self.forward_host(system.species, system.positions, system.batch, system.box,
                                     n_samples=system.n_samples)
            per_atom = self._last_plan.io["per_atom"].numpy().copy()
            return EnergyForces(e, f if forces else None, per_atom)
        spec = neighbors.spec
        if not spec.full_list:
            raise ValidationError(
                "graph forward needs a full neighbor list (messages flow both ways); "
                "build with full_list=True")
        if not spec.include_self_loops:
            raise ValidationError("TensorNet needs self loops; build with include_self_loops=True")
        if spec.cutoff_upper != self.config.cutoff_upper or spec.cutoff_lower != self.config.cutoff_lower:
            raise ValidationError(
                f"cutoff mismatch: neighbor list has ({spec.cutoff_lower}, {spec.cutoff_upper}), "
                f"model expects ({self.config.cutoff_lower}, {self.config.cutoff_upper})")
        if not neighbors.on_device or neighbors.row_ptr is None:
            raise ValidationError("evaluate() needs a device neighbor list from build_neighbor_list")
        if not spec.deterministic:
            # k_edge_rev bisects the sender's row by column, which needs rows sorted by sender
            raise ValidationError(
                "TensorNet needs rows sorted by sender: build the list with deterministic=True")
        dev = self.device
        n, ns, cap = system.n_atoms, system.n_samples, neighbors.capacity
        z = torch.as_tensor(np.ascontiguousarray(system.species, dtype=np.int32)).to(dev)
        b = torch.as_tensor(np.ascontiguousarray(system.batch, dtype=np.int32)).to(dev)
        need = ctypes.c_size_t(0)
        self._model.embed_projection = int(self._use_projection(system.species, n))
        _lib.check(self.lib.nnp_tn_workspace_bytes(ctypes.byref(self._model), n, cap, ns,
                                                   ctypes.byref(need)), "nnp_tn_workspace_bytes")
        ws = torch.empty(need.value, dtype=torch.uint8, device=dev)
        energy = torch.zeros(ns, dtype=torch.float32, device=dev)
        force_t = torch.zeros((n, 3), dtype=torch.float32, device=dev) if forces else None
        per_atom = torch.zeros(n, dtype=torch.float32, device=dev)
        deltas = neighbors.deltas.to(torch.float32).contiguous()
        dists = neighbors.distances.to(torch.float32).contiguous()
        rc = self.lib.nnp_tn_energy_forces(
            ctypes.byref(self._model), n, ns, cap, _lib.ptr(z), _lib.ptr(b), None,
            _lib.ptr(neighbors.row_ptr), _lib.ptr(neighbors.pairs), _lib.ptr(deltas), _lib.ptr(dists),
            None, _lib.ptr(energy), _lib.ptr(force_t), _lib.ptr(per_atom), _lib.ptr(ws), ws.numel(),
            _lib.current_stream())
        _lib.check(rc, "nnp_tn_energy_forces")
        out_f = force_t.cpu().numpy() if forces else None
        if out_f is not None and not np.all(np.isfinite(out_f)):
            raise NumericError("non-finite forces")
        return EnergyForces(energy.cpu().numpy(), out_f, per_atom.cpu().numpy())
