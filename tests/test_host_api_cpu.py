"""Host-side logic that needs no GPU: validation rules, strategy planning, radial tables, and
that the C-ABI library loads and exports every symbol include/nnp_b200.h declares."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import _lib, neighbors
from oracle import neighbors_oracle as O
from oracle import tensornet_oracle as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_are_exported():
    header = open(os.path.join(ROOT, "include", "nnp_b200.h")).read()
    declared = set(re.findall(r"\b(nnp_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations found"
    lib = ctypes.CDLL(_lib.LIB_PATH)        # load only; no compute call without a GPU
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in nnp_b200.h but not exported"
    assert set(_lib.EXPORTED_SYMBOLS) <= declared
    assert lib.nnp_version() == 102


def test_ctypes_struct_layouts_match_the_library():
    """The ctypes mirrors of the ABI structs have the size the library was compiled with (a field
    added on one side only would silently shift every later pointer)."""
    lib = ctypes.CDLL(_lib.LIB_PATH)
    assert lib.nnp_abi_sizeof(0) == ctypes.sizeof(_lib.NlParams)
    assert lib.nnp_abi_sizeof(1) == ctypes.sizeof(_lib.TnModel)
    assert lib.nnp_abi_sizeof(2) == ctypes.sizeof(_lib.PriorParams)
    assert lib.nnp_abi_sizeof(3) == -1


def test_workspace_queries_and_validation_run_on_host():
    lib = _lib.load()
    p = _lib.NlParams()
    p.n_atoms, p.n_samples, p.capacity, p.strategy, p.max_cells = 100, 1, 1000, 1, 64
    p.cutoff_lower, p.cutoff_upper = 0.0, 5.0
    need = ctypes.c_size_t(0)
    assert lib.nnp_nl_workspace_bytes(ctypes.byref(p), ctypes.byref(need)) == 0 and need.value > 0
    p.cutoff_lower = 6.0
    assert lib.nnp_nl_workspace_bytes(ctypes.byref(p), ctypes.byref(need)) == _lib.NNP_ERR_INVALID
    assert b"cutoff" in lib.nnp_last_error()
    with pytest.raises(P.ValidationError):
        _lib.check(_lib.NNP_ERR_INVALID, "x")


def test_product_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.ExtensionError, match="no CPU fallback"):
        P.build_neighbor_list(P.build_system([[0.0, 0, 0], [1.0, 0, 0]], [1, 1]),
                              P.NeighborSpec(cutoff_upper=2.0, capacity=4))
    with pytest.raises(P.ExtensionError):
        P.TensorNet(embedding_dimension=32)


def test_spec_box_and_system_validation():
    with pytest.raises(P.ValidationError):
        P.NeighborSpec(cutoff_upper=1.0, cutoff_lower=1.0, capacity=4)
    with pytest.raises(P.ValidationError):
        P.NeighborSpec(cutoff_upper=1.0, capacity=0)
    with pytest.raises(P.ValidationError):
        P.NeighborSpec(cutoff_upper=1.0, capacity=4, strategy="magic")
    assert P.capacity_heuristic(100, 64) == 6400
    with pytest.raises(P.ValidationError, match="lower triangular"):
        P.Box.triclinic([[5.0, 1.0, 0], [0, 5.0, 0], [0, 0, 5.0]])
    with pytest.raises(P.ValidationError, match="not reduced"):
        P.Box.triclinic([[5.0, 0, 0], [3.0, 5.0, 0], [0, 0, 5.0]])
    with pytest.raises(P.ValidationError, match="non-contiguous batch"):
        P.build_system(np.zeros((3, 3)), [1, 1, 1], batch=[0, 2, 2])
    with pytest.raises(P.ValidationError, match="length mismatch"):
        P.build_system(np.zeros((3, 3)), [1, 1])
    s = P.build_system(np.zeros((3, 3)), [1, 1, 1], batch=[0, 0, 1])
    assert s.n_samples == 2 and s.sample_sizes().tolist() == [2, 1]
    with pytest.raises(ValueError):
        s.positions[0, 0] = 1.0                      # inputs are immutable
    box = P.Box.triclinic([[9.0, 0, 0], [1.5, 8.5, 0], [-2.0, 1.0, 9.5]])
    assert np.array_equal(box.perpendicular_widths(), O.perpendicular_widths(box.vectors))


def test_minimum_image_property(rng):
    box = P.Box.triclinic([[9.0, 0, 0], [1.5, 8.5, 0], [-2.0, 1.0, 9.5]])
    d = (rng.uniform(-1, 1, (200, 3))) @ box.vectors
    red = np.linalg.norm(P.minimum_image(d, box), axis=1)
    shifts = np.array([(i, j, k) for i in (-1, 0, 1) for j in (-1, 0, 1) for k in (-1, 0, 1)]) @ box.vectors
    best = np.sqrt(((d[None] + shifts[:, None]) ** 2).sum(-1)).min(0)
    assert np.max(np.abs(red - best)) < 1e-12


def test_strategy_planning():
    box = P.Box.cubic(62.23)
    code, dims, max_cells, notes = neighbors.plan_strategy(23558, box, 5.0, "auto")
    assert code == _lib.STRATEGY_CELL and dims == (12, 12, 12) and max_cells == 1728 and notes == ()
    code, dims, _, notes = neighbors.plan_strategy(100, P.Box.cubic(10.0), 4.9, "cell")
    assert code == _lib.STRATEGY_BRUTE and any("fell back" in n for n in notes)
    assert neighbors.plan_strategy(9999, None, 5.0, "auto")[0] == _lib.STRATEGY_BRUTE
    assert neighbors.plan_strategy(10000, None, 5.0, "auto")[0] == _lib.STRATEGY_CELL
    with pytest.raises(P.ValidationError, match="cutoff too large"):
        neighbors.check_cutoff_against_box(P.Box.cubic(4.0), 2.5)


def test_radial_functions_match_oracle():
    d = np.linspace(0, 5.5, 100)
    for rl, ru in ((0.0, 5.0), (1.0, 4.0)):
        assert np.array_equal(P.cosine_cutoff(d, rl, ru), O.cosine_cutoff(d, rl, ru))
        assert np.array_equal(P.cosine_cutoff_grad(d, rl, ru), O.cosine_cutoff_grad(d, rl, ru))
        m, b = P.expnorm_initial_params(16, rl, ru)
        mo, bo = O.expnorm_initial_params(16, rl, ru)
        assert np.array_equal(m, mo) and np.array_equal(b, bo)
        assert np.array_equal(P.rbf_expnorm(d, m, b, rl), O.rbf_expnorm(d, m, b, rl))
    assert P.cosine_cutoff(np.array([5.0]), 0.0, 5.0)[0] == 0.0 and P.cosine_cutoff(np.array([0.0]), 0.0, 5.0)[0] == 1.0


@pytest.mark.parametrize("rl", [0.0, 0.8])
def test_radial_tables_reproduce_the_mlp(rl):
    """Hermite interpolation of the tables vs the oracle's direct radial MLP and its derivative."""
    cfg = P.TNConfig(embedding_dimension=32, num_layers=2, num_rbf=16, cutoff_lower=rl, cutoff_upper=4.5)
    params = P.init_params(cfg, 7)
    tables, u_min, u_step, err = P.build_radial_tables(params, cfg)
    assert tables.shape == (3, cfg.num_knots, 2, 3, 32) and err < 1e-6
    d = np.random.default_rng(0).uniform(max(rl, 0.0), 4.5, 4000)
    u = np.exp(rl - d)
    x = (u - u_min) / u_step
    k = np.clip(np.floor(x).astype(int), 0, cfg.num_knots - 2)
    t = (x - k)[:, None, None]
    a, b = tables.astype(np.float64)[:, k], tables.astype(np.float64)[:, k + 1]   # [tables, edges, 2, 3, C]
    t2, t3 = t * t, t * t * t
    val = ((2 * t3 - 3 * t2 + 1) * a[:, :, 0] + (t3 - 2 * t2 + t) * a[:, :, 1]
           + (-2 * t3 + 3 * t2) * b[:, :, 0] + (t3 - t2) * b[:, :, 1])
    dval = ((6 * t2 - 6 * t) * a[:, :, 0] + (3 * t2 - 4 * t + 1) * a[:, :, 1]
            + (-6 * t2 + 6 * t) * b[:, :, 0] + (3 * t2 - 2 * t) * b[:, :, 1]) / u_step * (-u)[:, None, None]
    rho = O.rbf_expnorm(d, params["rbf_means"], params["rbf_betas"], rl)
    drho = O.rbf_expnorm_dd(d, params["rbf_means"], params["rbf_betas"], rl)
    for l in range(2):
        ft, cache = T.radial_mlp(params, l, rho)
        dft = T.radial_mlp_dd(params, l, rho, drho, cache)
        ref = ft.reshape(-1, 32, 3).transpose(0, 2, 1)
        dref = dft.reshape(-1, 32, 3).transpose(0, 2, 1)
        assert np.max(np.abs(val[l + 1] - ref)) < 2e-6 * np.max(np.abs(ref))
        assert np.max(np.abs(dval[l + 1] - dref)) < 2e-4 * np.max(np.abs(dref))
    dp = np.stack([rho @ params["dp_w"][j].T + params["dp_b"][j] for j in range(3)], 1)
    assert np.max(np.abs(val[0] - dp)) < 2e-6 * np.max(np.abs(dp))


def test_config_validation_and_params():
    with pytest.raises(P.ValidationError):
        P.TNConfig(embedding_dimension=48)
    with pytest.raises(P.ValidationError):
        P.TNConfig(std=0.0)
    cfg = P.TNConfig(embedding_dimension=64, num_layers=1)
    a, b = P.init_params(cfg, 3), P.init_params(cfg, 3)
    assert all(np.array_equal(a[k], b[k]) for k in a)
    assert a["l0_t_w"].shape == (6, 64, 64) and a["h1_w"].shape == (32, 64)
