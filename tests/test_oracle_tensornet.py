"""Self-consistency of the TensorNet CPU oracle (parity unpinned: no reference TensorNet exists).

Replicates the reference's model-test methodology on the restatement:
scripted/independent re-evaluation (test_graphnet.py:98-126), forces vs central differences
(:207-229), invariances (:366-473), padding inertness (:299-363), batch independence.
"""

import numpy as np
import pytest

from oracle import neighbors_oracle as O
from oracle import tensornet_oracle as T


def make_case(rng, n=11, periodic=False, C=8, K=6, L=2, ru=4.0, rl=0.0):
    cfg = T.OracleConfig(embedding_dimension=C, num_layers=L, num_rbf=K, cutoff_lower=rl,
                         cutoff_upper=ru, max_z=10, mean=0.3, std=1.7)
    params = T.init_params(cfg, seed=int(rng.integers(1 << 30)))
    box = np.array([[9.0, 0, 0], [1.5, 8.5, 0], [-2.0, 1.0, 9.5]]) if periodic else None
    pos = rng.uniform(0, 1, (n, 3)) @ box if periodic else rng.uniform(0, 5, (n, 3))
    z = rng.choice([1, 6, 8], n)
    batch = np.repeat([0, 1], [n - n // 2, n // 2])
    return cfg, params, pos, z, batch, box


def lists(pos, batch, box, cfg, capacity=None):
    n = pos.shape[0]
    nl = O.build_neighbor_list(pos, batch, box, cfg.cutoff_upper, capacity or 4 * n * n,
                               cutoff_lower=cfg.cutoff_lower, full_list=True,
                               include_self_loops=True)
    return nl.valid()


def energy(cfg, params, pos, z, batch, box):
    pr, dl, ds = lists(pos, batch, box, cfg)
    return T.energy_forces_compact(params, cfg, z, batch, pr, dl, ds, want_forces=False)[0]


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("L", [0, 1, 2])
def test_two_implementations_agree(rng, periodic, L):
    cfg, params, pos, z, batch, box = make_case(rng, periodic=periodic, L=L)
    pr, dl, ds = lists(pos, batch, box, cfg)
    e1, f1, pa1 = T.energy_forces_torch(params, cfg, z, batch, pos, pr, dl)
    e2, f2, pa2 = T.energy_forces_compact(params, cfg, z, batch, pr, dl, ds)
    assert np.max(np.abs(e1 - e2)) < 1e-10
    assert np.max(np.abs(pa1 - pa2)) < 1e-10
    assert np.max(np.abs(f1 - f2)) < 1e-10
    assert np.max(np.abs(f1)) > 1e-5       # geometry really enters (also at L=0)


def test_lower_cutoff_variant(rng):
    cfg, params, pos, z, batch, box = make_case(rng, rl=0.8)
    pr, dl, ds = lists(pos, batch, box, cfg)
    e1, f1, _ = T.energy_forces_torch(params, cfg, z, batch, pos, pr, dl)
    e2, f2, _ = T.energy_forces_compact(params, cfg, z, batch, pr, dl, ds)
    assert np.max(np.abs(e1 - e2)) < 1e-10 and np.max(np.abs(f1 - f2)) < 1e-10


@pytest.mark.parametrize("periodic", [False, True])
def test_forces_match_central_differences(rng, periodic):
    cfg, params, pos, z, batch, box = make_case(rng, n=8, periodic=periodic)
    pr, dl, ds = lists(pos, batch, box, cfg)
    _, f, _ = T.energy_forces_compact(params, cfg, z, batch, pr, dl, ds)
    h = 1e-4
    fd = np.zeros_like(pos)
    for a in range(pos.shape[0]):
        for k in range(3):
            p, m = pos.copy(), pos.copy()
            p[a, k] += h
            m[a, k] -= h
            fd[a, k] = -(energy(cfg, params, p, z, batch, box).sum()
                         - energy(cfg, params, m, z, batch, box).sum()) / (2 * h)
    assert np.max(np.abs(fd - f)) / np.max(np.abs(f)) < 1e-6


def test_o3_translation_permutation_invariance(rng):
    cfg, params, pos, z, batch, box = make_case(rng)
    pr, dl, ds = lists(pos, batch, box, cfg)
    e0, f0, pa0 = T.energy_forces_compact(params, cfg, z, batch, pr, dl, ds)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    for R in (q, -q, np.diag([1.0, 1.0, -1.0])):            # proper, improper, mirror
        pos2 = pos @ R.T + np.array([1.7, -2.3, 0.9])
        pr2, dl2, ds2 = lists(pos2, batch, None, cfg)
        e1, f1, pa1 = T.energy_forces_compact(params, cfg, z, batch, pr2, dl2, ds2)
        assert np.max(np.abs(pa1 - pa0)) < 1e-10
        assert np.max(np.abs(f1 - f0 @ R.T)) < 1e-10
    # permutation inside each sample
    perm = np.concatenate([rng.permutation(6), 6 + rng.permutation(5)])
    pr3, dl3, ds3 = lists(pos[perm], batch, None, cfg)
    e3, f3, pa3 = T.energy_forces_compact(params, cfg, z[perm], batch, pr3, dl3, ds3)
    assert np.max(np.abs(e3 - e0)) < 1e-10 and np.max(np.abs(f3 - f0[perm])) < 1e-10


def test_capacity_padding_is_inert_and_batches_are_independent(rng):
    cfg, params, pos, z, batch, box = make_case(rng)
    a = lists(pos, batch, box, cfg)
    b = lists(pos, batch, box, cfg, capacity=10 * pos.shape[0] ** 2)
    ea, fa, _ = T.energy_forces_compact(params, cfg, z, batch, *a)
    eb, fb, _ = T.energy_forces_compact(params, cfg, z, batch, *b)
    assert np.array_equal(ea, eb) and np.array_equal(fa, fb)
    first = batch == 0
    pr, dl, ds = lists(pos[first], batch[first], None, cfg)
    e1, f1, _ = T.energy_forces_compact(params, cfg, z[first], batch[first], pr, dl, ds)
    assert abs(e1[0] - ea[0]) < 1e-12 and np.max(np.abs(f1 - fa[first])) < 1e-12


def test_energy_continuous_across_cutoff():
    cfg = T.OracleConfig(embedding_dimension=8, num_layers=1, num_rbf=6, cutoff_upper=4.0, max_z=10)
    params = T.init_params(cfg, 3)
    z, batch = np.array([1, 8, 6]), np.zeros(3, dtype=np.int64)
    jumps = []
    for eps in (1e-3, 1e-4, 1e-5):
        es = []
        for x in (4.0 - eps, 4.0 + eps):
            pos = np.array([[0.0, 0, 0], [x, 0, 0], [1.0, 1.0, 0]])
            es.append(energy(cfg, params, pos, z, batch, None)[0])
        jumps.append(abs(es[1] - es[0]))
    assert jumps[0] < 1e-4 and jumps[1] < jumps[0] / 5 and jumps[2] < jumps[1] / 5


def test_compact_basis_roundtrip(rng):
    M = rng.standard_normal((5, 3, 3))
    c9 = T.from_full(M)
    assert np.allclose(T.to_full(c9), M, atol=1e-15)
    N = rng.standard_normal((5, 3, 3))
    assert np.allclose(T.frob(c9, T.from_full(N)), (M * N).sum((-1, -2)))
