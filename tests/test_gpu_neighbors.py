"""Parity of the CUDA neighbor search (through the C ABI) with the reference.

Golden vectors come from the reference itself (tests/golden/make_golden.py); the CPU oracle
(oracle/neighbors_oracle.py, pinned bit-exactly to those vectors) extends the comparison to
inputs generated here.  Integer and float64 outputs must be BIT-EXACT.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from conftest import random_batch, random_reduced_box  # noqa: E402
from oracle import neighbors_oracle as O  # noqa: E402

import paper_2402_17660_b200 as P  # noqa: E402
from paper_2402_17660_b200 import synth  # noqa: E402


def make_system(pos, batch, box):
    b = None if box is None else P.Box.from_matrix(box)
    return P.build_system(pos, np.ones(len(pos), dtype=np.int64), batch=batch, box=b)


def assert_same_list(nl, ref, key=""):
    host = nl.as_reference()
    assert nl.count == ref.count, key
    c = ref.count
    assert np.array_equal(host.pairs[:c], ref.pairs[:c]), key
    assert np.array_equal(host.deltas[:c], ref.deltas[:c]), key       # bit-exact float64
    assert np.array_equal(host.distances[:c], ref.distances[:c]), key
    assert np.all(host.pairs[c:] == -1) and np.all(host.distances[c:] == 0.0)
    assert np.all(host.deltas[c:] == 0.0)


def test_golden_vectors_bit_exact(golden):
    arrays, manifest = golden
    for case in manifest["cases"]:
        key = case["key"]
        box = arrays[f"{key}_box"] if f"{key}_box" in arrays.files else None
        system = make_system(arrays[f"{key}_pos"], arrays[f"{key}_batch"], box)
        spec = P.NeighborSpec(
            cutoff_upper=case["cutoff_upper"], cutoff_lower=case["cutoff_lower"],
            capacity=case["capacity"], strategy=case["strategy"], full_list=case["full_list"],
            include_self_loops=case["include_self_loops"])
        nl = P.build_neighbor_list(system, spec)
        host = nl.as_reference()
        c = case["count"]
        assert nl.count == c, key
        assert np.array_equal(host.pairs[:c], arrays[f"{key}_pairs"]), key
        assert np.array_equal(host.deltas[:c], arrays[f"{key}_deltas"]), key
        assert np.array_equal(host.distances[:c], arrays[f"{key}_dists"]), key
        assert list(nl.notes) == case["notes"], key
        cp, cd = P.canonicalize(nl)
        assert np.array_equal(cp, arrays[f"{key}_canon_pairs"])
        assert np.array_equal(cd, arrays[f"{key}_canon_dists"])
        g = np.random.default_rng(case["pullback_seed"]).uniform(-1, 1, nl.capacity)
        pb = P.distance_pullback(nl, g)
        assert np.max(np.abs(pb - arrays[f"{key}_pullback"])) < 1e-12, key


COLLINEAR = [[0.0, 0, 0], [1.0, 0, 0], [2.0, 0, 0]]


def collinear():
    return P.build_system(COLLINEAR, [1, 1, 1])


def test_known_answers():
    nl = P.build_neighbor_list(collinear(), P.NeighborSpec(cutoff_upper=1.5, capacity=8))
    pairs, d = P.canonicalize(nl)
    assert pairs.tolist() == [[0, 1], [1, 2]] and np.allclose(d, 1.0)
    with pytest.raises(P.CapacityError) as err:
        P.build_neighbor_list(collinear(), P.NeighborSpec(cutoff_upper=1.5, capacity=1))
    assert err.value.required == 2 and err.value.capacity == 1
    assert P.build_with_auto_capacity(collinear(), P.NeighborSpec(cutoff_upper=1.5, capacity=1)).count == 2
    s = P.build_system([[0.1, 0, 0], [9.9, 0, 0]], [1, 1], box=P.Box.cubic(10.0))
    pairs, d = P.canonicalize(P.build_neighbor_list(s, P.NeighborSpec(cutoff_upper=0.5, capacity=4)))
    assert pairs.tolist() == [[0, 1]] and d[0] == pytest.approx(0.2, abs=1e-12)
    s = P.build_system([[0.0, 0, 0], [0.1, 0, 0], [0.2, 0, 0], [0.3, 0, 0]], [1] * 4, batch=[0, 0, 1, 1])
    pairs, _ = P.canonicalize(P.build_neighbor_list(s, P.NeighborSpec(cutoff_upper=1.0, capacity=16)))
    assert pairs.tolist() == [[0, 1], [2, 3]]
    s = P.build_system([[0.0, 0, 0]], [1], box=P.Box.cubic(4.0))
    with pytest.raises(P.ValidationError, match="cutoff too large"):
        P.build_neighbor_list(s, P.NeighborSpec(cutoff_upper=2.5, capacity=4))
    nl = P.build_neighbor_list(collinear(), P.NeighborSpec(cutoff_upper=2.5, cutoff_lower=1.5, capacity=8))
    pairs, d = P.canonicalize(nl)
    assert pairs.tolist() == [[0, 2]] and d[0] == pytest.approx(2.0)


def test_flags_and_views():
    nl = P.build_neighbor_list(collinear(), P.NeighborSpec(cutoff_upper=1.5, capacity=10, include_self_loops=True))
    pairs = nl.as_reference().pairs[: nl.count]
    assert sorted(pairs[pairs[:, 0] == pairs[:, 1]][:, 0].tolist()) == [0, 1, 2]
    full = P.build_neighbor_list(collinear(), P.NeighborSpec(cutoff_upper=1.5, capacity=10, full_list=True))
    assert full.count == 4
    host = full.as_reference()
    look = {tuple(p): d for p, d in zip(host.pairs[:4].tolist(), host.deltas[:4])}
    for (i, j), d in look.items():
        assert np.array_equal(look[(j, i)], -d)
    half = P.build_neighbor_list(collinear(), P.NeighborSpec(cutoff_upper=1.5, capacity=10))
    up = P.as_full_list(half)
    assert up.count == 2 * half.count and up.capacity == 2 * half.capacity
    assert np.array_equal(up.pairs[: up.count], host.pairs[:4])
    back = P.as_half_list(up)
    assert np.array_equal(back.pairs[: back.count], half.as_reference().pairs[: half.count])
    s = P.build_system([[0.0, 0, 0], [1.0, 0, 0]], [1, 1], box=P.Box.cubic(10.0))
    nl = P.build_neighbor_list(s, P.NeighborSpec(cutoff_upper=4.9, capacity=8, strategy="cell"))
    assert any("fell back" in n for n in nl.notes) and nl.count == 1


def test_pullback_errors_and_direction():
    s = P.build_system([[1.0, 0, 0], [0.0, 0, 0]], [1, 1])
    nl = P.build_neighbor_list(s, P.NeighborSpec(cutoff_upper=2.0, capacity=5))
    g = P.distance_pullback(nl, np.ones(nl.capacity))
    assert np.allclose(g, [[1.0, 0, 0], [-1.0, 0, 0]])
    bad = P.NeighborList(pairs=np.array([[0, 1], [-1, -1]]), deltas=np.zeros((2, 3)),
                         distances=np.zeros(2), count=1, n_atoms=2,
                         spec=P.NeighborSpec(cutoff_upper=1.0, capacity=2))
    with pytest.raises(P.NumericError, match=r"zero-distance pair \(0, 1\)"):
        P.distance_pullback(bad, np.ones(2))


def test_random_sweep_matches_oracle_exactly():
    """The reference's acceptance sweep (test_acceptance.py:86-135) against the CUDA path."""
    rng = np.random.default_rng(20240501)
    kinds = ("none", "orthorhombic", "triclinic")
    for trial in range(240):
        n = int(rng.integers(2, 257))
        kind = kinds[trial % 3]
        if kind == "none":
            box = None
            pos = rng.uniform(0.0, 10.0, (n, 3))
            r_upper = float(rng.uniform(1.2, 3.0))
        else:
            _, box = random_reduced_box(rng, lo=5.0, hi=12.0, kind=kind)
            pos = rng.uniform(0.0, 1.0, (n, 3)) @ box
            r_upper = float(O.perpendicular_widths(box).min() / 2 * rng.uniform(0.35, 0.99))
        r_lower = float(rng.choice([0.0, 0.3 * r_upper]))
        full = bool(rng.integers(0, 2))
        loops = bool(rng.integers(0, 2))
        batch = random_batch(rng, n, int(rng.integers(1, 9)))
        system = make_system(pos, batch, box)
        ref_pairs, ref_d = O.exhaustive_pair_set(pos, batch, box, r_lower, r_upper)
        for strategy in ("brute", "cell"):
            cap = 2 * n * n + n + 2
            spec = P.NeighborSpec(cutoff_upper=r_upper, cutoff_lower=r_lower, capacity=cap,
                                  strategy=strategy, full_list=full, include_self_loops=loops)
            nl = P.build_neighbor_list(system, spec)
            ref = O.build_neighbor_list(pos, batch, box, r_upper, cap, cutoff_lower=r_lower,
                                        strategy=strategy, full_list=full, include_self_loops=loops)
            assert_same_list(nl, ref, (trial, strategy))
            cp, cd = P.canonicalize(nl)
            cp = cp[cp[:, 0] != cp[:, 1]]
            assert cp.tolist() == ref_pairs.tolist(), (trial, strategy)


@pytest.mark.parametrize("n,kind", [(20000, "cubic"), (12000, "triclinic"), (6000, "open")])
def test_medium_systems_cell_bit_exact(n, kind):
    rng = np.random.default_rng(n)
    if kind == "cubic":
        _, pos, batch, box = synth.config_b_cloud(n, seed=5)
    elif kind == "triclinic":
        _, pos, batch, box = synth.config_e_triclinic(n, seed=6)
    else:
        pos = rng.uniform(0, 40.0, (n, 3)).astype(np.float32).astype(np.float64)
        batch = random_batch(rng, n, 3)
        box = None
    cap = 40 * n
    for full in (False, True):
        ref = O.build_neighbor_list(pos, batch, box, 5.0, cap * 2, strategy="cell", full_list=full)
        nl = P.build_neighbor_list(make_system(pos, batch, box),
                                   P.NeighborSpec(cutoff_upper=5.0, capacity=cap * 2, strategy="cell", full_list=full))
        assert_same_list(nl, ref, (n, kind, full))


def test_many_small_samples_brute():
    _, pos, batch, _ = synth.config_d_molecules(300, seed=9)
    n = len(pos)
    ref = O.build_neighbor_list(pos, batch, None, 5.0, 64 * n, strategy="brute", full_list=True,
                                include_self_loops=True)
    nl = P.build_neighbor_list(make_system(pos, batch, None),
                               P.NeighborSpec(cutoff_upper=5.0, capacity=64 * n, strategy="brute",
                                              full_list=True, include_self_loops=True))
    assert_same_list(nl, ref)


def test_long_rows_use_scratch_path():
    """Rows longer than the shared-memory list (256) take the global-scratch ranking path."""
    rng = np.random.default_rng(3)
    n = 700
    pos = rng.uniform(0, 6.0, (n, 3))
    ref = O.build_neighbor_list(pos, None, None, 5.0, n * n, strategy="brute", full_list=True)
    for strategy in ("brute", "cell"):
        nl = P.build_neighbor_list(P.build_system(pos, np.ones(n, dtype=np.int64)),
                                   P.NeighborSpec(cutoff_upper=5.0, capacity=n * n, strategy=strategy,
                                                  full_list=True))
        assert_same_list(nl, ref, strategy)


def test_determinism_translation_padding():
    rng = np.random.default_rng(1234)
    _, box = random_reduced_box(rng, kind="orthorhombic")
    pos = rng.uniform(0, 1, (40, 3)) @ box
    cutoff = min(2.5, 0.9 * O.perpendicular_widths(box).min() / 2)
    system = make_system(pos, None, box)
    spec = P.NeighborSpec(cutoff_upper=cutoff, capacity=1600)
    a = P.build_neighbor_list(system, spec).as_reference()
    b = P.build_neighbor_list(system, spec).as_reference()
    assert np.array_equal(a.pairs, b.pairs) and np.array_equal(a.deltas, b.deltas)
    moved = P.canonicalize(P.build_neighbor_list(make_system(pos + [1.7, -2.3, 0.9], None, box), spec))
    base = P.canonicalize(P.build_neighbor_list(system, spec))
    assert base[0].tolist() == moved[0].tolist()
    assert np.max(np.abs(base[1] - moved[1]), initial=0.0) < 1e-10
    padded = P.canonicalize(P.build_neighbor_list(system, P.NeighborSpec(cutoff_upper=cutoff, capacity=6400)))
    assert base[0].tolist() == padded[0].tolist() and np.array_equal(base[1], padded[1])


def test_full_size_sweep_point_properties():
    """262 144 atoms (config B): count equals the oracle's; full = 2 x half; CSR is consistent."""
    n = 262144
    _, pos, batch, box = synth.config_b_cloud(n, seed=0)
    system = make_system(pos, batch, box)
    half = P.build_neighbor_list(system, P.NeighborSpec(cutoff_upper=5.0, capacity=32 * n, strategy="cell"))
    ref = O.build_neighbor_list(pos, batch, box, 5.0, 32 * n, strategy="cell")
    assert half.count == ref.count
    hp = half.pairs[: half.count].cpu().numpy()
    assert np.array_equal(hp, ref.pairs[: ref.count])
    assert np.array_equal(half.deltas[: half.count].cpu().numpy(), ref.deltas[: ref.count])      # bit-exact float64
    assert np.array_equal(half.distances[: half.count].cpu().numpy(), ref.distances[: ref.count])
    full = P.build_neighbor_list(system, P.NeighborSpec(cutoff_upper=5.0, capacity=64 * n, strategy="cell",
                                                        full_list=True))
    assert full.count == 2 * half.count
    rp = full.row_ptr.cpu().numpy()
    assert rp[0] == 0 and rp[-1] == full.count and np.all(np.diff(rp) >= 0)
    fp = full.pairs[: full.count].cpu().numpy()
    assert np.array_equal(fp[:, 0], np.repeat(np.arange(n), np.diff(rp)))


def test_second_order_pullback_against_reference_golden(golden):
    """distance_pullback_second (neighbors.py:358-380) on device lists against outputs of the
    reference's own function (tests/golden/pullback2_golden.npz): gradient to 1e-12 (float64 atomics
    change the summation order), distance tangents to 1e-14, sentinel tail zero; same errors."""
    import os

    arrays, manifest = golden
    p2 = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pullback2_golden.npz"))
    cases = {c["key"]: c for c in manifest["cases"]}
    for key in (str(k) for k in p2["keys"]):
        case = cases[key]
        box = arrays[f"{key}_box"] if f"{key}_box" in arrays.files else None
        system = make_system(arrays[f"{key}_pos"], arrays[f"{key}_batch"], box)
        nl = P.build_neighbor_list(system, P.NeighborSpec(
            cutoff_upper=case["cutoff_upper"], cutoff_lower=case["cutoff_lower"], capacity=case["capacity"],
            strategy=case["strategy"], full_list=case["full_list"], include_self_loops=case["include_self_loops"]))
        grad, dtan = P.distance_pullback_second(nl, p2[f"{key}_g"], p2[f"{key}_tangent"])
        ref = p2[f"{key}_grad"]
        assert grad.shape == ref.shape and dtan.shape == (case["capacity"],)
        assert np.max(np.abs(grad - ref), initial=0.0) <= 1e-12 * max(np.max(np.abs(ref), initial=0.0), 1.0), key
        assert np.max(np.abs(dtan[: nl.count] - p2[f"{key}_dtan"]), initial=0.0) < 1e-14, key
        assert not np.any(dtan[nl.count:]), key
    # the host copy of a list works as well, and the reference's validation errors are kept
    host = nl.as_reference()
    g2, t2 = P.distance_pullback_second(host, p2[f"{key}_g"], p2[f"{key}_tangent"])
    assert np.allclose(g2, grad, rtol=0, atol=1e-12) and np.array_equal(t2, dtan)
    with pytest.raises(P.ValidationError, match="position tangent"):
        P.distance_pullback_second(nl, p2[f"{key}_g"], np.zeros((3, 3)))
    with pytest.raises(P.ValidationError, match="d_grad"):
        P.distance_pullback_second(nl, np.zeros(nl.count + 1), p2[f"{key}_tangent"])
    pos = np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    coincident = P.build_neighbor_list(make_system(pos, None, None), P.NeighborSpec(cutoff_upper=2.0, capacity=8))
    if coincident.count == 3:       # the zero-distance pair is listed when the lower cutoff admits it
        with pytest.raises(P.NumericError, match="zero-distance"):
            P.distance_pullback_second(coincident, np.ones(8), np.ones((3, 3)))


def test_config_e_triclinic_box_full_list_bit_exact():
    """The 100 000-atom triclinic box of config E with the flags the model uses (full list, self
    loops): pairs, deltas and distances equal the C oracle's bit for bit."""
    z, pos, batch, box = synth.config_e_triclinic()
    n = len(pos)
    system = make_system(pos, batch, box)
    spec = P.NeighborSpec(cutoff_upper=5.0, capacity=64 * n, strategy="cell", full_list=True,
                          include_self_loops=True)
    nl = P.build_neighbor_list(system, spec)
    ref = O.build_neighbor_list(pos, batch, box, 5.0, 64 * n, strategy="cell", full_list=True,
                                include_self_loops=True)
    c = ref.count
    assert nl.count == c
    assert np.array_equal(nl.pairs[:c].cpu().numpy(), ref.pairs[:c])
    assert np.array_equal(nl.deltas[:c].cpu().numpy(), ref.deltas[:c])
    assert np.array_equal(nl.distances[:c].cpu().numpy(), ref.distances[:c])


def test_one_million_atoms_bit_exact():
    """1 048 576 atoms (the largest point of config B's sweep): pairs, deltas and distances of the
    half list equal the C oracle's bit for bit (the oracle needs a few seconds on one core)."""
    n = 1048576
    _, pos, batch, box = synth.config_b_cloud(n, seed=0)
    system = make_system(pos, batch, box)
    nl = P.build_neighbor_list(system, P.NeighborSpec(cutoff_upper=5.0, capacity=32 * n, strategy="cell"))
    ref = O.build_neighbor_list(pos, batch, box, 5.0, 32 * n, strategy="cell")
    c = ref.count
    assert nl.count == c
    assert np.array_equal(nl.pairs[:c].cpu().numpy(), ref.pairs[:c])
    assert np.array_equal(nl.deltas[:c].cpu().numpy(), ref.deltas[:c])
    assert np.array_equal(nl.distances[:c].cpu().numpy(), ref.distances[:c])
    tail = nl.pairs[c:]
    assert bool((tail == -1).all()) and bool((nl.distances[c:] == 0).all())


def test_nondeterministic_lists_hold_the_same_rows_grouped_by_receiver(rng):
    """deterministic=False (the reference's timing mode, neighbors.py:44,221) skips the in-row
    ranking: the same rows, bit for bit, grouped by i, in an unspecified order inside a group."""
    _, box = random_reduced_box(rng, 13.0, 17.0, kind="triclinic")
    pos = rng.uniform(0, 1, (400, 3)) @ box
    batch = random_batch(rng, 400, 3)
    for strategy in ("cell", "brute"):
        for full, loops in ((False, False), (True, True)):
            system = make_system(pos, batch, box)
            kw = dict(cutoff_upper=4.0, capacity=40000, strategy=strategy, full_list=full,
                      include_self_loops=loops)
            sorted_nl = P.build_neighbor_list(system, P.NeighborSpec(**kw)).as_reference()
            loose = P.build_neighbor_list(system, P.NeighborSpec(deterministic=False, **kw))
            host = loose.as_reference()
            c = sorted_nl.count
            assert loose.count == c
            assert np.all(np.diff(host.pairs[:c, 0]) >= 0)                     # still CSR by receiver
            order = np.lexsort((host.pairs[:c, 1], host.pairs[:c, 0]))
            assert np.array_equal(host.pairs[:c][order], sorted_nl.pairs[:c])
            assert np.array_equal(host.deltas[:c][order], sorted_nl.deltas[:c])
            assert np.array_equal(host.distances[:c][order], sorted_nl.distances[:c])
            assert np.all(host.pairs[c:] == -1)
