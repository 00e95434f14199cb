"""The CPU oracle against the reference's own outputs (golden vectors) and known answers.

Runs without a GPU.  Golden vectors were produced by tests/golden/make_golden.py running
nnpkit itself; known-answer cases restate reference tests/test_neighbors.py:42-108.
"""

import numpy as np
import pytest

from oracle import neighbors_oracle as O


def _case_inputs(arrays, case):
    key = case["key"]
    box = arrays[f"{key}_box"] if f"{key}_box" in arrays.files else None
    return arrays[f"{key}_pos"], arrays[f"{key}_batch"], box


def test_golden_lists_bit_exact(golden):
    arrays, manifest = golden
    assert len(manifest["cases"]) >= 90
    for case in manifest["cases"]:
        pos, batch, box = _case_inputs(arrays, case)
        nl = O.build_neighbor_list(
            pos, batch, box, case["cutoff_upper"], case["capacity"],
            cutoff_lower=case["cutoff_lower"], strategy=case["strategy"],
            include_self_loops=case["include_self_loops"], full_list=case["full_list"],
            deterministic=case["deterministic"],
        )
        key = case["key"]
        assert nl.count == case["count"], key
        assert np.array_equal(nl.pairs[: nl.count], arrays[f"{key}_pairs"]), key
        # bit-exact float64: same operation order, no FMA contraction
        assert np.array_equal(nl.deltas[: nl.count], arrays[f"{key}_deltas"]), key
        assert np.array_equal(nl.distances[: nl.count], arrays[f"{key}_dists"]), key
        assert np.all(nl.pairs[nl.count:] == -1)
        assert list(nl.notes) == case["notes"]
        cp, cd = O.canonicalize(nl.pairs, nl.distances, nl.count)
        assert np.array_equal(cp, arrays[f"{key}_canon_pairs"])
        assert np.array_equal(cd, arrays[f"{key}_canon_dists"])
        g = np.random.default_rng(case["pullback_seed"]).uniform(-1, 1, nl.capacity)
        pb = O.distance_pullback(nl.pairs, nl.deltas, nl.distances, nl.count, nl.n_atoms, g)
        assert np.array_equal(pb, arrays[f"{key}_pullback"]), key


def test_golden_matches_exhaustive_oracle(golden):
    arrays, manifest = golden
    for case in manifest["cases"][::5]:
        pos, batch, box = _case_inputs(arrays, case)
        ref_pairs, ref_d = O.exhaustive_pair_set(
            pos, batch, box, case["cutoff_lower"], case["cutoff_upper"]
        )
        key = case["key"]
        canon = arrays[f"{key}_canon_pairs"]
        canon = canon[canon[:, 0] != canon[:, 1]]
        assert canon.tolist() == ref_pairs.tolist()


def test_box_widths_golden(golden):
    arrays, _ = golden
    for row in arrays["box_widths"]:
        assert np.array_equal(O.perpendicular_widths(row[:9].reshape(3, 3)), row[9:])


def test_radial_golden(golden):
    arrays, _ = golden
    d = arrays["radial_d"]
    for tag in "abc":
        rl, ru, k = arrays[f"radial_{tag}_cfg"]
        means, betas = O.expnorm_initial_params(int(k), rl, ru)
        assert np.array_equal(means, arrays[f"radial_{tag}_means"])
        assert np.array_equal(betas, arrays[f"radial_{tag}_betas"])
        assert np.array_equal(O.rbf_expnorm(d, means, betas, rl), arrays[f"radial_{tag}_rbf"])
        assert np.array_equal(O.rbf_expnorm_dd(d, means, betas, rl), arrays[f"radial_{tag}_rbf_dd"])
        assert np.array_equal(O.cosine_cutoff(d, rl, ru), arrays[f"radial_{tag}_cut"])
        assert np.array_equal(O.cosine_cutoff_grad(d, rl, ru), arrays[f"radial_{tag}_cut_grad"])


def test_activation_and_segment_golden(golden):
    arrays, _ = golden
    assert np.array_equal(O.silu(arrays["act_x"]), arrays["act_silu"])
    assert np.array_equal(O.silu_grad(arrays["act_x"]), arrays["act_silu_grad"])
    assert np.array_equal(O.segment_sum(arrays["seg_values"], arrays["seg_index"], 7), arrays["seg_out"])


# ---- known answers restated from the reference's tests/test_neighbors.py ----

COLLINEAR = np.array([[0.0, 0, 0], [1.0, 0, 0], [2.0, 0, 0]])


def test_collinear_pairs():
    nl = O.build_neighbor_list(COLLINEAR, None, None, 1.5, 8)
    p, d = O.canonicalize(nl.pairs, nl.distances, nl.count)
    assert p.tolist() == [[0, 1], [1, 2]]
    assert np.allclose(d, 1.0)


def test_overflow_reports_required():
    with pytest.raises(O.OracleCapacityError) as err:
        O.build_neighbor_list(COLLINEAR, None, None, 1.5, 1)
    assert err.value.required == 2 and err.value.capacity == 1
    assert O.build_with_auto_capacity(COLLINEAR, None, None, 1.5, 1).count == 2


def test_minimum_image_pair():
    pos = np.array([[0.1, 0, 0], [9.9, 0, 0]])
    nl = O.build_neighbor_list(pos, None, np.eye(3) * 10.0, 0.5, 4)
    p, d = O.canonicalize(nl.pairs, nl.distances, nl.count)
    assert p.tolist() == [[0, 1]]
    assert d[0] == pytest.approx(0.2, abs=1e-12)


def test_batch_masking():
    pos = np.array([[0.0, 0, 0], [0.1, 0, 0], [0.2, 0, 0], [0.3, 0, 0]])
    nl = O.build_neighbor_list(pos, np.array([0, 0, 1, 1]), None, 1.0, 16)
    p, _ = O.canonicalize(nl.pairs, nl.distances, nl.count)
    assert p.tolist() == [[0, 1], [2, 3]]


def test_cutoff_too_large_for_box():
    with pytest.raises(O.OracleValidationError, match="cutoff too large"):
        O.build_neighbor_list(np.zeros((1, 3)), None, np.eye(3) * 4.0, 2.5, 4)


def test_sentinels_and_lower_cutoff():
    nl = O.build_neighbor_list(COLLINEAR, None, None, 1.5, 10)
    assert np.all(nl.pairs[nl.count:] == -1) and np.all(nl.distances[nl.count:] == 0.0)
    nl = O.build_neighbor_list(COLLINEAR, None, None, 2.5, 8, cutoff_lower=1.5)
    p, d = O.canonicalize(nl.pairs, nl.distances, nl.count)
    assert p.tolist() == [[0, 2]] and d[0] == pytest.approx(2.0)


def test_flags():
    nl = O.build_neighbor_list(COLLINEAR, None, None, 1.5, 10, include_self_loops=True)
    p = nl.pairs[: nl.count]
    assert sorted(p[p[:, 0] == p[:, 1]][:, 0].tolist()) == [0, 1, 2]
    nl = O.build_neighbor_list(COLLINEAR, None, None, 1.5, 10, full_list=True)
    assert nl.count == 4
    half = O.build_neighbor_list(COLLINEAR, None, None, 1.5, 10)
    full = O.as_full_list(half)
    assert full.count == 2 * half.count and full.capacity == 2 * half.capacity
    back = O.as_half_list(full)
    assert np.array_equal(back.pairs[: back.count], half.pairs[: half.count])


def test_cell_fallback_note():
    pos = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    nl = O.build_neighbor_list(pos, None, np.eye(3) * 10.0, 4.9, 8, strategy="cell")
    assert any("fell back" in n for n in nl.notes) and nl.count == 1


def test_pullback_single_pair_and_zero_distance():
    pos = np.array([[1.0, 0, 0], [0.0, 0, 0]])
    nl = O.build_neighbor_list(pos, None, None, 2.0, 5)
    g = O.distance_pullback(nl.pairs, nl.deltas, nl.distances, nl.count, 2, np.ones(5))
    assert np.allclose(g, [[1.0, 0, 0], [-1.0, 0, 0]])
    with pytest.raises(O.OracleNumericError, match=r"zero-distance pair \(0, 1\)"):
        O.distance_pullback(np.array([[0, 1]]), np.zeros((1, 3)), np.zeros(1), 1, 2, np.ones(1))


def test_second_order_pullback_oracle_matches_reference_golden():
    """oracle.distance_pullback_second against outputs of the reference's own function
    (tests/golden/make_pullback2_golden.py) on 32 of the golden lists: bit-exact."""
    import json
    import os

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    arrays = np.load(os.path.join(here, "neighbors_golden.npz"))
    p2 = np.load(os.path.join(here, "pullback2_golden.npz"))
    manifest = json.load(open(os.path.join(here, "neighbors_golden.json")))
    cases = {c["key"]: c for c in manifest["cases"]}
    assert len(p2["keys"]) == 32
    for key in p2["keys"]:
        key = str(key)
        case = cases[key]
        pairs, deltas, dists = arrays[f"{key}_pairs"], arrays[f"{key}_deltas"], arrays[f"{key}_dists"]
        n = len(arrays[f"{key}_pos"])
        grad, dtan = O.distance_pullback_second(pairs, deltas, dists, case["count"], n, case["capacity"],
                                                p2[f"{key}_g"], p2[f"{key}_tangent"])
        assert np.array_equal(grad, p2[f"{key}_grad"]), key
        assert np.array_equal(dtan[: case["count"]], p2[f"{key}_dtan"]), key
        assert dtan.shape == (case["capacity"],) and not np.any(dtan[case["count"]:])
