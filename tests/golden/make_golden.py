"""Generate golden vectors by running the REFERENCE ITSELF (nnpkit, imported
read-only from /root/reference/pkg/src).  Run in the build container only:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

/root/reference does not exist on the GPU box; tests read only the committed
``neighbors_golden.npz`` written here.  Inputs are stored next to outputs so
the oracle and the CUDA path are run on identical bits.
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import nnpkit  # noqa: E402
from nnpkit import (  # noqa: E402
    Box, NeighborSpec, build_neighbor_list, build_system, canonicalize, distance_pullback,
)
from nnpkit.radial import (  # noqa: E402
    cosine_cutoff, cosine_cutoff_grad, expnorm_initial_params, rbf_expnorm, rbf_expnorm_with_grads,
)
from nnpkit._ops import segment_sum, silu, silu_grad  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def random_box(rng, kind, lo=5.0, hi=12.0):
    ax, by, cz = rng.uniform(lo, hi, 3)
    if kind == "orthorhombic":
        return Box.orthorhombic(ax, by, cz)
    return Box.triclinic(
        [
            [ax, 0.0, 0.0],
            [rng.uniform(-ax / 2, ax / 2), by, 0.0],
            [rng.uniform(-ax / 2, ax / 2), rng.uniform(-by / 2, by / 2), cz],
        ]
    )


def random_batch(rng, n, n_batches):
    n_batches = min(n_batches, n)
    cuts = np.sort(rng.choice(np.arange(1, n), size=n_batches - 1, replace=False))
    sizes = np.diff(np.concatenate([[0], cuts, [n]]))
    return np.repeat(np.arange(len(sizes), dtype=np.int64), sizes)


def main():
    rng = np.random.default_rng(20260117)
    arrays = {}
    manifest = {"nnpkit_version": nnpkit.__version__, "cases": []}
    case_id = 0
    kinds = ("none", "orthorhombic", "triclinic")
    for trial in range(48):
        kind = kinds[trial % 3]
        n = int(rng.integers(2, 97))
        big = trial >= 42          # a few larger boxes so the cell grid has > 3 cells per axis
        if kind == "none":
            box = None
            positions = rng.uniform(0.0, 14.0 if big else 9.0, (n if not big else 160, 3))
        else:
            box = random_box(rng, kind, lo=16.0, hi=22.0) if big else random_box(rng, kind)
            positions = rng.uniform(0.0, 1.0, (n if not big else 160, 3)) @ box.vectors
        n = positions.shape[0]
        # half the cases hold float32-representable positions (what the GPU model path sees)
        if trial % 2 == 0:
            positions = positions.astype(np.float32).astype(np.float64)
        if box is None:
            r_upper = float(rng.uniform(1.5, 4.0))
        else:
            r_upper = float(box.min_width() / 2 * rng.uniform(0.35, 0.99))
            if big:
                r_upper = float(rng.uniform(2.5, 4.5))
        r_lower = float(rng.choice([0.0, 0.3 * r_upper]))
        batch = random_batch(rng, n, int(rng.integers(1, 5)))
        system = build_system(positions, np.ones(n, dtype=np.int64), batch=batch, box=box)
        for strategy in ("brute", "cell"):
            full = bool((trial // 3) % 2)
            loops = bool((trial // 6) % 2)
            det = True
            spec = NeighborSpec(
                cutoff_upper=r_upper, cutoff_lower=r_lower, capacity=2 * n * n + n + 2,
                strategy=strategy, full_list=full, include_self_loops=loops, deterministic=det,
            )
            nl = build_neighbor_list(system, spec)
            cp, cd = canonicalize(nl)
            key = f"c{case_id}"
            arrays[f"{key}_pos"] = positions
            arrays[f"{key}_batch"] = batch
            if box is not None:
                arrays[f"{key}_box"] = np.asarray(box.vectors)
            c = nl.count
            arrays[f"{key}_pairs"] = nl.pairs[:c].astype(np.int32)
            arrays[f"{key}_deltas"] = nl.deltas[:c]
            arrays[f"{key}_dists"] = nl.distances[:c]
            arrays[f"{key}_canon_pairs"] = cp.astype(np.int32)
            arrays[f"{key}_canon_dists"] = cd
            g = np.random.default_rng(case_id).uniform(-1, 1, nl.capacity)
            arrays[f"{key}_pullback"] = distance_pullback(nl, g)
            manifest["cases"].append(
                dict(
                    key=key, kind=kind, n=n, strategy=strategy, full_list=full,
                    include_self_loops=loops, deterministic=det, cutoff_upper=r_upper,
                    cutoff_lower=r_lower, capacity=spec.capacity, count=int(c),
                    notes=list(nl.notes), pullback_seed=case_id,
                )
            )
            case_id += 1

    # box widths
    wb = []
    for k in range(8):
        b = random_box(rng, "triclinic")
        wb.append(np.concatenate([b.vectors.ravel(), b.perpendicular_widths()]))
    arrays["box_widths"] = np.array(wb)

    # radial functions and activations
    d = np.concatenate([np.linspace(0.0, 5.5, 221), rng.uniform(0, 5, 64)])
    arrays["radial_d"] = d
    for tag, (rl, ru, k) in {"a": (0.0, 5.0, 32), "b": (1.0, 4.0, 8), "c": (0.0, 4.5, 32)}.items():
        means, betas = expnorm_initial_params(k, rl, ru)
        f, dfdd, _, _ = rbf_expnorm_with_grads(d, means, betas, rl)
        arrays[f"radial_{tag}_cfg"] = np.array([rl, ru, k])
        arrays[f"radial_{tag}_means"] = means
        arrays[f"radial_{tag}_betas"] = betas
        arrays[f"radial_{tag}_rbf"] = rbf_expnorm(d, means, betas, rl)
        arrays[f"radial_{tag}_rbf_dd"] = dfdd
        arrays[f"radial_{tag}_cut"] = cosine_cutoff(d, rl, ru)
        arrays[f"radial_{tag}_cut_grad"] = cosine_cutoff_grad(d, rl, ru)
    x = np.concatenate([np.linspace(-30, 30, 121), rng.standard_normal(32)])
    arrays["act_x"] = x
    arrays["act_silu"] = silu(x)
    arrays["act_silu_grad"] = silu_grad(x)
    v = rng.standard_normal((50, 4))
    idx = rng.integers(0, 7, 50)
    arrays["seg_values"] = v
    arrays["seg_index"] = idx
    arrays["seg_out"] = segment_sum(v, idx, 7)

    np.savez_compressed(os.path.join(HERE, "neighbors_golden.npz"), **arrays)
    with open(os.path.join(HERE, "neighbors_golden.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print(f"wrote {case_id} neighbor cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
