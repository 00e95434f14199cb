"""Golden vectors of ``distance_pullback_second`` from the REFERENCE ITSELF (nnpkit imported read-only
from /root/reference/pkg/src), on the neighbor lists of the committed golden cases.  Build container only:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_pullback2_golden.py

Writes tests/golden/pullback2_golden.npz: per case the seeded d_grad and position tangent, the
reference's gradient [n_atoms, 3] and distance tangents (the first ``count`` entries; the sentinel tail
is asserted to be zero here).
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from nnpkit import Box, NeighborSpec, build_neighbor_list, build_system  # noqa: E402
from nnpkit.neighbors import distance_pullback_second  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
arrays = np.load(os.path.join(HERE, "neighbors_golden.npz"))
manifest = json.load(open(os.path.join(HERE, "neighbors_golden.json")))
out = {}
keys = []
for n, case in enumerate(manifest["cases"]):
    if n % 3:            # a third of the 96 cases (all box kinds, strategies and list flavours occur)
        continue
    key = case["key"]
    box = None
    if f"{key}_box" in arrays.files:
        m = arrays[f"{key}_box"]
        diagonal = np.count_nonzero(m - np.diag(np.diag(m))) == 0
        box = Box.orthorhombic(*np.diag(m)) if diagonal else Box.triclinic(m)
    pos = arrays[f"{key}_pos"]
    system = build_system(pos, np.ones(len(pos), dtype=np.int64), batch=arrays[f"{key}_batch"], box=box)
    spec = NeighborSpec(cutoff_upper=case["cutoff_upper"], cutoff_lower=case["cutoff_lower"],
                        capacity=case["capacity"], strategy=case["strategy"], full_list=case["full_list"],
                        include_self_loops=case["include_self_loops"])
    nl = build_neighbor_list(system, spec)
    assert nl.count == case["count"]
    rng = np.random.default_rng(case["pullback_seed"] + 7)
    g = rng.uniform(-1, 1, nl.capacity)
    tangent = rng.standard_normal((len(pos), 3))
    grad, dtan = distance_pullback_second(nl, g, tangent)
    assert dtan.shape == (nl.capacity,) and not np.any(dtan[nl.count:])      # sentinel tail is zero
    c = nl.count
    out[f"{key}_g"], out[f"{key}_tangent"], out[f"{key}_grad"], out[f"{key}_dtan"] = g[:c], tangent, grad, dtan[:c]
    keys.append(key)
out["keys"] = np.array(keys)
np.savez_compressed(os.path.join(HERE, "pullback2_golden.npz"), **out)
print(len(keys), "cases written")
