"""Generate tests/golden/priors_golden.npz by running the REFERENCE's own prior terms
(/root/reference/pkg/src/nnpkit/priors.py) in this container.  Run once; the fixture is committed."""
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from nnpkit import NeighborSpec, build_neighbor_list, build_system  # noqa: E402
from nnpkit.priors import Atomref, Coulomb, D2Dispersion, PriorStack, ZBL, evaluate_prior_stack  # noqa: E402
from nnpkit.system import Box  # noqa: E402


def main():
    rng = np.random.default_rng(77)
    out = {}
    cases = [("open_half", 40, None, False, 6.0), ("open_full", 33, None, True, 5.0),
             ("cubic_half", 60, Box.cubic(13.0), False, 5.5), ("tric_full", 50, "tric", True, 4.5)]
    for name, n, box, full, cutoff in cases:
        if box == "tric":
            box = Box.triclinic(np.array([[12.0, 0, 0], [2.5, 11.0, 0], [-3.0, 1.5, 12.5]]))
        if box is None:
            pos = rng.uniform(0.0, 9.0, (n, 3))
        else:
            pos = rng.uniform(0.0, 1.0, (n, 3)) @ box.vectors
        # keep atoms apart a little so that the repulsion stays finite and well conditioned
        species = rng.choice([1, 6, 7, 8, 9, 16, 17], n)
        batch = np.sort(rng.integers(0, 3, n)) if box is None else None
        if batch is not None:
            batch = np.unique(batch, return_inverse=True)[1]
        charges = rng.normal(0.0, 0.4, n)
        system = build_system(pos, species, batch=batch, box=box, charges=charges)
        nl = build_neighbor_list(system, NeighborSpec(cutoff_upper=cutoff, capacity=n * n, full_list=full))
        table = {1: -13.6, 6: -1029.0, 7: -1485.0, 8: -2042.0, 9: -2713.0, 16: -10832.0, 17: -12516.0}
        stacks = {"atomref": (Atomref(table),), "coulomb": (Coulomb(2.5),), "zbl": (ZBL(),),
                  "d2": (D2Dispersion(s6=0.75, d_steep=18.0),),
                  "all": (Atomref(table), Coulomb(1.8), ZBL(), D2Dispersion())}
        pairs, deltas, dists = nl.valid()
        out.update({f"{name}_pos": pos, f"{name}_species": species, f"{name}_charges": charges,
                    f"{name}_batch": system.batch, f"{name}_pairs": pairs, f"{name}_deltas": deltas,
                    f"{name}_dists": dists, f"{name}_meta": np.array([float(full), cutoff]),
                    f"{name}_box": np.zeros((3, 3)) if box is None else box.vectors})
        for key, terms in stacks.items():
            res = evaluate_prior_stack(system, nl, PriorStack(terms))
            out[f"{name}_{key}_e"], out[f"{name}_{key}_f"], out[f"{name}_{key}_pa"] = res.energy, res.forces, res.per_atom_energy
    here = os.path.dirname(os.path.abspath(__file__))
    np.savez_compressed(os.path.join(here, "priors_golden.npz"), **out)
    print("wrote priors_golden.npz,", len(out), "arrays")


if __name__ == "__main__":
    main()
