"""Generate tests/golden/md_golden.npz by running the REFERENCE's own integrator
(/root/reference/pkg/src/nnpkit/md.py) in this container.  Run once; the fixture is committed.

Each case steps a few atoms in a harmonic tether (the potential of the reference's own MD tests,
tests/test_md.py:29-46) and records, per step, the forces the reference saw and the state it
produced, so that the oracle (and the device kernel) can be checked step by step.
"""
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from nnpkit import ComposedPotential, PriorStack, build_system, initialize_state, langevin_middle_step  # noqa: E402
from nnpkit._ops import segment_sum  # noqa: E402
from nnpkit.md import MDState, default_masses  # noqa: E402
from nnpkit.priors import PriorTerm  # noqa: E402
from nnpkit.system import EnergyForces  # noqa: E402


class Tether(PriorTerm):
    needs_neighbors = False

    def __init__(self, stiffness, centers):
        self.stiffness, self.centers = stiffness, np.asarray(centers, dtype=np.float64)

    def evaluate(self, system, neighbors=None):
        disp = system.positions - self.centers
        per_atom = 0.5 * self.stiffness * np.sum(disp ** 2, axis=1)
        return EnergyForces(energy=segment_sum(per_atom, system.batch, system.n_samples),
                            forces=-self.stiffness * disp, per_atom_energy=per_atom)


def main():
    out = {}
    rng = np.random.default_rng(123)
    cases = [("nve", 7, 0.5, 50.0, 0.0, 11), ("nvt", 12, 1.0, 300.0, 5.0, 42), ("hot", 5, 2.0, 900.0, 50.0, 3)]
    for name, n, dt, temp, gamma, seed in cases:
        pos0 = rng.uniform(0.0, 6.0, (n, 3))
        species = rng.choice([1, 6, 8, 18], n)
        system = build_system(pos0, species)
        centers = pos0 + rng.normal(0.0, 0.2, (n, 3))
        stiffness = 3.5
        potential = ComposedPotential(priors=PriorStack((Tether(stiffness, centers),)))
        state = initialize_state(system, temp, seed=seed)
        xs, vs, fs = [np.array(state.system.positions)], [np.array(state.velocities)], []
        for _ in range(6):
            fs.append(-stiffness * (state.system.positions - centers))   # what the reference evaluates
            state = langevin_middle_step(state, potential, dt, temp, gamma)
            xs.append(np.array(state.system.positions))
            vs.append(np.array(state.velocities))
        out.update({f"{name}_x": np.array(xs), f"{name}_v": np.array(vs), f"{name}_f": np.array(fs),
                    f"{name}_masses": default_masses(species), f"{name}_species": species,
                    f"{name}_par": np.array([dt, temp, gamma, seed], dtype=np.float64)})
    here = os.path.dirname(os.path.abspath(__file__))
    np.savez_compressed(os.path.join(here, "md_golden.npz"), **out)
    print("wrote md_golden.npz with", sorted(out))


if __name__ == "__main__":
    main()
