"""CPU restatement of the reference's analytic prior terms.  TEST INFRASTRUCTURE ONLY: imported by
tests/ (and nothing in the product path).

Follows /root/reference/pkg/src/nnpkit/priors.py: the pair assembly ``_pair_term_energy_forces``
(:61-88), ``Atomref`` (:92-117), ``Coulomb`` (:121-151), ``ZBL`` (:155-187), ``D2Dispersion``
(:191-247) and the stack sum (:270-283), with the constants of units.py:9-33 and priors.py:24-44.
Pinned bit for bit against outputs of the reference itself (tests/golden/make_priors_golden.py ->
tests/golden/priors_golden.npz, tests/test_oracle_priors.py).
"""

from __future__ import annotations

import numpy as np

from .neighbors_oracle import cosine_cutoff, cosine_cutoff_grad

COULOMB_CONSTANT = 14.399645
BOHR_RADIUS = 0.529177
JNM6_PER_MOL_TO_EV_A6 = 1e6 / (6.02214076e23 * 1.602176634e-19)
D2_TABLE_JNM6 = {1: (0.14, 1.001), 6: (1.75, 1.452), 7: (1.23, 1.397), 8: (0.70, 1.342),
                 9: (0.75, 1.287), 16: (5.57, 1.683), 17: (5.07, 1.639)}
ZBL_COEFFS = np.array([0.18175, 0.50986, 0.28022, 0.02817])
ZBL_EXPONENTS = np.array([3.19980, 0.94229, 0.40290, 0.20162])
ZBL_SCREENING_PREFACTOR = 0.8854 * BOHR_RADIUS


def segment_sum(values, index, n):
    """_ops.py:6-19: row-order scatter add."""
    values = np.asarray(values, dtype=np.float64)
    if values.ndim == 1:
        return np.bincount(index, weights=values, minlength=n)
    return np.stack([np.bincount(index, weights=values[:, k], minlength=n) for k in range(values.shape[1])], 1)


def half_rows(pairs, deltas, dists, full_list: bool):
    """What as_half_list + the loop filter of priors.py:73-76 leave: rows with i < j."""
    keep = pairs[:, 0] < pairs[:, 1] if full_list else pairs[:, 0] != pairs[:, 1]
    return pairs[keep], deltas[keep], dists[keep]


def assemble(n_atoms, batch, n_samples, pairs, deltas, dists, energy_pair, de_dd):
    """priors.py:79-88."""
    if pairs.shape[0] == 0:
        return np.zeros(n_samples), np.zeros((n_atoms, 3)), np.zeros(n_atoms)
    i, j = pairs[:, 0], pairs[:, 1]
    per_atom = 0.5 * (segment_sum(energy_pair, i, n_atoms) + segment_sum(energy_pair, j, n_atoms))
    energy = segment_sum(per_atom, batch, n_samples)
    pair_force = -de_dd[:, None] * (deltas / dists[:, None])
    forces = segment_sum(pair_force, i, n_atoms) - segment_sum(pair_force, j, n_atoms)
    return energy, forces, per_atom


def coulomb_pair(pairs, d, charges, switch_radius):
    """priors.py:139-148."""
    qq = COULOMB_CONSTANT * charges[pairs[:, 0]] * charges[pairs[:, 1]]
    inside = d < switch_radius
    phase = np.pi * d / switch_radius
    switch = np.where(inside, 0.5 * (1.0 - np.cos(phase)), 1.0)
    dswitch = np.where(inside, 0.5 * np.pi / switch_radius * np.sin(phase), 0.0)
    return qq * switch / d, qq * (dswitch / d - switch / d ** 2)


def zbl_pair(pairs, d, species, cutoff):
    """priors.py:170-185."""
    z = np.asarray(species, dtype=np.float64)
    z_i, z_j = z[pairs[:, 0]], z[pairs[:, 1]]
    a = ZBL_SCREENING_PREFACTOR / (z_i ** 0.23 + z_j ** 0.23)
    x = d / a
    terms = ZBL_COEFFS * np.exp(-ZBL_EXPONENTS * x[:, None])
    screen = terms.sum(axis=1)
    dscreen = -(terms * ZBL_EXPONENTS).sum(axis=1) / a
    bare = COULOMB_CONSTANT * z_i * z_j / d
    env, denv = cosine_cutoff(d, 0.0, cutoff), cosine_cutoff_grad(d, 0.0, cutoff)
    energy = bare * screen * env
    de_dd = -bare / d * screen * env + bare * dscreen * env + bare * screen * denv
    return energy, de_dd


def d2_pair(pairs, d, species, cutoff, s6=1.0, d_steep=20.0):
    """priors.py:222-245 with the shipped element table (priors.py:27-38)."""
    c6_z = np.array([D2_TABLE_JNM6[int(z)][0] * JNM6_PER_MOL_TO_EV_A6 for z in species])
    r_z = np.array([D2_TABLE_JNM6[int(z)][1] for z in species])
    c6 = np.sqrt(c6_z[pairs[:, 0]] * c6_z[pairs[:, 1]])
    r_sum = r_z[pairs[:, 0]] + r_z[pairs[:, 1]]
    arg = d_steep * (d / r_sum - 1.0)
    damp = np.empty_like(d)
    pos = arg >= 0
    damp[pos] = 1.0 / (1.0 + np.exp(-arg[pos]))
    ex = np.exp(arg[~pos])
    damp[~pos] = ex / (1.0 + ex)
    ddamp = damp * (1.0 - damp) * d_steep / r_sum
    inv6 = d ** -6
    env, denv = cosine_cutoff(d, 0.0, cutoff), cosine_cutoff_grad(d, 0.0, cutoff)
    energy = -s6 * c6 * inv6 * damp * env
    de_dd = -s6 * c6 * (-6.0 * inv6 / d * damp * env + inv6 * ddamp * env + inv6 * damp * denv)
    return energy, de_dd


def evaluate_terms(terms, positions, species, batch, charges, pairs, deltas, dists, full_list, cutoff):
    """Sum of the listed terms (priors.py:270-283).  ``terms`` is a list of tuples:
    ("atomref", table), ("coulomb", switch_radius), ("zbl",), ("d2", s6, d_steep)."""
    n = len(species)
    batch = np.zeros(n, dtype=np.int64) if batch is None else np.asarray(batch)
    ns = int(batch[-1]) + 1
    energy, forces, per_atom = np.zeros(ns), np.zeros((n, 3)), np.zeros(n)
    hp, hd, hr = half_rows(pairs, deltas, dists, full_list)
    for term in terms:
        if term[0] == "atomref":
            pa = np.array([term[1][int(z)] for z in species], dtype=np.float64)
            e, f = segment_sum(pa, batch, ns), np.zeros((n, 3))
        else:
            if term[0] == "coulomb":
                ep, de = coulomb_pair(hp, hr, np.asarray(charges, dtype=np.float64), term[1])
            elif term[0] == "zbl":
                ep, de = zbl_pair(hp, hr, species, cutoff)
            else:
                ep, de = d2_pair(hp, hr, species, cutoff, term[1], term[2])
            e, f, pa = assemble(n, batch, ns, hp, hd, hr, ep, de)
        energy, forces, per_atom = energy + e, forces + f, per_atom + pa
    return energy, forces, per_atom
