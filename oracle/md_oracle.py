"""CPU restatement of the reference's Langevin "middle" integrator.  TEST INFRASTRUCTURE ONLY:
imported by tests/, __graft_entry__.smoke() and bench.py's CPU legs, never by the product path.

Follows /root/reference/pkg/src/nnpkit/md.py:
  * ``langevin_middle_update``  -- md.py:114-145 with the force evaluation factored out (the
    reference calls ``evaluate_auto`` at md.py:123; here the caller passes the forces so the same
    statement checks the integrator for any potential),
  * ``maxwell_boltzmann_velocities`` -- md.py:83-87,
  * ``throughput`` -- md.py:34-44, ``rmsd`` -- md.py:226-250.
Pinned bit for bit against trajectories produced by the reference itself
(tests/golden/make_md_golden.py -> tests/golden/md_golden.npz, tests/test_oracle_md.py).
"""

from __future__ import annotations

import numpy as np

# units.py:9-33 (CODATA-derived)
ELEMENTARY_CHARGE_C = 1.602176634e-19
ATOMIC_MASS_KG = 1.66053906660e-27
BOLTZMANN_EV = 8.617333262e-5
FORCE_TO_ACCELERATION = ELEMENTARY_CHARGE_C / ATOMIC_MASS_KG * 1e-10
VELOCITY_SQ_TO_EV = 1.0 / FORCE_TO_ACCELERATION
SECONDS_PER_DAY = 86400.0


def ou_coefficients(dt_fs: float, gamma_per_ps: float):
    """md.py:128-129."""
    c1 = np.exp(-gamma_per_ps * dt_fs / 1000.0)
    c2 = np.sqrt(1.0 - c1 * c1)
    return float(c1), float(c2)


def thermal_sigma(masses: np.ndarray, temperature: float) -> np.ndarray:
    """md.py:131-133 / md.py:86."""
    return np.sqrt(BOLTZMANN_EV * temperature * FORCE_TO_ACCELERATION / np.asarray(masses, dtype=np.float64))


def maxwell_boltzmann_velocities(masses, temperature, rng):
    """md.py:83-87."""
    masses = np.asarray(masses, dtype=np.float64)
    return rng.standard_normal((masses.size, 3)) * thermal_sigma(masses, temperature)[:, None]


def langevin_middle_update(positions, velocities, masses, forces, dt_fs, temperature, gamma_per_ps,
                           rng=None, noise=None):
    """One step given the forces at ``positions``; returns (new positions, new velocities, noise
    used or None).  Operation order as md.py:126-137."""
    positions = np.asarray(positions, dtype=np.float64)
    velocities = np.asarray(velocities, dtype=np.float64)
    masses = np.asarray(masses, dtype=np.float64)
    forces = np.asarray(forces, dtype=np.float64)
    accel = forces * (FORCE_TO_ACCELERATION / masses[:, None])
    v = velocities + dt_fs * accel
    x = positions + 0.5 * dt_fs * v
    c1, c2 = ou_coefficients(dt_fs, gamma_per_ps)
    used = None
    if c2 > 0.0:
        sigma = thermal_sigma(masses, temperature)
        used = rng.standard_normal((masses.size, 3)) if noise is None else np.asarray(noise, dtype=np.float64)
        v = c1 * v + c2 * sigma[:, None] * used
    x = x + 0.5 * dt_fs * v
    return x, v, used


def kinetic_energy(masses, velocities) -> float:
    """md.py:68-71."""
    return 0.5 * VELOCITY_SQ_TO_EV * float(np.sum(np.asarray(masses)[:, None] * np.asarray(velocities) ** 2))


def throughput(steps: int, wall_seconds: float, dt_fs: float):
    """md.py:34-44: (million steps per day, ns per day)."""
    msteps = steps * SECONDS_PER_DAY / (wall_seconds * 1e6)
    return msteps, msteps * dt_fs


def rmsd(reference, frame, align: bool = True) -> float:
    """md.py:226-250."""
    reference = np.asarray(reference, dtype=np.float64)
    frame = np.asarray(frame, dtype=np.float64)
    if align:
        ref = reference - reference.mean(axis=0)
        mov = frame - frame.mean(axis=0)
        u, _, vt = np.linalg.svd(mov.T @ ref)
        d = np.diag([1.0, 1.0, np.sign(np.linalg.det(u @ vt))])
        diff = mov @ (u @ d @ vt) - ref
    else:
        diff = frame - reference
    return float(np.sqrt(np.mean(np.sum(diff ** 2, axis=1))))
