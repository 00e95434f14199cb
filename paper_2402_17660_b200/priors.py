"""Analytic physical energy terms evaluated on the device.

Class names, constructor fields and validation messages follow the reference's
``nnpkit/priors.py`` (Atomref :92-117, Coulomb :121-151, ZBL :155-187, D2Dispersion :191-247,
PriorStack :250-267, evaluate_prior_stack :270-283).  What differs is where the work happens:
a stack is compiled into ONE launch of ``nnp_priors_pair_terms`` -- every enabled pair term is
evaluated in the same pass over the device neighbor list, in float64 -- and only the per-element
reference energies (a table lookup without geometry) stay on the host.
"""

from __future__ import annotations

import ctypes
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .errors import ValidationError
from .neighbors import NeighborList
from .system import EnergyForces, System

COULOMB_CONSTANT = 14.399645                 # eV A / e^2 (units.py:13)
BOHR_RADIUS = 0.529177                       # A (units.py:19)
JNM6_PER_MOL_TO_EV_A6 = 1e6 / (6.02214076e23 * 1.602176634e-19)
ZBL_SCREENING_PREFACTOR = 0.8854 * BOHR_RADIUS

# DFT-D2 parameters of the shipped elements: C6 in J nm^6 / mol, van der Waals radius in A
_D2_ELEMENTS = {1: (0.14, 1.001), 6: (1.75, 1.452), 7: (1.23, 1.397), 8: (0.70, 1.342),
                9: (0.75, 1.287), 16: (5.57, 1.683), 17: (5.07, 1.639)}
D2_C6_EV_A6 = {z: c6 * JNM6_PER_MOL_TO_EV_A6 for z, (c6, _) in _D2_ELEMENTS.items()}
D2_VDW_RADII = {z: radius for z, (_, radius) in _D2_ELEMENTS.items()}


class PriorTerm:
    """A physical energy term.  Pair terms describe themselves to the device kernel through
    ``_configure``; terms without geometry implement ``_host_energies``."""

    needs_neighbors = True

    def _configure(self, params: "_lib.PriorParams", system: System, inputs: dict) -> None:
        raise NotImplementedError

    def evaluate(self, system: System, neighbors: Optional[NeighborList] = None) -> EnergyForces:
        return evaluate_prior_stack(system, neighbors, PriorStack((self,)))


class Atomref(PriorTerm):
    """Per-element reference energies; no forces.  ``learnable`` is carried for the trainer."""

    needs_neighbors = False

    def __init__(self, table: Dict[int, float], learnable: bool = False):
        self.table, self.learnable = dict(table), bool(learnable)

    def _host_energies(self, system: System) -> np.ndarray:
        missing = sorted(set(int(z) for z in system.species) - set(self.table))
        if missing:
            raise ValidationError(f"missing reference for element {missing[0]}")
        lookup = np.zeros(int(system.species.max()) + 1)
        for z, value in self.table.items():
            if 0 <= int(z) < lookup.size:
                lookup[int(z)] = value
        return lookup[system.species]


class Coulomb(PriorTerm):
    """k q_i q_j S(d) / d with a cosine switch S that rises from 0 at d = 0 to 1 at the switch radius."""

    def __init__(self, switch_radius: float):
        if switch_radius <= 0:
            raise ValidationError("switch radius must be positive")
        self.switch_radius = float(switch_radius)

    def _configure(self, params, system, inputs):
        if system.charges is None:
            raise ValidationError("missing charges: the electrostatic prior needs per-atom "
                                  "partial charges on the system")
        params.flags |= _lib.PRIOR_COULOMB
        params.switch_radius = self.switch_radius
        inputs["charge"] = np.asarray(system.charges, dtype=np.float64)


class ZBL(PriorTerm):
    """Screened nuclear repulsion (universal four-exponential screening, length
    0.8854 a0 / (Z_i^0.23 + Z_j^0.23)) under the cosine envelope of the list's cutoff."""

    def _configure(self, params, system, inputs):
        if np.any(system.species <= 0):
            raise ValidationError("screened repulsion requires positive atomic numbers")
        params.flags |= _lib.PRIOR_ZBL
        z = system.species.astype(np.float64)
        inputs["znum"], inputs["zpow"] = z, z ** 0.23


class D2Dispersion(PriorTerm):
    """-s6 C6 / d^6 with sigmoid damping below the summed van der Waals radii, geometric-mean C6,
    cosine envelope at the cutoff.  The shipped table covers H, C, N, O, F, S, Cl."""

    def __init__(self, s6: float = 1.0, d_steep: float = 20.0, c6_table: Optional[dict] = None,
                 radii_table: Optional[dict] = None):
        if s6 <= 0:
            raise ValidationError("dispersion scale s6 must be positive")
        self.s6, self.d_steep = float(s6), float(d_steep)
        self.c6_table = dict(D2_C6_EV_A6 if c6_table is None else c6_table)
        self.radii_table = dict(D2_VDW_RADII if radii_table is None else radii_table)

    def _configure(self, params, system, inputs):
        known = set(self.c6_table) & set(self.radii_table)
        for z in np.unique(system.species):
            if int(z) not in known:
                raise ValidationError(f"element {int(z)} outside the dispersion parameter table")
        params.flags |= _lib.PRIOR_D2
        params.d2_s6, params.d2_steep = self.s6, self.d_steep
        inputs["c6"] = np.array([self.c6_table[int(z)] for z in system.species], dtype=np.float64)
        inputs["rvdw"] = np.array([self.radii_table[int(z)] for z in system.species], dtype=np.float64)


class PriorStack:
    """Ordered collection of prior terms evaluated as a sum."""

    def __init__(self, terms: Sequence[PriorTerm] = ()):
        self.terms: Tuple[PriorTerm, ...] = tuple(terms)

    def __len__(self) -> int:
        return len(self.terms)

    @property
    def needs_neighbors(self) -> bool:
        return any(t.needs_neighbors for t in self.terms)

    def learnable_atomref(self) -> Optional[Atomref]:
        return next((t for t in self.terms if isinstance(t, Atomref) and t.learnable), None)


def _device_list(neighbors: NeighborList, torch, device):
    """(pairs int32, deltas f64, distances f64) on the device, uploading a host list if needed."""
    if neighbors.on_device:
        return neighbors.pairs, neighbors.deltas.to(torch.float64), neighbors.distances.to(torch.float64)
    return (torch.as_tensor(np.ascontiguousarray(neighbors.pairs, dtype=np.int32)).to(device),
            torch.as_tensor(np.ascontiguousarray(neighbors.deltas, dtype=np.float64)).to(device),
            torch.as_tensor(np.ascontiguousarray(neighbors.distances, dtype=np.float64)).to(device))


def _new_params() -> "_lib.PriorParams":
    params = _lib.PriorParams()
    params.coulomb_constant, params.zbl_prefactor = COULOMB_CONSTANT, ZBL_SCREENING_PREFACTOR
    params.d2_s6, params.d2_steep, params.switch_radius = 1.0, 20.0, 1.0
    return params


def _run_pair_pass(params, inputs: dict, system: System, neighbors: NeighborList):
    """One launch of the fused pair kernel; returns (per-atom energies, forces) as numpy float64."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    n = system.n_atoms
    device = neighbors.pairs.device if neighbors.on_device else torch.device("cuda")
    pairs, deltas, dists = _device_list(neighbors, torch, device)
    params.cutoff_upper = float(neighbors.spec.cutoff_upper)
    dev = {k: torch.as_tensor(np.array(v, dtype=np.float64)).to(device) for k, v in inputs.items()}
    out_e = torch.empty(n, dtype=torch.float64, device=device)
    out_f = torch.empty((n, 3), dtype=torch.float64, device=device)
    rc = lib.nnp_priors_pair_terms(
        ctypes.byref(params), _lib.ptr(pairs), _lib.ptr(deltas), _lib.ptr(dists), None, int(neighbors.count),
        int(bool(neighbors.spec.full_list)), _lib.ptr(dev.get("charge")), _lib.ptr(dev.get("znum")),
        _lib.ptr(dev.get("zpow")), _lib.ptr(dev.get("c6")), _lib.ptr(dev.get("rvdw")), n,
        _lib.ptr(out_e), _lib.ptr(out_f), _lib.current_stream())
    _lib.check(rc, "nnp_priors_pair_terms")
    return out_e.cpu().numpy(), out_f.cpu().numpy()


def evaluate_prior_stack(system: System, neighbors: Optional[NeighborList], stack: PriorStack) -> EnergyForces:
    """Element-wise sum of all term outputs; an empty stack gives zeros (priors.py:270-283).
    Pair terms are fused: one device pass over ``neighbors`` evaluates one term of each kind, so a
    usual stack (Coulomb + ZBL + D2) is a single launch."""
    n, ns = system.n_atoms, system.n_samples
    per_atom = np.zeros(n)
    forces = np.zeros((n, 3))
    batches, used = [], 0
    for term in stack.terms:
        if not term.needs_neighbors:
            per_atom = per_atom + term._host_energies(system)
            continue
        probe = _new_params()
        term._configure(probe, system, {})
        if not batches or (used & probe.flags):
            batches.append((_new_params(), {}))
            used = 0
        term._configure(*batches[-1][:1], system, batches[-1][1])
        used |= probe.flags
    if batches and neighbors is None:
        raise ValidationError("this potential needs a neighbor list")
    for params, inputs in batches:
        e, f = _run_pair_pass(params, inputs, system, neighbors)
        per_atom, forces = per_atom + e, forces + f
    energy = np.bincount(system.batch, weights=per_atom, minlength=ns)
    return EnergyForces(energy=energy, forces=forces, per_atom_energy=per_atom)
