"""Analytic priors on the device (nnp_priors_pair_terms) against the reference's own outputs
(tests/golden/priors_golden.npz) and the CPU oracle: float64, agreement to rounding (the kernel's
atomic summation order and the device libm are the only differences), every term alone, the fused
stack, half and full lists, open / cubic / triclinic boxes, and composition with the network."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_17660_b200 as P  # noqa: E402
from oracle import priors_oracle as O  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "priors_golden.npz")
TABLE = {1: -13.6, 6: -1029.0, 7: -1485.0, 8: -2042.0, 9: -2713.0, 16: -10832.0, 17: -12516.0}
CASES = ["open_half", "open_full", "cubic_half", "tric_full"]


def stacks():
    return {"atomref": P.PriorStack((P.Atomref(TABLE),)), "coulomb": P.PriorStack((P.Coulomb(2.5),)),
            "zbl": P.PriorStack((P.ZBL(),)), "d2": P.PriorStack((P.D2Dispersion(s6=0.75, d_steep=18.0),)),
            "all": P.PriorStack((P.Atomref(TABLE), P.Coulomb(1.8), P.ZBL(), P.D2Dispersion()))}


def load_case(g, case):
    boxm = g[f"{case}_box"]
    box = P.Box.from_matrix(boxm) if boxm.any() else None
    system = P.build_system(g[f"{case}_pos"], g[f"{case}_species"], batch=g[f"{case}_batch"], box=box,
                            charges=g[f"{case}_charges"])
    full, cutoff = bool(g[f"{case}_meta"][0]), float(g[f"{case}_meta"][1])
    return system, full, cutoff


def close(a, b, tol=2e-12):
    scale = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(np.asarray(a) - b))) <= tol * scale


@pytest.mark.parametrize("case", CASES)
def test_device_priors_match_reference_outputs(case):
    g = np.load(GOLDEN)
    system, full, cutoff = load_case(g, case)
    n = system.n_atoms
    spec = P.NeighborSpec(cutoff_upper=cutoff, capacity=n * n, full_list=full)
    device_list = P.build_neighbor_list(system, spec)
    # the reference's own list, uploaded (host arrays), and the list built on the device
    host_list = P.NeighborList(pairs=g[f"{case}_pairs"], deltas=g[f"{case}_deltas"], distances=g[f"{case}_dists"],
                               count=len(g[f"{case}_dists"]), n_atoms=n, spec=spec)
    for key, stack in stacks().items():
        for nl in (host_list, device_list):
            res = P.evaluate_prior_stack(system, nl, stack)
            assert close(res.energy, g[f"{case}_{key}_e"]), (case, key)
            assert close(res.per_atom_energy, g[f"{case}_{key}_pa"]), (case, key)
            assert close(res.forces, g[f"{case}_{key}_f"], 2e-11) or not g[f"{case}_{key}_f"].any(), (case, key)


def test_repeated_kinds_validation_and_empty():
    g = np.load(GOLDEN)
    system, full, cutoff = load_case(g, "open_half")
    nl = P.build_neighbor_list(system, P.NeighborSpec(cutoff_upper=cutoff, capacity=system.n_atoms ** 2))
    two = P.evaluate_prior_stack(system, nl, P.PriorStack((P.Coulomb(2.5), P.Coulomb(1.0))))
    a = P.evaluate_prior_stack(system, nl, P.PriorStack((P.Coulomb(2.5),)))
    b = P.evaluate_prior_stack(system, nl, P.PriorStack((P.Coulomb(1.0),)))
    assert close(two.energy, a.energy + b.energy) and close(two.forces, a.forces + b.forces, 1e-11)
    zero = P.evaluate_prior_stack(system, None, P.PriorStack())
    assert not zero.energy.any() and not zero.forces.any()
    with pytest.raises(P.ValidationError):
        P.evaluate_prior_stack(system, None, P.PriorStack((P.ZBL(),)))
    with pytest.raises(P.ValidationError):
        P.Coulomb(0.0)
    with pytest.raises(P.ValidationError):
        P.D2Dispersion(s6=0.0)
    no_charge = P.build_system(system.positions, system.species)
    with pytest.raises(P.ValidationError):
        P.evaluate_prior_stack(no_charge, nl, P.PriorStack((P.Coulomb(2.0),)))
    heavy = P.build_system(system.positions, np.full(system.n_atoms, 26))
    with pytest.raises(P.ValidationError):
        P.evaluate_prior_stack(heavy, nl, P.PriorStack((P.D2Dispersion(),)))
    with pytest.raises(P.ValidationError):
        P.evaluate_prior_stack(system, nl, P.PriorStack((P.Atomref({1: 0.0}),)))


def test_composed_network_plus_priors_and_prior_only():
    rng = np.random.default_rng(4)
    pos = rng.uniform(0, 7, (30, 3))
    z = rng.choice([1, 6, 8], 30)
    system = P.build_system(pos, z, charges=rng.normal(0, 0.3, 30))
    model = P.TensorNet(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_upper=4.5, max_z=20, seed=2)
    stack = P.PriorStack((P.ZBL(), P.D2Dispersion(), P.Coulomb(1.5)))
    both = P.evaluate_auto(P.ComposedPotential(network=model, priors=stack), system)
    net = P.evaluate_auto(P.ComposedPotential(network=model), system)
    # the priors on the half of the network's directed list == the oracle on that list
    nl = P.build_neighbor_list(system, P.ComposedPotential(network=model).neighbor_spec(30)).as_reference()
    pr, dl, ds = nl.valid()
    e_ref, f_ref, pa_ref = O.evaluate_terms([("zbl",), ("d2", 1.0, 20.0), ("coulomb", 1.5)], pos, z, None,
                                            system.charges, pr, dl, ds, True, 4.5)
    assert close(both.energy - net.energy, e_ref, 1e-9)
    assert close(both.forces - net.forces, f_ref, 1e-9)
    assert close(both.per_atom_energy - net.per_atom_energy, pa_ref, 1e-9)
    only = P.ComposedPotential(priors=stack, cutoff=4.5)
    alone = P.evaluate_auto(only, system)
    assert close(alone.energy, e_ref) and close(alone.forces, f_ref, 2e-11)
    assert P.evaluate_auto(P.ComposedPotential(priors=stack, cutoff=4.5, derivative=False), system).forces is None
    with pytest.raises(P.ValidationError):
        P.ComposedPotential(priors=stack).resolve_cutoff()
    with pytest.raises(P.ValidationError):
        P.ComposedPotential()
