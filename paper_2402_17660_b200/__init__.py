"""B200-native drop-in for the accelerator hot path of ``nnpkit`` (arXiv 2402.17660):
cutoff neighbor search + TensorNet energy-and-forces step, as hand-written sm_100a CUDA behind
the C ABI of ``include/nnp_b200.h``.  Names follow ``nnpkit/__init__.py`` for this path."""

from .errors import (
    CapacityError, DataError, ExtensionError, NumericError, ParseError, ToolkitError, ValidationError,
)
from .system import Box, EnergyForces, System, build_system, minimum_image
from .radial import cosine_cutoff, cosine_cutoff_grad, expnorm_initial_params, rbf_expnorm
from .neighbors import (
    NeighborList, NeighborSpec, as_full_list, as_half_list, build_neighbor_list,
    build_with_auto_capacity, canonicalize, capacity_heuristic, distance_pullback,
    distance_pullback_second,
)
from .tensornet import TNConfig, TensorNet, build_radial_tables, init_params
from .priors import Atomref, Coulomb, D2Dispersion, PriorStack, PriorTerm, ZBL, evaluate_prior_stack
from .compose import ComposedPotential, evaluate, evaluate_auto
from .md import (
    MDState, Trajectory, default_masses, initialize_state, langevin_middle_step,
    maxwell_boltzmann_velocities, rmsd, run_simulation, throughput,
)

from .structio import Frame, load_extxyz, load_structure, load_weights, save_weights, write_extxyz

__version__ = "0.1.0"
