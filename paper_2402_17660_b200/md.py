"""NVT Langevin dynamics (middle-thermostat splitting) around the device energy/forces step.

Mirrors the reference's ``nnpkit.md`` for the hot path: ``MDState``,
``initialize_state``, ``maxwell_boltzmann_velocities``, ``default_masses``,
``langevin_middle_step``, ``run_simulation``, ``Trajectory``, ``throughput``, ``rmsd``
(md.py:28-250).  The integrator itself is one CUDA kernel behind ``nnp_md_langevin_middle``;
state is float64 like the reference, forces are the float32 output of the TensorNet step.

Two ways to step:

* ``langevin_middle_step(state, model, ...)`` -- the reference's call shape: host state in, host
  state out, noise drawn from the state's NumPy Philox generator exactly as md.py:134 does, so
  a seed pins the trajectory the same way (positions agree with the reference integrator bit for
  bit given equal forces).
* ``run_simulation(state, model, steps, ...)`` -- the whole loop on the device: neighbor search,
  TensorNet step and integrator are one CUDA graph replayed per step, noise comes from a
  counter-based Philox4x32-10 generator on the device (seed + step + atom), frames are copied
  out every ``stride`` steps.  The random stream differs from NumPy's (documented departure);
  a seed still pins the trajectory.

There is no CPU fallback: without the CUDA extension and a device these raise ``ExtensionError``.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .errors import NumericError, ValidationError
from .system import System

# units.py:9-33 (CODATA-derived)
BOLTZMANN_EV = 8.617333262e-5
FORCE_TO_ACCELERATION = 1.602176634e-19 / 1.66053906660e-27 * 1e-10
VELOCITY_SQ_TO_EV = 1.0 / FORCE_TO_ACCELERATION
SECONDS_PER_DAY = 86400.0

# IUPAC abridged standard atomic weights, Z = 1..54 (index 0 unused), amu
_ATOMIC_WEIGHTS = (
    0.0, 1.008, 4.0026, 6.94, 9.0122, 10.81, 12.011, 14.007, 15.999, 18.998, 20.180,
    22.990, 24.305, 26.982, 28.085, 30.974, 32.06, 35.45, 39.948, 39.098, 40.078,
    44.956, 47.867, 50.942, 51.996, 54.938, 55.845, 58.933, 58.693, 63.546, 65.38,
    69.723, 72.630, 74.922, 78.971, 79.904, 83.798, 85.468, 87.62, 88.906, 91.224,
    92.906, 95.95, 98.0, 101.07, 102.91, 106.42, 107.87, 112.41, 114.82, 118.71,
    121.76, 127.60, 126.90, 131.29,
)


def atomic_mass(z: int) -> float:
    """Standard atomic weight of element ``z`` (elements.py:46-50)."""
    if not 1 <= int(z) < len(_ATOMIC_WEIGHTS):
        raise ValidationError(f"no atomic mass for Z = {z}")
    return _ATOMIC_WEIGHTS[int(z)]


def default_masses(species) -> np.ndarray:
    """md.py:79-80."""
    return np.array([atomic_mass(int(z)) for z in np.asarray(species)])


@dataclass(frozen=True)
class Throughput:
    msteps_per_day: float
    ns_per_day: float


def throughput(steps: int, wall_seconds: float, dt_fs: float) -> Throughput:
    """Million steps per day and the simulated ns/day (md.py:34-44): 10^6 steps per day at 1 fs
    is exactly 1 ns/day."""
    if wall_seconds <= 0:
        raise ValidationError("wall_seconds must be positive")
    msteps = steps * SECONDS_PER_DAY / (wall_seconds * 1e6)
    return Throughput(msteps_per_day=msteps, ns_per_day=msteps * dt_fs)


@dataclass
class MDState:
    """Positions (in ``system``), velocities (angstrom/fs), masses (amu) and the RNG (md.py:47-76)."""

    system: System
    velocities: np.ndarray
    masses: np.ndarray
    time_fs: float = 0.0
    rng: np.random.Generator = None
    seed: int = 0

    def __post_init__(self):
        n = self.system.n_atoms
        self.velocities = np.asarray(self.velocities, dtype=np.float64)
        self.masses = np.asarray(self.masses, dtype=np.float64)
        if self.velocities.shape != (n, 3):
            raise ValidationError(f"velocities must have shape ({n}, 3)")
        if self.masses.shape != (n,):
            raise ValidationError(f"masses must have shape ({n},)")
        if np.any(self.masses <= 0):
            raise ValidationError("masses must be positive")
        if self.rng is None:
            self.rng = np.random.Generator(np.random.Philox(self.seed))

    def kinetic_energy(self) -> float:
        return 0.5 * VELOCITY_SQ_TO_EV * float(np.sum(self.masses[:, None] * self.velocities ** 2))

    def kinetic_temperature(self) -> float:
        dof = 3 * self.system.n_atoms
        return 2.0 * self.kinetic_energy() / (dof * BOLTZMANN_EV)


def thermal_sigma(masses: np.ndarray, temperature: float) -> np.ndarray:
    return np.sqrt(BOLTZMANN_EV * temperature * FORCE_TO_ACCELERATION / np.asarray(masses, dtype=np.float64))


def maxwell_boltzmann_velocities(masses: np.ndarray, temperature: float,
                                 rng: np.random.Generator) -> np.ndarray:
    """md.py:83-87."""
    masses = np.asarray(masses, dtype=np.float64)
    return rng.standard_normal((masses.size, 3)) * thermal_sigma(masses, temperature)[:, None]


def initialize_state(system: System, temperature: float, seed: int = 0,
                     masses: Optional[np.ndarray] = None,
                     velocities: Optional[np.ndarray] = None) -> MDState:
    """Fresh state with element masses and thermal velocities by default (md.py:90-104)."""
    masses = default_masses(system.species) if masses is None else np.asarray(masses)
    rng = np.random.Generator(np.random.Philox(seed))
    if velocities is None:
        velocities = maxwell_boltzmann_velocities(masses, temperature, rng)
    return MDState(system=system, velocities=velocities, masses=masses, rng=rng, seed=seed)


def ou_coefficients(dt_fs: float, gamma_per_ps: float):
    """md.py:128-129."""
    c1 = float(np.exp(-gamma_per_ps * dt_fs / 1000.0))
    return c1, float(np.sqrt(1.0 - c1 * c1))


class DeviceIntegrator:
    """Device-resident MD state around one TensorNet plan: positions are the plan's float64
    position buffer, so the step graph reads what the integrator wrote."""

    def __init__(self, model, system: System, velocities: np.ndarray, masses: np.ndarray,
                 temperature: float, seed: int = 0, max_num_neighbors: Optional[int] = None):
        torch = _lib.require_cuda()
        self.torch, self.model, self.lib = torch, model, _lib.load()
        dev = model.device
        n = system.n_atoms
        self.n = n
        self.system = system
        if max_num_neighbors is not None and max_num_neighbors != model.config.max_num_neighbors:
            # the reference sizes the list from this argument (md.py:107-111 -> compose.py:59-71):
            # directed rows incl. self loops = 2 * N * max_num_neighbors; a larger learned size wins
            key = (n, system.n_samples)
            model._capacity_hint[key] = max(model._capacity_hint.get(key, 0), 2 * n * int(max_num_neighbors))
        # one checked float64 step creates (and captures) the plan whose pos64 buffer we own
        model.forward(system.species, system.positions, system.batch if system.n_samples > 1 else None,
                      system.box, n_samples=system.n_samples, check=True, clone=False)
        self.plan = model._last_plan
        f64 = dict(dtype=torch.float64, device=dev)
        self.vel = torch.as_tensor(np.ascontiguousarray(velocities, dtype=np.float64)).to(dev)
        self.acc_scale = torch.as_tensor(FORCE_TO_ACCELERATION / np.asarray(masses, dtype=np.float64)).to(dev)
        self.sigma = torch.as_tensor(thermal_sigma(masses, temperature)).to(dev)
        self.noise = torch.zeros((n, 3), **f64)
        self.counter = torch.zeros(1, dtype=torch.int64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.seed = int(seed)
        self.graph = None
        self._graph_key = None
        self._forces_current = True      # the checked step above left forces for these positions

    # ------------------------------------------------------------------ pieces
    def _enqueue_integrator(self, dt, c1, c2, device_noise: bool) -> None:
        p = self.plan
        rc = self.lib.nnp_md_langevin_middle(
            _lib.ptr(p.pos64), _lib.ptr(self.vel), _lib.ptr(p.forces), _lib.ptr(self.acc_scale),
            _lib.ptr(self.sigma), None if device_noise else _lib.ptr(self.noise),
            ctypes.c_uint64(self.seed), _lib.ptr(self.counter) if device_noise else None,
            dt, c1, c2, None, _lib.ptr(self.flag), self.n, _lib.ptr(p.engine.counts), p.capacity,
            _lib.current_stream())
        _lib.check(rc, "nnp_md_langevin_middle")

    def step_with_noise(self, dt_fs, gamma_per_ps, noise: Optional[np.ndarray]) -> None:
        """Forces at the current positions, then one integrator step with caller-supplied noise."""
        c1, c2 = ou_coefficients(dt_fs, gamma_per_ps)
        if c2 > 0.0:
            self.noise.copy_(self.torch.as_tensor(np.ascontiguousarray(noise, dtype=np.float64)))
        if not self._forces_current:
            self.model.replay(self.plan)
        self._enqueue_integrator(dt_fs, c1, c2, device_noise=False)
        self._forces_current = False

    def run_device(self, steps: int, dt_fs: float, gamma_per_ps: float) -> None:
        """``steps`` graph replays of [neighbor search + TensorNet step + integrator]."""
        torch = self.torch
        c1, c2 = ou_coefficients(dt_fs, gamma_per_ps)
        key = (dt_fs, c1, c2)
        if self.graph is None or self._graph_key != key:
            self.model._enqueue(self.plan)                       # warm-up outside capture
            torch.cuda.synchronize(self.model.device)
            saved = (self.plan.pos64.clone(), self.vel.clone(), self.counter.clone())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                self.model._enqueue(self.plan)
                self._enqueue_integrator(dt_fs, c1, c2, device_noise=True)
            self.graph, self._graph_key = graph, key
            self.plan.pos64.copy_(saved[0])
            self.vel.copy_(saved[1])
            self.counter.copy_(saved[2])
        for _ in range(steps):
            self.graph.replay()
        if steps > 0:
            self._forces_current = False

    # ------------------------------------------------------------------ host views
    def positions(self) -> np.ndarray:
        return self.plan.pos64.cpu().numpy()

    def velocities(self) -> np.ndarray:
        return self.vel.cpu().numpy()

    def potential_energy(self) -> float:
        """Energy at the CURRENT positions (one extra energy/forces step)."""
        if not self._forces_current:
            self.model.replay(self.plan)
            self._forces_current = True
        return float(self.plan.energy.sum().item())

    def check_finite(self, what: str) -> None:
        """NumericError on non-finite forces; CapacityError when a step found more neighbor rows than
        the plan holds.  In that case the integrator kernel froze the state at the last good step
        (positions, velocities and the noise counter untouched), so ``regrow`` + more steps resume it."""
        flag = int(self.flag.item())
        if flag == 1:
            raise NumericError(f"non-finite forces {what}")
        required = int(self.plan.engine.counts[0].item())
        if flag == 2 or required > self.plan.capacity:
            from .errors import CapacityError

            raise CapacityError(required=required, capacity=self.plan.capacity)

    def steps_done(self) -> int:
        """Integrator steps actually taken by ``run_device`` so far (frozen steps do not count)."""
        return int(self.counter.item())

    def regrow(self) -> None:
        """After a CapacityError: a plan with room for the rows the frozen step asked for (the model's
        own overflow loop, neighbors.py:238-247), the state carried over, graphs re-captured lazily."""
        torch = self.torch
        positions = self.plan.pos64.clone()
        s = self.system
        self.model.forward(s.species, positions, s.batch if s.n_samples > 1 else None, s.box,
                           n_samples=s.n_samples, check=True, clone=False)
        self.plan = self.model._last_plan
        self.plan.pos64.copy_(positions)
        self.flag.zero_()
        self.graph, self._graph_key = None, None
        self._forces_current = True
        torch.cuda.synchronize(self.model.device)


def network_of(potential):
    """The TensorNet a device MD loop integrates.  The reference integrates whatever
    ``evaluate_auto`` returns for the composed potential (md.py:107-111, 192-204); the device loop
    runs the network's captured step only, so a potential whose priors or ``derivative=False``
    would change the forces is refused instead of being integrated wrongly."""
    if not hasattr(potential, "network"):
        return potential
    if potential.network is None:
        raise ValidationError("device MD needs a TensorNet network; a prior-only potential has none")
    if len(potential.priors):
        raise ValidationError(
            "device MD integrates the network's forces only: a ComposedPotential with analytic "
            "priors is not supported (evaluate it with evaluate_auto instead)")
    if not potential.derivative:
        raise ValidationError("device MD needs forces: potential.derivative is False")
    return potential.network


def langevin_middle_step(state: MDState, potential, dt_fs: float, temperature: float,
                         gamma_per_ps: float, max_num_neighbors: int = 64) -> MDState:
    """Advance one step; returns a new state sharing the RNG stream (md.py:114-145).
    ``potential`` is a ``TensorNet`` (or a ``ComposedPotential`` wrapping one, without priors)."""
    model = network_of(potential)
    integ = DeviceIntegrator(model, state.system, state.velocities, state.masses, temperature, state.seed,
                             max_num_neighbors=max_num_neighbors)
    _, c2 = ou_coefficients(dt_fs, gamma_per_ps)
    noise = state.rng.standard_normal((state.masses.size, 3)) if c2 > 0.0 else None
    integ.step_with_noise(dt_fs, gamma_per_ps, noise)
    try:
        integ.check_finite(f"at t = {state.time_fs} fs")
    except NumericError:
        raise
    return MDState(system=state.system.replace_positions(integ.positions()), velocities=integ.velocities(),
                   masses=state.masses, time_fs=state.time_fs + dt_fs, rng=state.rng, seed=state.seed)


@dataclass
class Trajectory:
    """Captured frames plus the run metadata needed to reproduce them (md.py:148-163)."""

    stride: int
    dt_fs: float
    temperature_k: float
    gamma_per_ps: float
    seed: int
    species: np.ndarray
    frames: list = field(default_factory=list)
    energies: list = field(default_factory=list)

    @property
    def n_frames(self) -> int:
        return len(self.frames)


def run_simulation(state: MDState, potential, steps: int, dt_fs: float, temperature: float,
                   gamma_per_ps: float, stride: int = 1, max_num_neighbors: int = 64):
    """Repeated stepping on the device with periodic frame capture and a wall-time report
    (md.py:166-223).  Frame zero is the initial configuration; 1 + floor(steps/stride) frames."""
    if steps < 0 or stride < 1:
        raise ValidationError("steps must be >= 0 and stride >= 1")
    model = network_of(potential)
    torch = _lib.require_cuda()
    trajectory = Trajectory(stride=stride, dt_fs=dt_fs, temperature_k=temperature,
                            gamma_per_ps=gamma_per_ps, seed=state.seed, species=state.system.species)
    integ = DeviceIntegrator(model, state.system, state.velocities, state.masses, temperature, state.seed,
                             max_num_neighbors=max_num_neighbors)

    def capture():
        trajectory.frames.append(integ.positions())
        trajectory.energies.append(integ.potential_energy())

    capture()
    torch.cuda.synchronize(model.device)
    start = time.perf_counter()
    from .errors import CapacityError

    done = 0
    while done < steps:
        chunk = min(stride - done % stride, steps - done)
        integ.run_device(chunk, dt_fs, gamma_per_ps)
        try:
            integ.check_finite(f"(detected by step {done + chunk})")
        except CapacityError:
            # the list overflowed part-way through the chunk: the state is frozen at the last good
            # step; grow the plan like build_with_auto_capacity and take the remaining steps
            done = integ.steps_done()
            integ.regrow()
            continue
        done += chunk
        if done % stride == 0:
            capture()
    torch.cuda.synchronize(model.device)
    wall = time.perf_counter() - start
    rates = throughput(steps, wall, dt_fs) if steps > 0 and wall > 0 else None
    final = MDState(system=state.system.replace_positions(integ.positions()), velocities=integ.velocities(),
                    masses=state.masses, time_fs=state.time_fs + steps * dt_fs, rng=state.rng, seed=state.seed)
    report = {"steps": steps, "wall_seconds": wall,
              "msteps_per_day": rates.msteps_per_day if rates else float("nan"),
              "ns_per_day": rates.ns_per_day if rates else float("nan"), "final_state": final}
    return trajectory, report


def rmsd(reference: np.ndarray, frame: np.ndarray, align: bool = True) -> float:
    """Root mean square deviation, optionally after optimal superposition (md.py:226-250)."""
    reference = np.asarray(reference, dtype=np.float64)
    frame = np.asarray(frame, dtype=np.float64)
    if reference.shape != frame.shape or reference.ndim != 2 or reference.shape[1] != 3:
        raise ValidationError("frames must share one (N, 3) shape")
    if not align:
        return float(np.sqrt(np.mean(np.sum((frame - reference) ** 2, axis=1))))
    ref = reference - reference.mean(axis=0)
    mov = frame - frame.mean(axis=0)
    u, _, vt = np.linalg.svd(mov.T @ ref)
    flip = np.diag([1.0, 1.0, np.sign(np.linalg.det(u @ vt))])
    diff = mov @ (u @ flip @ vt) - ref
    return float(np.sqrt(np.mean(np.sum(diff ** 2, axis=1))))
