"""Device Langevin integrator (nnp_md_langevin_middle) and the MD driver: bit-exact against the
CPU oracle for equal forces and noise, the reference's golden trajectories, and the size-independent
properties the reference tests (tests/test_md.py of the reference): deterministic at zero friction,
seeded reruns identical, thermal variance of the thermostat, energy conservation."""

import ctypes
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2402_17660_b200 as P  # noqa: E402
from paper_2402_17660_b200 import _lib, md as M, synth  # noqa: E402
from oracle import md_oracle as O  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "md_golden.npz")


def device_update(x, v, masses, forces32, dt, temp, gamma, noise=None, seed=0, counter=None):
    lib = _lib.load()
    n = len(masses)
    xd, vd = torch.as_tensor(x).cuda().clone(), torch.as_tensor(v).cuda().clone()
    fd = torch.as_tensor(forces32).cuda()
    acc = torch.as_tensor(M.FORCE_TO_ACCELERATION / masses).cuda()
    sg = torch.as_tensor(M.thermal_sigma(masses, temp)).cuda()
    nd = None if noise is None else torch.as_tensor(noise).cuda()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    c1, c2 = M.ou_coefficients(dt, gamma)
    rc = lib.nnp_md_langevin_middle(xd.data_ptr(), vd.data_ptr(), fd.data_ptr(), acc.data_ptr(), sg.data_ptr(),
                                    _lib.ptr(nd), ctypes.c_uint64(seed), _lib.ptr(counter), dt, c1, c2, None,
                                    flag.data_ptr(), n, None, 0, torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    return xd.cpu().numpy(), vd.cpu().numpy(), int(flag.item())


@pytest.mark.parametrize("case", ["nve", "nvt", "hot"])
def test_kernel_reproduces_reference_golden_steps(case):
    """Forces rounded to float32 (what the device step delivers), noise from the reference's own
    Philox stream: device state == oracle state bit for bit, step after step."""
    g = np.load(GOLDEN)
    dt, temp, gamma, seed = g[f"{case}_par"]
    masses = g[f"{case}_masses"]
    rng = np.random.Generator(np.random.Philox(int(seed)))
    v = O.maxwell_boltzmann_velocities(masses, temp, rng)
    x = g[f"{case}_x"][0]
    xd, vd = x.copy(), v.copy()
    for k in range(len(g[f"{case}_f"])):
        f32 = g[f"{case}_f"][k].astype(np.float32)
        x, v, noise = O.langevin_middle_update(x, v, masses, f32.astype(np.float64), dt, temp, gamma, rng=rng)
        xd, vd, flag = device_update(xd, vd, masses, f32, dt, temp, gamma, noise=noise)
        assert flag == 0
        assert np.array_equal(xd, x) and np.array_equal(vd, v), (case, k)
        # and the float64-force reference trajectory is reproduced to float32 force rounding
        assert np.allclose(xd, g[f"{case}_x"][k + 1], rtol=0, atol=1e-6)


def test_random_large_update_bit_exact_and_flag():
    rng = np.random.default_rng(5)
    n = 20000
    masses = rng.choice([1.008, 12.011, 15.999], n)
    x, v = rng.uniform(0, 60, (n, 3)), rng.normal(0, 0.01, (n, 3))
    f = rng.normal(0, 1.0, (n, 3)).astype(np.float32)
    noise = rng.standard_normal((n, 3))
    xo, vo, _ = O.langevin_middle_update(x, v, masses, f.astype(np.float64), 0.5, 310.0, 2.0, noise=noise)
    xd, vd, flag = device_update(x, v, masses, f, 0.5, 310.0, 2.0, noise=noise)
    assert flag == 0 and np.array_equal(xd, xo) and np.array_equal(vd, vo)
    f[17, 1] = np.nan
    assert device_update(x, v, masses, f, 0.5, 310.0, 2.0, noise=noise)[2] == 1


def test_device_philox_noise_is_standard_normal_and_counter_based():
    """With zero forces and c1 = 0 (huge friction) the new velocity is sigma * xi: the device
    generator's samples are recovered exactly."""
    n = 200000
    masses = np.full(n, 39.948)
    x, v = np.zeros((n, 3)), np.zeros((n, 3))
    f = np.zeros((n, 3), dtype=np.float32)
    sigma = M.thermal_sigma(masses, 300.0)[0]
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    draws = []
    for _ in range(3):
        _, vd, _ = device_update(x, v, masses, f, 1.0, 300.0, 1e9, seed=1234, counter=counter)
        draws.append(vd / sigma)
    assert int(counter.item()) == 3
    xi = np.concatenate(draws).ravel()
    assert abs(xi.mean()) < 5e-3 and abs(xi.var() - 1.0) < 5e-3
    assert abs(np.mean(xi ** 3)) < 2e-2 and abs(np.mean(xi ** 4) - 3.0) < 5e-2
    assert np.abs(xi).max() > 4.0                            # tails are populated
    assert not np.array_equal(draws[0], draws[1])            # the counter advances the stream
    # same seed and counter -> same numbers; another seed -> other numbers
    c2 = torch.zeros(1, dtype=torch.int64, device="cuda")
    again = device_update(x, v, masses, f, 1.0, 300.0, 1e9, seed=1234, counter=c2)[1] / sigma
    other = device_update(x, v, masses, f, 1.0, 300.0, 1e9, seed=99, counter=torch.zeros_like(c2))[1] / sigma
    assert np.array_equal(again, draws[0]) and not np.array_equal(other, draws[0])
    # components of one atom and neighbouring atoms are uncorrelated
    a = draws[0]
    assert abs(np.corrcoef(a[:, 0], a[:, 1])[0, 1]) < 0.01 and abs(np.corrcoef(a[:-1, 0], a[1:, 0])[0, 1]) < 0.01


def small_model():
    return P.TensorNet(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_upper=4.0, max_z=20, seed=3)


def test_drop_in_step_matches_oracle_with_device_forces():
    """langevin_middle_step(state, model, ...) == oracle update fed the model's own forces."""
    rng = np.random.default_rng(1)
    pos = rng.uniform(0, 5, (14, 3))
    z = rng.choice([1, 6, 8], 14)
    system = P.build_system(pos, z)
    model = small_model()
    state = P.initialize_state(system, 250.0, seed=21)
    ref_rng = np.random.Generator(np.random.Philox(21))
    v = O.maxwell_boltzmann_velocities(state.masses, 250.0, ref_rng)
    assert np.array_equal(v, state.velocities)
    x = pos
    for _ in range(3):
        _, forces = model(torch.as_tensor(z), torch.as_tensor(x))          # float64 positions
        f32 = forces.cpu().numpy()
        x, v, _ = O.langevin_middle_update(x, v, state.masses, f32.astype(np.float64), 0.7, 250.0, 3.0, rng=ref_rng)
        state = P.langevin_middle_step(state, model, 0.7, 250.0, 3.0)
        assert np.array_equal(state.system.positions, x) and np.array_equal(state.velocities, v)
    assert state.time_fs == pytest.approx(2.1)


def test_composed_potentials_the_device_loop_cannot_integrate_are_refused():
    """The reference integrates evaluate_auto of the whole composed potential (md.py:107-111); the
    device loop runs the network's step only, so priors / derivative=False / no network raise."""
    rng = np.random.default_rng(3)
    system = P.build_system(rng.uniform(0, 5, (10, 3)), rng.choice([1, 6, 8], 10))
    model = small_model()
    state = P.initialize_state(system, 250.0, seed=1)
    ok = P.langevin_middle_step(state, P.ComposedPotential(network=model), 0.5, 250.0, 1.0)
    assert ok.time_fs == pytest.approx(0.5)
    with pytest.raises(P.ValidationError, match="priors"):
        P.langevin_middle_step(state, P.ComposedPotential(network=model, priors=P.PriorStack((P.ZBL(),))),
                               0.5, 250.0, 1.0)
    with pytest.raises(P.ValidationError, match="prior-only"):
        P.run_simulation(state, P.ComposedPotential(priors=P.PriorStack((P.ZBL(),)), cutoff=4.0), 2, 0.5, 250.0, 1.0)
    with pytest.raises(P.ValidationError, match="derivative"):
        P.run_simulation(state, P.ComposedPotential(network=model, derivative=False), 2, 0.5, 250.0, 1.0)


def test_neighbor_overflow_mid_run_freezes_regrows_and_resumes():
    """Atoms that start beyond the cutoff of each other and fly together: the list outgrows a plan
    sized for one neighbour per atom part-way through a chunk.  The integrator kernel must freeze the
    state at the last good step (no update from stale forces, noise counter not advanced), the driver
    regrows the plan and resumes: the trajectory equals, bit for bit, the one of a roomy model."""
    g = np.arange(3) * 4.6
    pos = np.stack(np.meshgrid(g[:2], g[:2], g, indexing="ij"), -1).reshape(-1, 3).astype(np.float64)
    z = np.full(len(pos), 6)
    centre = pos.mean(0)
    vel = -0.06 * (pos - centre) / np.linalg.norm(pos - centre, axis=1, keepdims=True)
    kw = dict(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_upper=4.0, max_z=20, seed=3)
    tight, roomy = P.TensorNet(max_num_neighbors=1, **kw), P.TensorNet(**kw)
    out = {}
    for name, model in (("tight", tight), ("roomy", roomy)):
        system = P.build_system(pos, z)
        state = P.initialize_state(system, 300.0, seed=5, velocities=vel.copy())
        traj, report = P.run_simulation(state, model, 24, 1.0, 300.0, 2.0, stride=8)
        out[name] = (traj, report["final_state"])
    first_capacity = 2 * len(pos) * 1
    assert tight._last_plan.capacity > first_capacity          # it did overflow and regrow
    a, b = out["tight"], out["roomy"]
    assert a[0].n_frames == b[0].n_frames == 4
    for fa, fb in zip(a[0].frames, b[0].frames):
        assert np.array_equal(fa, fb)
    assert np.array_equal(a[1].velocities, b[1].velocities)
    assert a[0].energies == b[0].energies


def test_run_simulation_frames_determinism_and_energy_conservation():
    rng = np.random.default_rng(2)
    pos = rng.uniform(0, 6, (24, 3))
    pos = pos[np.argsort(pos[:, 0])]
    z = rng.choice([1, 6, 8], 24)
    system = P.build_system(pos, z)
    model = P.TensorNet(embedding_dimension=32, num_layers=2, num_rbf=16, cutoff_upper=4.5, max_z=20, seed=8)
    state = P.initialize_state(system, 50.0, seed=42)
    traj, report = P.run_simulation(state, model, 103, 0.25, 50.0, 0.0, stride=10)
    assert traj.n_frames == 1 + 103 // 10 and report["steps"] == 103          # reference test_md.py:149-156
    assert np.array_equal(traj.frames[0], pos)
    assert report["msteps_per_day"] > 0 and report["final_state"].time_fs == pytest.approx(103 * 0.25)
    # zero friction: the kick-drift scheme (md.py:1-8) is symplectic Euler, so kinetic and potential
    # energy exchange with a bounded O(dt) mismatch (measured: 1.3 % of the exchanged energy at
    # 0.5 fs, halving with dt)
    final = report["final_state"]
    d_kin = final.kinetic_energy() - state.kinetic_energy()
    model_e = float(model(torch.as_tensor(z), torch.as_tensor(final.system.positions.copy()))[0][0])
    d_pot = model_e - traj.energies[0]
    assert abs(d_kin) > 0.05, d_kin                       # the run does exchange energy
    assert abs(d_kin + d_pot) < 0.015 * abs(d_kin), (d_kin, d_pot)
    # seeded rerun is identical (reference test_md.py:158-168), another seed differs (NVT)
    runs = []
    for seed in (7, 7, 8):
        st = P.initialize_state(system, 300.0, seed=seed)
        t, _ = P.run_simulation(st, model, 40, 0.5, 300.0, 5.0, stride=5)
        runs.append(np.array(t.frames))
    assert np.array_equal(runs[0], runs[1]) and not np.array_equal(runs[0], runs[2])
    zero, _ = P.run_simulation(state, model, 0, 1.0, 300.0, 1.0)
    assert zero.n_frames == 1
    with pytest.raises(P.ValidationError):
        P.run_simulation(state, model, -1, 1.0, 300.0, 1.0)


def test_thermostat_equipartition_free_particles():
    """Atoms out of each other's range feel no force; the OU thermostat must hold every velocity
    component at k_B T / m (reference test_md.py:120-131 uses one tethered oscillator)."""
    n = 4096
    g = np.arange(16) * 12.0
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3).astype(np.float64)
    z = np.full(n, 18)
    system = P.build_system(pos, z)
    model = small_model()
    state = P.initialize_state(system, 298.5, seed=5)
    _, report = P.run_simulation(state, model, 60, 1.0, 298.5, 200.0, stride=60)
    var = report["final_state"].velocities.var(axis=0).mean()
    expected = M.BOLTZMANN_EV * 298.5 * M.FORCE_TO_ACCELERATION / 39.948
    assert var == pytest.approx(expected, rel=0.05)
