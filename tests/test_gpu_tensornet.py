"""Parity of the CUDA TensorNet step (through the C ABI) with the float64 CPU oracle.

Tolerances are the north star's: per-sample energy |E_gpu - E_ref| / max(|E_ref|, 1) <= 1e-5,
forces max|F_gpu - F_ref| / max|F_ref| <= 1e-4 (FP32 on the device, float64 oracle).
The oracle itself is parity-unpinned (no reference TensorNet exists; see its header).
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import torch  # noqa: E402

from oracle import neighbors_oracle as O  # noqa: E402
from oracle import tensornet_oracle as T  # noqa: E402

import paper_2402_17660_b200 as P  # noqa: E402
from paper_2402_17660_b200 import _lib, synth  # noqa: E402

E_TOL = 1e-5
F_TOL = 1e-4


def oracle_eval(model, z, pos, batch, box, forces=True):
    cfg = model.config
    ocfg = T.OracleConfig(cfg.embedding_dimension, cfg.num_layers, cfg.num_rbf, cfg.cutoff_lower,
                          cfg.cutoff_upper, cfg.max_z, cfg.mean, cfg.std)
    n = len(pos)
    nl = O.build_with_auto_capacity(pos, batch, box, cfg.cutoff_upper, 64 * n,
                                    cutoff_lower=cfg.cutoff_lower,
                                    strategy="cell" if n > 3000 else "brute",
                                    full_list=True, include_self_loops=True)
    pr, dl, ds = nl.valid()
    return T.energy_forces_compact(model.params, ocfg, z, batch, pr, dl, ds, want_forces=forces)


def check(model, z, pos, batch, box, e_tol=E_TOL, f_tol=F_TOL):
    e, f = model(torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32),
                 None if batch is None else torch.as_tensor(batch), box)
    b = np.zeros(len(pos), dtype=np.int64) if batch is None else batch
    e_ref, f_ref, _ = oracle_eval(model, z, pos, b, box)
    e_err = np.max(np.abs(e.cpu().numpy() - e_ref) / np.maximum(np.abs(e_ref), 1.0))
    f_err = np.max(np.abs(f.cpu().numpy() - f_ref)) / np.max(np.abs(f_ref))
    assert e_err <= e_tol, f"energy rel err {e_err:.3e}"
    assert f_err <= f_tol, f"force rel err {f_err:.3e}"
    return e_err, f_err


@pytest.mark.parametrize("mode", [5, 3, 1, 0])
def test_gemm_tile_engine(mode):
    """All inner loops (streaming tcgen05 with W in tensor memory, per-tile tcgen05, mma.sync, FFMA)
    against float64."""
    lib = _lib.load()
    lib.nnp_set_gemm_mode(mode)
    try:
        g = torch.Generator(device="cuda").manual_seed(0)
        for M, N, K in [(64, 64, 32), (200, 128, 128), (333, 384, 256), (70, 16, 64), (129, 96, 16),
                        (1000, 256, 128), (5000, 128, 64), (128, 32, 384), (40000, 128, 128)]:
            A = torch.randn(M, K, device="cuda", generator=g)
            W = torch.randn(N, K, device="cuda", generator=g)
            bias = torch.randn(N, device="cuda", generator=g)
            out = torch.empty(M, N, device="cuda")
            gw = _lib.GemmWeight(W.data_ptr())
            rc = lib.nnp_test_gemm_nt(A.data_ptr(), ctypes.byref(gw), bias.data_ptr(), out.data_ptr(),
                                      M, N, K, torch.cuda.current_stream().cuda_stream)
            assert rc == 0
            ref = (A.double() @ W.double().T + bias.double())
            err = (out.double() - ref).abs().max().item() / ref.abs().max().item()
            assert err < 5e-6, (mode, M, N, K, err)   # FP32-level accuracy from the 3xTF32 split
    finally:
        lib.nnp_set_gemm_mode(_lib.DEFAULT_GEMM_MODE)


def small_open(rng, n=20):
    pos = rng.uniform(0, 5.0, (n, 3)).astype(np.float32).astype(np.float64)
    z = rng.choice([1, 6, 7, 8], n)
    batch = np.repeat([0, 1], [n - n // 2, n // 2])
    return z, pos, batch, None


@pytest.mark.parametrize("C", [32, 64, 128])
@pytest.mark.parametrize("L", [0, 1, 2])
def test_small_open_system(rng, C, L):
    model = P.TensorNet(embedding_dimension=C, num_layers=L, num_rbf=16, cutoff_upper=4.0,
                        max_z=10, mean=0.3, std=1.7, seed=3)
    assert model.table_error < 1e-6
    check(model, *small_open(rng))


@pytest.mark.parametrize("gemm_mode", [5, 3, 1, 0])
def test_periodic_triclinic_and_lower_cutoff(rng, gemm_mode):
    _lib.load().nnp_set_gemm_mode(gemm_mode)
    try:
        box = np.array([[11.0, 0, 0], [2.5, 10.5, 0], [-3.0, 1.5, 12.0]])
        pos = (rng.uniform(0, 1, (90, 3)) @ box).astype(np.float32).astype(np.float64)
        z = rng.choice([1, 6, 8], 90)
        model = P.TensorNet(embedding_dimension=32, num_layers=2, num_rbf=8, cutoff_upper=4.5,
                            max_z=10, seed=5)
        check(model, z, pos, None, box)
        model = P.TensorNet(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_lower=0.7,
                            cutoff_upper=4.5, max_z=10, seed=6)
        check(model, z, pos, None, box)
    finally:
        _lib.load().nnp_set_gemm_mode(_lib.DEFAULT_GEMM_MODE)


def test_config_a_alanine_sized_molecule():
    z, pos, batch, box = synth.config_a_molecule()
    model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0)
    check(model, z, pos, None, None)


def test_cell_path_with_renumbering_medium_periodic():
    """3 000 atoms at water density: cell strategy, cell-sorted internal numbering."""
    z, pos, batch, box = synth.config_c_box(n=3000, edge=31.0, seed=7)
    model = P.TensorNet(embedding_dimension=32, num_layers=2, num_rbf=16, cutoff_upper=5.0,
                        max_z=10, seed=1, strategy="cell")
    check(model, z, pos, None, box)
    brute = P.TensorNet(embedding_dimension=32, num_layers=2, num_rbf=16, cutoff_upper=5.0,
                        max_z=10, seed=1, strategy="brute")
    e1, f1 = model(torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), None, box)
    e2, f2 = brute(torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), None, box)
    assert abs(float(e1[0] - e2[0])) / max(abs(float(e2[0])), 1.0) < 1e-5
    assert float((f1 - f2).abs().max() / f2.abs().max()) < 1e-4


def test_batched_molecules():
    z, pos, batch, _ = synth.config_d_molecules(64, seed=4)
    model = P.TensorNet(embedding_dimension=64, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=2)
    check(model, z, pos, batch, None)
    # batch independence: a slice of samples gives the same numbers
    sel = batch < 8
    e_all, f_all = model(torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), torch.as_tensor(batch))
    e_sub, f_sub = model(torch.as_tensor(z[sel]), torch.as_tensor(pos[sel], dtype=torch.float32),
                         torch.as_tensor(batch[sel]))
    assert torch.allclose(e_all[:8], e_sub, rtol=1e-6, atol=1e-6)
    assert torch.allclose(f_all[: int(sel.sum())], f_sub, rtol=1e-5, atol=1e-7)


def test_lattice_ties_long_rows_and_isolated_atom():
    """Rows far longer than a warp, many exactly equal distances (the in-row ordering by table
    coordinate must break ties consistently), an atom whose only edge is its self loop, and the
    capacity growth that a 200-neighbour row forces."""
    g = np.arange(5) * 1.3
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    pos = np.concatenate([pos, [[40.0, 40.0, 40.0]]]).astype(np.float32).astype(np.float64)
    z = np.resize([1, 6, 8], len(pos))
    for C, L in ((32, 2), (128, 1)):
        model = P.TensorNet(embedding_dimension=C, num_layers=L, num_rbf=16, cutoff_upper=5.0,
                            max_z=10, seed=9)
        check(model, z, pos, None, None)


def test_three_layer_triclinic_config_e_shape():
    """Config E's shape at a size the oracle finishes quickly: triclinic box, 3 layers."""
    L = 24.0
    box = np.array([[L, 0, 0], [0.3 * L, L, 0], [0.2 * L, -0.25 * L, L]])
    rng = np.random.default_rng(5)
    pos = (rng.uniform(0, 1, (700, 3)) @ box).astype(np.float32).astype(np.float64)
    z = rng.choice([1, 8], 700, p=[2 / 3, 1 / 3])
    model = P.TensorNet(embedding_dimension=64, num_layers=3, num_rbf=32, cutoff_upper=5.0,
                        max_z=10, seed=4, strategy="cell")
    check(model, z, pos, None, box)


def test_graph_replay_equals_eager_and_is_deterministic(rng):
    z, pos, batch, _ = small_open(rng, 30)
    args = (torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), torch.as_tensor(batch))
    a = P.TensorNet(embedding_dimension=32, num_layers=2, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=1)
    b = P.TensorNet(embedding_dimension=32, num_layers=2, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=1,
                    use_graph=False)
    e1, f1 = a(*args)
    e2, f2 = a(*args)          # second call replays the captured graph
    e3, f3 = b(*args)
    assert torch.equal(e1, e2) and torch.equal(f1, f2)
    assert torch.equal(e1, e3) and torch.equal(f1, f3)


def test_overflow_grows_capacity(rng):
    z, pos, batch, _ = small_open(rng, 40)
    tight = P.TensorNet(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_upper=4.0, max_z=10,
                        seed=1, max_num_neighbors=1)
    roomy = P.TensorNet(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=1)
    args = (torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), torch.as_tensor(batch))
    e1, f1 = tight(*args)
    e2, f2 = roomy(*args)
    assert torch.equal(e1, e2) and torch.equal(f1, f2)


def test_evaluate_call_shapes_and_validation(rng):
    z, pos, batch, _ = small_open(rng, 24)
    model = P.TensorNet(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=1)
    system = P.build_system(pos, z, batch=batch)
    pot = P.ComposedPotential(network=model)
    res = P.evaluate_auto(pot, system)
    e, f = model(torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), torch.as_tensor(batch))
    assert np.allclose(res.energy, e.cpu().numpy(), rtol=1e-6, atol=1e-6)
    assert np.allclose(res.forces, f.cpu().numpy(), rtol=1e-5, atol=1e-7)
    assert np.allclose(np.bincount(batch, weights=res.per_atom_energy), res.energy, rtol=1e-5)
    half = P.build_neighbor_list(system, P.NeighborSpec(cutoff_upper=4.0, capacity=2000))
    with pytest.raises(P.ValidationError, match="full neighbor list"):
        model.evaluate(system, half)
    other = P.build_neighbor_list(system, P.NeighborSpec(cutoff_upper=3.0, capacity=2000, full_list=True,
                                                         include_self_loops=True))
    with pytest.raises(P.ValidationError, match="cutoff mismatch"):
        model.evaluate(system, other)
    with pytest.raises(P.ValidationError, match="out of range"):
        model.evaluate(P.build_system(pos, np.full(len(pos), 11), batch=batch))
    # forward(): the species check is remembered for an unmodified tensor and redone after a write
    zt, pt = torch.as_tensor(z.copy()), torch.as_tensor(pos, dtype=torch.float32)
    e1, _ = model(zt, pt, torch.as_tensor(batch))
    e2, _ = model(zt, pt, torch.as_tensor(batch))
    assert torch.equal(e1, e2)
    zt[0] = 10
    with pytest.raises(P.ValidationError, match="out of range"):
        model(zt, pt, torch.as_tensor(batch))
    zt[0] = -1
    with pytest.raises(P.ValidationError, match=">= 0"):
        model(zt, pt, torch.as_tensor(batch))
    zn = z.copy()
    model(zn, pos.astype(np.float32), batch)
    zn[0] = 12                                          # numpy input mutated in place: checked every call
    with pytest.raises(P.ValidationError, match="out of range"):
        model(zn, pos.astype(np.float32), batch)


def test_unsorted_lists_and_bad_batches_are_refused(rng):
    """evaluate() bisects rows by sender, so a deterministic=False list is rejected; forward(check=True)
    validates the sample codes the way build_system does in the reference."""
    z, pos, batch, _ = small_open(rng, 24)
    model = P.TensorNet(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=1)
    system = P.build_system(pos, z, batch=batch)
    loose = P.build_neighbor_list(system, P.NeighborSpec(cutoff_upper=4.0, capacity=2000, full_list=True,
                                                         include_self_loops=True, deterministic=False))
    with pytest.raises(P.ValidationError, match="sorted by sender"):
        model.evaluate(system, loose)
    zt, pt = torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32)
    bad = batch.copy()
    bad[3] = 1                                     # 0 0 0 1 0 ...: decreasing
    with pytest.raises(P.ValidationError, match="non-decreasing"):
        model(zt, pt, torch.as_tensor(bad))
    with pytest.raises(P.ValidationError, match="n_samples"):
        model(zt, pt, torch.as_tensor(batch), n_samples=1)
    with pytest.raises(P.ValidationError, match="n_samples"):
        model(zt, pt, torch.as_tensor(batch - 1))
    # gaps (empty samples) are fine: energies of the empty samples are zero
    e, _ = model(zt, pt, torch.as_tensor(batch * 2))
    e0, _ = model(zt, pt, torch.as_tensor(batch))
    assert e.shape == (3,) and float(e[1]) == 0.0
    assert torch.equal(e[[0, 2]], e0)


def test_gemm_engine_is_per_model_and_thread_safe(rng):
    """The GEMM engine travels in the model struct (nnp_tn_model.gemm_mode), not in a process
    global: two models with different engines evaluated from two threads at once give exactly
    what each gives alone, and the same as the library-wide switch gives."""
    import threading

    z, pos, batch, _ = small_open(rng, 40)
    args = (torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), torch.as_tensor(batch))
    kw = dict(embedding_dimension=64, num_layers=2, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=1,
              use_graph=False)
    ffma, mma = P.TensorNet(gemm_mode=8, **kw), P.TensorNet(gemm_mode=1, **kw)
    plain = P.TensorNet(**kw)
    alone = {"ffma": ffma(*args), "mma": mma(*args)}
    for mode, key in ((0, "ffma"), (1, "mma")):
        _lib.load().nnp_set_gemm_mode(mode)
        try:
            e, f = plain(*args)
        finally:
            _lib.load().nnp_set_gemm_mode(_lib.DEFAULT_GEMM_MODE)
        assert torch.equal(e, alone[key][0]) and torch.equal(f, alone[key][1])
    out = {}

    def work(name, model):
        torch.cuda.set_device(0)
        with torch.cuda.stream(torch.cuda.Stream()):
            for _ in range(20):
                out[name] = model(*args)
            torch.cuda.current_stream().synchronize()

    threads = [threading.Thread(target=work, args=(n, m)) for n, m in (("ffma", ffma), ("mma", mma))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for key in ("ffma", "mma"):
        assert torch.equal(out[key][0], alone[key][0]) and torch.equal(out[key][1], alone[key][1])
    with pytest.raises(P.ValidationError, match="gemm_mode"):
        P.TensorNet(gemm_mode=2, **kw)


def test_saved_weights_and_a_structure_file_reproduce_the_model(tmp_path, rng):
    """TensorNet.save / TensorNet.load (structio weights container) and load_structure: the reloaded
    model gives bit-identical energies and forces on a structure read back from an XYZ file."""
    z, pos, _, _ = small_open(rng, 18)
    P.write_extxyz(tmp_path / "mol.xyz", [P.Frame(positions=pos, species=np.where(z == 7, 8, z).astype(np.int64), energy=0.0)])
    pos2, z2 = P.load_structure(tmp_path / "mol.xyz")
    assert np.array_equal(pos2, pos)
    a = P.TensorNet(embedding_dimension=64, num_layers=2, num_rbf=16, cutoff_upper=4.5, max_z=12, mean=0.1, std=2.0, seed=8)
    a.save(tmp_path / "model.tnw")
    b = P.TensorNet.load(tmp_path / "model.tnw")
    assert b.config == a.config
    args = (torch.as_tensor(z2), torch.as_tensor(pos2, dtype=torch.float32))
    e1, f1 = a(*args)
    e2, f2 = b(*args)
    assert torch.equal(e1, e2) and torch.equal(f1, f2)


def test_invariances_on_device(rng):
    z, pos, batch, _ = small_open(rng, 26)
    model = P.TensorNet(embedding_dimension=32, num_layers=2, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=2)
    e0, f0 = model(torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), torch.as_tensor(batch))
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    pos2 = pos @ (-q).T + np.array([1.5, -0.7, 2.2])           # improper rotation + shift
    e1, f1 = model(torch.as_tensor(z), torch.as_tensor(pos2, dtype=torch.float32), torch.as_tensor(batch))
    assert np.max(np.abs((e1 - e0).cpu().numpy()) / np.maximum(np.abs(e0.cpu().numpy()), 1.0)) < 2e-5
    fr = f0.cpu().numpy() @ (-q).T
    assert np.max(np.abs(f1.cpu().numpy() - fr)) / np.max(np.abs(fr)) < 5e-4
    # net force vanishes (translation invariance)
    assert float(f0.sum(0).abs().max()) < 1e-4 * float(f0.abs().max()) * len(pos)


def test_cell_path_full_model_forces_medium_periodic():
    """1 500 atoms at config-C density, full-size model (128 channels, 2 layers), cell strategy:
    energy and forces against the float64 oracle (the oracle needs ~30 s here)."""
    z, pos, batch, box = synth.config_c_box(n=1500, edge=24.85, seed=11)
    model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0,
                        strategy="cell")
    # The tensor cores add into their accumulators with truncation; chained over K that is a
    # systematic ~5e-6 relative shrink of every per-atom energy (all atoms off in the same
    # direction).  Every 3xTF32 engine now sums short accumulator chains in FP32 registers: hold
    # each of them to a tenth of the energy tolerance and a mean per-atom error below 1e-7.
    e_ref, f_ref, pa_ref = oracle_eval(model, z, pos, np.zeros(len(z), dtype=np.int64), box)
    for mode in (5, 3, 1):
        _lib.load().nnp_set_gemm_mode(mode)
        try:
            e, f = model(torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), None, box)
            pa = model.last_per_atom_energy(len(z)).cpu().numpy()
        finally:
            _lib.load().nnp_set_gemm_mode(_lib.DEFAULT_GEMM_MODE)
        assert abs(float(e[0]) - e_ref[0]) / abs(e_ref[0]) < 1e-6, mode
        assert abs(np.mean(pa - pa_ref)) < 1e-7, mode
        assert np.max(np.abs(f.cpu().numpy() - f_ref)) / np.max(np.abs(f_ref)) < 1e-5, mode


def test_config_c_full_size_properties():
    """23 558 atoms, 2 layers, 128 channels: finite, deterministic, zero net force, per-atom
    energies sum to the sample energy, and per-atom energies of the atoms at the centre of the
    box equal the oracle's on the sub-system inside their receptive field ((L+1) * r_u = 15 A;
    the float64 oracle on the whole box would take minutes)."""
    z, pos, batch, box = synth.config_c_box()
    n = len(pos)
    model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0)
    zt, pt = torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32)
    e1, f1 = model(zt, pt, None, box)
    per_atom = model.last_per_atom_energy(n).cpu().numpy().astype(np.float64)
    e2, f2 = model(zt, pt, None, box)
    assert torch.isfinite(e1).all() and torch.isfinite(f1).all()
    assert torch.equal(e1, e2) and torch.equal(f1, f2)
    assert float(f1.sum(0).abs().max()) < 1e-3 * float(f1.abs().max()) * 50
    assert abs(per_atom.sum() - float(e1[0])) / abs(float(e1[0])) < 1e-6
    edge = box[0, 0]
    centre = np.full(3, edge / 2)
    d = pos - centre
    d -= edge * np.rint(d / edge)
    r = np.linalg.norm(d, axis=1)
    sub = np.where(r <= 17.0)[0]
    inner = np.where(r[sub] <= 2.0)[0]
    assert len(inner) >= 2
    cfg = model.config
    ocfg = T.OracleConfig(cfg.embedding_dimension, cfg.num_layers, cfg.num_rbf, cfg.cutoff_lower,
                          cfg.cutoff_upper, cfg.max_z, cfg.mean, cfg.std)
    sp = centre + d[sub]
    nl = O.build_neighbor_list(sp, None, None, 5.0, 80 * len(sub), strategy="cell", full_list=True,
                               include_self_loops=True)
    pr, dl, ds = nl.valid()
    _, _, pa_ref = T.energy_forces_compact(model.params, ocfg, z[sub], np.zeros(len(sub), np.int64),
                                           pr, dl, ds, want_forces=False)
    err = np.max(np.abs(per_atom[sub[inner]] - pa_ref[inner]))
    assert err < 5e-6, f"per-atom energy error {err:.3e}"


def test_config_d_full_size_properties():
    """8 192 molecules (~147 k atoms): finite, every molecule's forces sum to zero, per-atom energies
    sum to the sample energies, and the first molecules evaluated on their own give the same numbers
    (batch independence at full size; brute strategy inside each sample)."""
    z, pos, batch, _ = synth.config_d_molecules(8192)
    ns = int(batch[-1]) + 1
    model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0)
    zt, pt, bt = torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), torch.as_tensor(batch)
    e, f = model(zt, pt, bt)
    assert e.shape == (ns,) and torch.isfinite(e).all() and torch.isfinite(f).all()
    net = torch.zeros((ns, 3), device=f.device).index_add_(0, bt.to(f.device), f)
    assert float(net.abs().max()) < 2e-5 * max(float(f.abs().max()), 1.0)
    per_atom = model.last_per_atom_energy(len(pos), ns)
    sums = torch.zeros(ns, device=f.device).index_add_(0, bt.to(f.device), per_atom)
    assert torch.allclose(sums, e, rtol=2e-6, atol=1e-5)
    sel = batch < 16
    e_sub, f_sub = model(zt[sel], pt[sel], bt[sel])
    assert torch.allclose(e[:16], e_sub, rtol=1e-6, atol=1e-6)
    assert torch.allclose(f[: int(sel.sum())], f_sub, rtol=1e-5, atol=1e-7)
    # and against the float64 oracle on those 16 molecules
    e_ref, f_ref, _ = oracle_eval(model, z[sel], pos[sel], batch[sel], None)
    assert np.max(np.abs(e_sub.cpu().numpy() - e_ref) / np.maximum(np.abs(e_ref), 1.0)) < E_TOL
    assert np.max(np.abs(f_sub.cpu().numpy() - f_ref)) / np.max(np.abs(f_ref)) < F_TOL


def test_config_e_full_size_properties():
    """100 000 atoms in the triclinic box, 3 layers: finite, deterministic, zero net force, and
    invariant under a rigid shift of all atoms (which re-wraps them through the periodic images and
    reorders the cell lists): energy to 1e-6, forces to 1e-4 relative."""
    z, pos, batch, box = synth.config_e_triclinic()
    model = P.TensorNet(embedding_dimension=128, num_layers=3, num_rbf=32, cutoff_upper=5.0, seed=0)
    zt = torch.as_tensor(z)
    e1, f1 = model(zt, torch.as_tensor(pos, dtype=torch.float32), None, box)
    e2, f2 = model(zt, torch.as_tensor(pos, dtype=torch.float32), None, box)
    assert torch.isfinite(e1).all() and torch.isfinite(f1).all()
    assert torch.equal(e1, e2) and torch.equal(f1, f2)
    assert float(f1.sum(0).abs().max()) < 1e-3 * float(f1.abs().max()) * 100
    shifted = (pos + np.array([3.7, -11.3, 27.9])).astype(np.float32)
    e3, f3 = model(zt, torch.as_tensor(shifted), None, box)
    assert abs(float(e3[0] - e1[0])) / abs(float(e1[0])) < 2e-6
    assert float((f3 - f1).abs().max() / f1.abs().max()) < 2e-4   # float32 positions move by ~1e-6 A


# ---------------------------------------------------------------- projected embedding reverse
def _cloud22(seed):
    """Config A's 22-point cloud (0.9 A minimum separation) for another seed."""
    return synth.config_a_molecule(seed)[1]


def _both_embed_paths(z, pos, batch, box, **kw):
    """Forces from the node-projected embedding reverse and from the per-channel edge kernel."""
    out = []
    for proj in (True, False):
        model = P.TensorNet(embedding_dimension=128, num_rbf=32, embed_projection=proj, **kw)
        e, f = model(torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32),
                     None if batch is None else torch.as_tensor(batch), box)
        assert model._last_plan.proj == proj
        out.append((model, e.cpu().numpy(), f.cpu().numpy()))
    return out


@pytest.mark.parametrize("L", [0, 2])
@pytest.mark.parametrize("species", [[7], [1, 6, 8], [1, 35, 60, 99], [1, 6, 7, 8, 9], [2, 3, 5, 7, 11, 13, 17, 19, 23]])
def test_embed_projection_matches_oracle_and_edge_kernel(rng, L, species):
    """1-4 species run the projected kernels, 5 and 9 species fall back on the device; both must
    agree with the oracle and with each other (sparse species codes up to max_z - 1 included)."""
    n = 22
    pos = _cloud22(5)
    z = rng.choice(species, n)
    z[: len(species)] = species
    (mp, ep, fp), (mo, eo, fo) = _both_embed_paths(z, pos, None, None, num_layers=L, cutoff_upper=5.0,
                                                   max_z=100, seed=0)
    check(mp, z, pos, None, None)
    check(mo, z, pos, None, None)
    assert np.array_equal(ep, eo)                      # the forward sweep is the same code
    assert np.max(np.abs(fp - fo)) / np.max(np.abs(fo)) < 2e-5


def test_embed_projection_lower_cutoff_triclinic_and_batches(rng):
    box = np.array([[11.0, 0, 0], [2.5, 10.5, 0], [-3.0, 1.5, 12.0]])
    pos = (rng.uniform(0, 1, (90, 3)) @ box).astype(np.float32).astype(np.float64)
    z = rng.choice([1, 6, 8], 90)
    (mp, ep, fp), (mo, eo, fo) = _both_embed_paths(z, pos, None, box, num_layers=1, cutoff_lower=0.7,
                                                   cutoff_upper=4.5, max_z=10, seed=6)
    check(mp, z, pos, None, box)
    assert np.max(np.abs(fp - fo)) / np.max(np.abs(fo)) < 2e-5
    z, pos, batch, _ = synth.config_d_molecules(48, seed=8)
    z = np.where(z == 9, 8, z)                         # four species: the projected kernels run
    (mp, ep, fp), (mo, eo, fo) = _both_embed_paths(z, pos, batch, None, num_layers=2, cutoff_upper=5.0, seed=2)
    check(mp, z, pos, batch, None)
    assert np.max(np.abs(fp - fo)) / np.max(np.abs(fo)) < 2e-5


def test_embed_projection_species_set_changes_between_replays(rng):
    """The slot table and the species-weighted GEMM weights are rebuilt on the device every step, so
    one captured graph serves inputs with different species sets (and falls back when they exceed
    four)."""
    n = 22
    pos = _cloud22(6)
    model = P.TensorNet(embedding_dimension=128, num_layers=1, num_rbf=32, cutoff_upper=5.0, max_z=20, seed=3,
                        embed_projection=True)
    for species in ([1, 8], [6, 7, 8, 9], [1, 2, 3, 4, 5, 6], [14]):
        z = rng.choice(species, n)
        z[: len(species)] = species
        check(model, z, pos, None, None)
    assert len(model._plans) == 1 and model._last_plan.proj


def test_embed_projection_is_chosen_by_size_and_species():
    """Auto mode: projected reverse from 1 024 atoms on when at most four species are present."""
    model = P.TensorNet(embedding_dimension=128, num_layers=1, num_rbf=32, cutoff_upper=5.0, seed=1)
    z = np.resize([1, 6, 7, 8], 5000)
    assert model._use_projection(z, 5000) and model._use_projection(torch.as_tensor(z), 5000)
    assert model._use_projection(torch.as_tensor(z).cuda(), 5000)
    assert not model._use_projection(z[:1000], 1000)
    assert not model._use_projection(np.resize([1, 6, 7, 8, 9], 5000), 5000)
    small = P.TensorNet(embedding_dimension=64, num_layers=1, num_rbf=32, cutoff_upper=5.0, seed=1)
    assert not small._use_projection(z, 5000)
    with pytest.raises(P.ValidationError):
        P.TensorNet(embedding_dimension=64, num_layers=1, num_rbf=32, embed_projection=True)


def test_forward_host_equals_forward_and_regrows(rng):
    """forward_host (numpy in, numpy out, one graph with the copies inside, one synchronisation) returns
    exactly what forward returns, with and without batch codes, for float32 and float64 positions, when
    the inputs change between calls, and after a capacity overflow."""
    z, pos, batch, _ = small_open(rng, 36)
    model = P.TensorNet(embedding_dimension=32, num_layers=2, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=1)
    for dtype in (np.float32, np.float64):
        p = pos.astype(dtype)
        for b in (batch, None):
            e, f = model(torch.as_tensor(z), torch.as_tensor(p), None if b is None else torch.as_tensor(b))
            eh, fh = model.forward_host(z, p, b)
            assert eh.dtype == np.float32 and fh.shape == (len(z), 3)
            assert np.array_equal(eh, e.cpu().numpy()) and np.array_equal(fh, f.cpu().numpy())
            p2 = (p + rng.normal(0, 0.05, p.shape)).astype(dtype)          # same shape, new numbers: graph replay
            e2, f2 = model(torch.as_tensor(z), torch.as_tensor(p2), None if b is None else torch.as_tensor(b))
            eh2, fh2 = model.forward_host(z, p2, b, copy=False)
            assert np.array_equal(eh2, e2.cpu().numpy()) and np.array_equal(fh2, f2.cpu().numpy())
    tight = P.TensorNet(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=1,
                        max_num_neighbors=1)
    sparse = (np.arange(36)[:, None] * np.array([4.5, 0.0, 0.0])).astype(np.float32)
    tight.forward_host(z, sparse)                                             # fits: self loops only
    eh, fh = tight.forward_host(z, pos.astype(np.float32))                    # overflows, regrows, answers
    e, f = model.__class__(embedding_dimension=32, num_layers=1, num_rbf=8, cutoff_upper=4.0, max_z=10, seed=1)(
        torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32))
    assert np.array_equal(eh, e.cpu().numpy()) and np.array_equal(fh, f.cpu().numpy())
    with pytest.raises(P.ValidationError, match="host arrays"):
        model.forward_host(torch.as_tensor(z).cuda(), torch.as_tensor(pos).cuda())
    res = model.evaluate(P.build_system(pos, z, batch=batch))
    e, f = model(torch.as_tensor(z), torch.as_tensor(pos), torch.as_tensor(batch))
    assert np.array_equal(res.energy, e.cpu().numpy()) and np.array_equal(res.forces, f.cpu().numpy())
    assert np.allclose(np.bincount(batch, weights=res.per_atom_energy), res.energy, rtol=1e-5)
