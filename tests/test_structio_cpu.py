"""Structure and weights I/O against fixtures written and parsed by the
reference itself (tests/golden/make_structio_golden.py): same arrays, same bytes out, the same
exception type and message for every malformed input."""

import json
import os

import numpy as np
import pytest

from paper_2402_17660_b200 import errors, structio
from paper_2402_17660_b200.tensornet import TNConfig, init_params

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "structio")


def test_reference_written_file_parses_to_the_reference_arrays():
    frames = structio.load_extxyz(os.path.join(HERE, "frames.xyz"))
    ref = np.load(os.path.join(HERE, "frames.npz"))
    assert len(frames) == int(ref["n_frames"]) == 4
    for k, f in enumerate(frames):
        assert np.array_equal(f.positions, ref[f"pos{k}"]) and np.array_equal(f.species, ref[f"z{k}"])
        assert f.energy == float(ref[f"e{k}"])
        assert (f.forces is None) == (f"f{k}" not in ref.files)
        if f.forces is not None:
            assert np.array_equal(f.forces, ref[f"f{k}"])
        assert f.species.dtype == np.int64 and f.n_atoms == len(f.species)


def test_writer_reproduces_the_reference_bytes(tmp_path):
    frames = structio.load_extxyz(os.path.join(HERE, "frames.xyz"))
    out = tmp_path / "again.xyz"
    structio.write_extxyz(out, frames, extra_comment='note="two words" step=3')
    assert out.read_bytes() == open(os.path.join(HERE, "frames.xyz"), "rb").read()


def test_load_structure_needs_no_energy_and_accepts_atomic_numbers():
    pos, z = structio.load_structure(os.path.join(HERE, "plain.xyz"))
    ref = np.load(os.path.join(HERE, "plain.npz"))
    assert np.array_equal(pos, ref["pos"]) and np.array_equal(z, ref["z"])
    assert z.tolist() == [8, 1, 1, 8]


def test_malformed_inputs_raise_the_reference_errors(tmp_path):
    table = json.load(open(os.path.join(HERE, "errors.json")))
    assert len(table) == 14
    for name, rec in table.items():
        path = tmp_path / f"{name}.xyz"
        path.write_text(rec["text"])
        for label, fn in (("load_extxyz", structio.load_extxyz), ("load_structure", structio.load_structure)):
            expected = rec[label]
            if expected is None:
                fn(path)
                continue
            with pytest.raises(getattr(errors, expected[0])) as info:
                fn(path)
            assert str(info.value) == expected[1], (name, label)
    with pytest.raises(errors.DataError, match="no such file"):
        structio.load_extxyz(tmp_path / "absent.xyz")


def test_symbols():
    assert structio.symbol_to_z("Xe") == 54 and structio.z_to_symbol(35) == "Br"
    with pytest.raises(errors.ValidationError):
        structio.symbol_to_z("h")
    with pytest.raises(errors.ValidationError):
        structio.z_to_symbol(0)


def test_weights_round_trip_and_refusals(tmp_path):
    cfg = TNConfig(embedding_dimension=32, num_layers=2, num_rbf=8, cutoff_upper=4.5, max_z=12, mean=0.25, std=1.5)
    params = init_params(cfg, seed=5)
    path = tmp_path / "model.tnw"
    structio.save_weights(path, cfg, params)
    cfg2, params2 = structio.load_weights(path)
    assert cfg2 == cfg and set(params2) == set(params)
    for k in params:
        assert np.array_equal(np.asarray(params2[k]), np.asarray(params[k])), k
        assert np.asarray(params2[k]).shape == np.asarray(params[k]).shape, k
    raw = path.read_bytes()
    (tmp_path / "cut.tnw").write_bytes(raw[: len(raw) // 2])
    with pytest.raises(errors.DataError, match="truncated"):
        structio.load_weights(tmp_path / "cut.tnw")
    (tmp_path / "ckpt.bin").write_bytes(b"MDKC" + raw[4:])
    with pytest.raises(errors.DataError, match="trainer checkpoint"):
        structio.load_weights(tmp_path / "ckpt.bin")
    (tmp_path / "other.bin").write_bytes(b"ABCD" + raw[4:])
    with pytest.raises(errors.DataError, match="not a TensorNet weights file"):
        structio.load_weights(tmp_path / "other.bin")
    with pytest.raises(errors.DataError, match="no such weights file"):
        structio.load_weights(tmp_path / "absent.tnw")
    fewer = dict(params)
    del fewer["h2_w"]
    structio.save_weights(tmp_path / "fewer.tnw", cfg, fewer)
    with pytest.raises(errors.DataError, match="missing array 'h2_w'"):
        structio.load_weights(tmp_path / "fewer.tnw")
