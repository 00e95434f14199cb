"""Full-size TensorNet fixtures from the float64 CPU oracle (oracle/tensornet_oracle.py).

The oracle needs minutes per headline configuration, which is too slow for the GPU test run, so
its answers are computed once in the build container and committed:

    python tests/golden/make_tn_golden.py [C] [D] [E]      ->  tests/golden/tn_golden_{C,D,E}.npz

* C: 23 558-atom periodic box, 2 layers, 128 channels        (BASELINE.json configs[2])
* D: the first 256 molecules of the 8 192-molecule batch      (configs[3])
* E: 100 000-atom triclinic box, **3 layers**, 128 channels   (configs[4])

Inputs are regenerated from ``synth`` by seed at test time (an input checksum is stored and
compared, so a drifting generator fails loudly instead of silently comparing different systems);
weights are ``init_params(seed=0)``.  Stored: per-sample energies (float64), forces and per-atom
energies (float32: 6e-8 relative rounding, three orders below the 1e-4 force tolerance).
"""

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import neighbors_oracle as O  # noqa: E402
from oracle import tensornet_oracle as T  # noqa: E402
from paper_2402_17660_b200 import synth  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
D_MOLECULES = 256


def checksum(z, pos, batch, box):
    h = hashlib.sha256()
    for a in (np.asarray(z, np.int64), np.asarray(pos, np.float64), np.asarray(batch, np.int64)):
        h.update(np.ascontiguousarray(a).tobytes())
    if box is not None:
        h.update(np.ascontiguousarray(box, dtype=np.float64).tobytes())
    return h.hexdigest()


def inputs(name):
    if name == "C":
        return synth.config_c_box(), 2
    if name == "D":
        z, pos, batch, box = synth.config_d_molecules(8192)
        sel = batch < D_MOLECULES
        return (z[sel], pos[sel], batch[sel], None), 2
    if name == "E":
        return synth.config_e_triclinic(), 3
    raise SystemExit(f"unknown config {name}")


def run(name):
    (z, pos, batch, box), layers = inputs(name)
    cfg = T.OracleConfig(embedding_dimension=128, num_layers=layers, num_rbf=32, cutoff_upper=5.0)
    params = T.init_params(cfg, seed=0)
    n = len(pos)
    t0 = time.time()
    nl = O.build_with_auto_capacity(pos, batch, box, cfg.cutoff_upper, 64 * n,
                                    strategy="cell" if box is not None else "brute",
                                    full_list=True, include_self_loops=True)
    pr, dl, ds = nl.valid()
    e, f, pa = T.energy_forces_compact(params, cfg, z, batch, pr, dl, ds)
    dt = time.time() - t0
    out = os.path.join(HERE, f"tn_golden_{name}.npz")
    np.savez_compressed(out, energy=e, forces=f.astype(np.float32), per_atom=pa.astype(np.float32),
                        n_edges=np.int64(len(pr)), layers=np.int64(layers),
                        inputs_sha256=np.array(checksum(z, pos, batch, box)),
                        oracle_seconds=np.float64(dt))
    print(f"{name}: {n} atoms, {len(pr)} directed edges, {layers} layers, E[0]={e[0]:.9g}, "
          f"max|F|={np.abs(f).max():.6g}, {dt:.0f} s -> {out}", flush=True)


if __name__ == "__main__":
    for name in (sys.argv[1:] or ["D", "C", "E"]):
        run(name)
