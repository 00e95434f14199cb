"""Extended-XYZ fixtures written and parsed by the REFERENCE ITSELF (nnpkit.data, imported read-only
from /root/reference/pkg/src).  Build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_structio_golden.py

Writes tests/golden/structio/: ``frames.xyz`` (reference writer), ``frames.npz`` (what the reference's
parser returns for it), ``plain.xyz`` (+ ``plain.npz`` from load_structure) and ``errors.json``:
malformed inputs with the reference's exact exception type and message.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from nnpkit.data import Frame, load_extxyz, load_structure, write_extxyz  # noqa: E402
from nnpkit.errors import ToolkitError  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "structio")
rng = np.random.default_rng(7)
frames = []
for k, n in enumerate((3, 7, 1, 12)):
    z = rng.choice([1, 6, 7, 8, 9, 16, 17, 35], n)
    frames.append(Frame(positions=rng.normal(0, 3, (n, 3)), species=z.astype(np.int64),
                        energy=float(rng.normal(-50, 10)), forces=rng.normal(0, 1, (n, 3)) if k % 2 == 0 else None))
path = os.path.join(OUT, "frames.xyz")
write_extxyz(path, frames, extra_comment='note="two words" step=3')
back = load_extxyz(path)
arrays = {"n_frames": np.int64(len(back))}
for k, f in enumerate(back):
    arrays[f"pos{k}"], arrays[f"z{k}"], arrays[f"e{k}"] = f.positions, f.species, np.float64(f.energy)
    if f.forces is not None:
        arrays[f"f{k}"] = f.forces
np.savez(os.path.join(OUT, "frames.npz"), **arrays)
plain = "4\nwater dimer fragment, no energy here\nO 0.0 0.0 0.117\n1 0.0 0.757 -0.469\nH 0.0 -0.757 -0.469\n8 2.9 0.1 0.0\n"
open(os.path.join(OUT, "plain.xyz"), "w").write(plain)
p, s = load_structure(os.path.join(OUT, "plain.xyz"))
np.savez(os.path.join(OUT, "plain.npz"), pos=p, z=s)
bad = {
    "count": "x3\nenergy=1.0\nH 0 0 0\n",
    "zero_atoms": "0\nenergy=1.0\n",
    "no_comment": "1\n",
    "no_energy": "1\nfoo=2\nH 0 0 0\n",
    "bad_energy": "1\nenergy=abc\nH 0 0 0\n",
    "inf_energy": "1\nenergy=inf\nH 0 0 0\n",
    "quote": "1\nenergy=1.0 note=\"open\nH 0 0 0\n",
    "symbol": "1\nenergy=1.0\nQq 0 0 0\n",
    "negative_z": "1\nenergy=1.0\n-3 0 0 0\n",
    "fields": "1\nenergy=1.0\nH 0 0\n",
    "coordinate": "1\nenergy=1.0\nH 0 zero 0\n",
    "truncated": "2\nenergy=1.0\nH 0 0 0\n",
    "mixed_forces": "2\nenergy=1.0\nH 0 0 0 1 1 1\nH 1 0 0\n",
    "empty": "\n\n",
}
errors = {}
for name, text in bad.items():
    f = os.path.join(OUT, f"bad_{name}.xyz")
    open(f, "w").write(text)
    rec = {"text": text}
    for label, fn in (("load_extxyz", load_extxyz), ("load_structure", load_structure)):
        try:
            fn(f)
            rec[label] = None
        except ToolkitError as err:
            rec[label] = [type(err).__name__, str(err)]
    os.remove(f)
    errors[name] = rec
json.dump(errors, open(os.path.join(OUT, "errors.json"), "w"), indent=1)
print("frames", len(back), "errors", len(errors))
