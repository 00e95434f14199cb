"""Per-kernel timing of one config-C step under the current NNP_* environment (GPU box)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import _lib, synth

wl = sys.argv[1] if len(sys.argv) > 1 else "C"
if wl == "C":
    z, pos, batch, box = synth.config_c_box()
elif wl == "A":
    z, pos, batch, box = synth.config_a_molecule()
elif wl == "D":
    z, pos, batch, box = synth.config_d_molecules(1024)
model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0)
ns = int(batch[-1]) + 1
plan = model.prepare(torch.from_numpy(z.astype(np.int32)), torch.from_numpy(pos.astype(np.float32)),
                     None if ns == 1 else torch.from_numpy(batch.astype(np.int32)), box, n_samples=ns)
for _ in range(3):
    model.enqueue_eager(plan)
torch.cuda.synchronize()
acc = {}
R = 5
for _ in range(R):
    for k, (ms, c) in _lib.profile_step(lambda: model.enqueue_eager(plan)).items():
        acc[k] = acc.get(k, 0.0) + ms / R
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    model.replay(plan)
s.record()
for _ in range(20):
    model.replay(plan)
e.record(); torch.cuda.synchronize()
env = {k: v for k, v in os.environ.items() if k.startswith("NNP_")}
top = sorted(acc.items(), key=lambda kv: -kv[1])[:40]
print(json.dumps({"env": env, "wl": wl, "graph_ms": round(s.elapsed_time(e) / 20, 4),
                  "top": {k: round(v, 4) for k, v in top}, "E": float(plan.energy[0])}))
