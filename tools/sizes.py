"""Step time vs atom count for periodic boxes at the density of config C (GPU box)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import synth
model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0)
rows = []
for n in (166, 2489, 5807, 23558, 100000):
    if n == 166:
        z, pos, batch, box = synth.config_d_molecules(9, seed=1)      # ~166 atoms in one open cluster
        z, pos = z[:166], pos[:166] * 0.0 + np.random.default_rng(0).uniform(0, 12.0, (166, 3))
        box = None
    else:
        edge = (n / 0.09776) ** (1.0 / 3.0)
        z, pos, batch, box = synth.config_c_box(n=n, edge=edge, seed=3)
    plan = model.prepare(torch.from_numpy(z.astype(np.int32)), torch.from_numpy(pos.astype(np.float32)), None, box, n_samples=1)
    for _ in range(5): model.replay(plan)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50 if n < 50000 else 10
    s.record()
    for _ in range(reps): model.replay(plan)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    rows.append({"atoms": n, "edges": int(plan.engine.counts[0].item()), "ms_per_step": round(ms, 4),
                 "steps_per_s": round(1000 / ms, 1), "msteps_per_day": round(86.4 / ms, 2), "us_per_atom": round(1000 * ms / n, 3)})
    print(json.dumps(rows[-1]))
