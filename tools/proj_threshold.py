"""Step time with the projected embedding reverse forced on / off, by atom count (GPU box)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import synth
for n in (1000, 2489, 4096, 5807, 12000):
    edge = (n / 0.09776) ** (1.0 / 3.0)
    z, pos, batch, box = synth.config_c_box(n=n, edge=edge, seed=3)
    out = {"atoms": n}
    for proj in (True, False):
        model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0, embed_projection=proj)
        plan = model.prepare(torch.from_numpy(z.astype(np.int32)), torch.from_numpy(pos.astype(np.float32)), None, box, n_samples=1)
        for _ in range(5): model.replay(plan)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50): model.replay(plan)
        e.record(); torch.cuda.synchronize()
        out["proj" if proj else "edge"] = round(s.elapsed_time(e) / 50, 4)
    print(json.dumps(out))
