"""Accuracy and speed of the radial tables vs number of knots (config C, GPU box)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import synth
z, pos, batch, box = synth.config_c_box()
zt, pt = torch.from_numpy(z.astype(np.int32)), torch.from_numpy(pos.astype(np.float32))
ref = None
for nk in (2048, 512, 384, 256, 192, 128):
    model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0, num_knots=nk)
    plan = model.prepare(zt, pt, None, box, n_samples=1)
    for _ in range(3): model.replay(plan)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): model.replay(plan)
    e.record(); torch.cuda.synchronize()
    E, F = float(plan.energy[0]), plan.forces.clone()
    if ref is None: ref = (E, F)
    print(json.dumps({"knots": nk, "ms": round(s.elapsed_time(e)/20, 4), "table_err": model.table_error, "E": E,
                      "dE_rel": abs(E-ref[0])/abs(ref[0]), "dF_rel": float((F-ref[1]).abs().max()/ref[1].abs().max())}))
    del model, plan
    torch.cuda.empty_cache()
