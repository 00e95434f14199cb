"""Projected embedding reverse at config D's edge density (18 neighbours per atom): the 8 192-molecule
batch with fluorine relabelled as oxygen (four species, so the projection applies), step time with
the projection forced on / off (GPU box).  Decides whether widening the projection to eight species
slots (two more GEMMs per step) could pay for the five-species config D."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import _lib, synth
z, pos, batch, _ = synth.config_d_molecules(8192)
z = np.where(z == 9, 8, z)
ns = int(batch[-1]) + 1
out = {"atoms": len(z), "species": sorted(set(z.tolist()))}
for proj in (True, False):
    model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0, embed_projection=proj)
    plan = model.prepare(torch.from_numpy(z.astype(np.int32)), torch.from_numpy(pos.astype(np.float32)),
                         torch.from_numpy(batch.astype(np.int32)), None, n_samples=ns)
    for _ in range(3): model.replay(plan)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): model.replay(plan)
    e.record(); torch.cuda.synchronize()
    key = "projected" if proj else "per_channel"
    out[key + "_ms"] = round(s.elapsed_time(e) / 10, 3)
    prof = _lib.profile_step(lambda: model.enqueue_eager(plan))
    out[key + "_kernels"] = {k: round(v[0], 3) for k, v in prof.items() if "embed" in k}
    out["edges"] = int(plan.engine.counts[0].item())
print(json.dumps(out))
