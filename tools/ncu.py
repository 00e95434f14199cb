"""Two eager config-C steps and nothing else: the command ncu wraps (GPU box)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import synth

wl = sys.argv[1] if len(sys.argv) > 1 else "C"
z, pos, batch, box = {"C": synth.config_c_box, "A": synth.config_a_molecule}[wl]()
model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0)
plan = model.prepare(torch.from_numpy(z.astype(np.int32)), torch.from_numpy(pos.astype(np.float32)), None, box, n_samples=1)
for _ in range(int(os.environ.get("NCU_STEPS", "2"))):
    model.enqueue_eager(plan)
torch.cuda.synchronize()
print("E", float(plan.energy[0]))
