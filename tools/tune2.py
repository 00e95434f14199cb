"""Per-kernel timing at a given atom count (periodic box at config-C density)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import _lib, synth
n = int(sys.argv[1])
edge = (n / 0.09776) ** (1.0 / 3.0)
z, pos, batch, box = synth.config_c_box(n=n, edge=edge, seed=3)
model = P.TensorNet(embedding_dimension=128, num_layers=2, num_rbf=32, cutoff_upper=5.0, seed=0)
plan = model.prepare(torch.from_numpy(z.astype(np.int32)), torch.from_numpy(pos.astype(np.float32)), None, box, n_samples=1)
for _ in range(3): model.enqueue_eager(plan)
torch.cuda.synchronize()
acc = {}
for _ in range(5):
    for k, (ms, c) in _lib.profile_step(lambda: model.enqueue_eager(plan)).items():
        acc[k] = acc.get(k, 0.0) + ms / 5
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5): model.replay(plan)
s.record()
for _ in range(50): model.replay(plan)
e.record(); torch.cuda.synchronize()
print(json.dumps({"n": n, "env": {k: v for k, v in os.environ.items() if k.startswith("NNP_")}, "graph_ms": round(s.elapsed_time(e) / 50, 4), "sum_kernels": round(sum(acc.values()), 3),
                  "top": {k: round(v, 4) for k, v in sorted(acc.items(), key=lambda kv: -kv[1])[:14]}}))
