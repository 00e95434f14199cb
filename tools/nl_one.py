"""One neighbor build of config B at n atoms (half list, cell strategy): the command ncu wraps."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import synth
from paper_2402_17660_b200.neighbors import NeighborEngine, plan_strategy
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
_, pos, batch, boxm = synth.config_b_cloud(n)
box = P.Box.from_matrix(boxm)
code, dims, mc, _ = plan_strategy(n, box, 5.0, "cell")
eng = NeighborEngine(n, 1, 32 * n, box, 0.0, 5.0, code, dims, mc, 0)
dp = torch.from_numpy(pos).cuda(); db = torch.zeros(n, dtype=torch.int32, device="cuda")
for _ in range(2): eng.build(dp, db)
torch.cuda.synchronize()
print("pairs", int(eng.counts[0]))
