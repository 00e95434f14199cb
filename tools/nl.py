"""Neighbor-build kernel breakdown (GPU box)."""
import json, sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import _lib, synth
from paper_2402_17660_b200.neighbors import NeighborEngine, plan_strategy
for n, strategy in ((1000, "cell"), (1000, "brute"), (65536, "cell"), (1048576, "cell")):
    _, pos, batch, boxm = synth.config_b_cloud(n)
    box = P.Box.from_matrix(boxm)
    code, dims, mc, _ = plan_strategy(n, box, 5.0, strategy)
    eng = NeighborEngine(n, 1, 32 * n, box, 0.0, 5.0, code, dims, mc, 0)
    dp = torch.from_numpy(pos).cuda(); db = torch.zeros(n, dtype=torch.int32, device="cuda")
    for _ in range(3): eng.build(dp, db)
    torch.cuda.synchronize()
    _lib.load().nnp_launch_count(1)
    prof = _lib.profile_step(lambda: eng.build(dp, db))
    launches = _lib.load().nnp_launch_count(1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        eng.build(dp, db)
    g.replay(); torch.cuda.synchronize()
    s.record()
    for _ in range(10): g.replay()
    e.record(); torch.cuda.synchronize()
    print(json.dumps({"n": n, "strategy": strategy, "launches": launches, "graph_us": round(100 * s.elapsed_time(e), 1),
                      "pairs": int(eng.counts[0]), "kernels_us": {k: round(1000 * v[0], 1) for k, v in prof.items()}}))
