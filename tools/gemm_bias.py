import sys, numpy as np, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2402_17660_b200 as P
from paper_2402_17660_b200 import _lib, synth
import test_gpu_tensornet as TT
z, pos, batch, box = synth.config_c_box(n=3000, edge=31.0, seed=7)
ref = None
for mode in (0, 1, 3, 5):
    _lib.load().nnp_set_gemm_mode(mode)
    m = P.TensorNet(embedding_dimension=128, num_rbf=32, num_layers=2, cutoff_upper=5.0, seed=0, strategy="cell")
    e, f = m(torch.as_tensor(z), torch.as_tensor(pos, dtype=torch.float32), None, box)
    if ref is None:
        ref = TT.oracle_eval(m, z, pos, np.zeros(len(z), dtype=np.int64), box)
    e_ref, f_ref, pa = ref
    per = m.last_per_atom_energy(len(z)).cpu().numpy()
    d = per - pa
    print("mode", mode, "E", e_ref[0], "E err", float(e[0]) - e_ref[0], "rel", (float(e[0]) - e_ref[0]) / abs(e_ref[0]), "per-atom |e| mean", np.abs(pa).mean(),
          "err mean", d.mean(), "std", d.std(), "F rel", np.max(np.abs(f.cpu().numpy() - f_ref)) / np.max(np.abs(f_ref)))
