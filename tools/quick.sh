#!/bin/bash
# Quick GPU check: selected tests (-k "$1"), then the headline bench with and without the projected embedding reverse.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensornet.py -m gpu -x -q --timeout 300 -p no:cacheprovider -k "${1:-embed_projection}" 2>&1 | tail -15
for W in ${2:-C}; do
  for P in 1 0; do
    NNP_EMBED_PROJ=$P timeout 600 python bench.py --workload $W --steps 30 --warmup 5 --no-sweep --no-cpu --no-md > gpurun_out/q_$W$P.json 2>gpurun_out/q_$W$P.err || tail -5 gpurun_out/q_$W$P.err
    python - <<PY
import json
d=json.loads(open("gpurun_out/q_$W$P.json").read().strip().splitlines()[-1])
print("$W proj=$P", d["ms_per_step"], "ms", {k: round(v,4) for k,v in list(d["kernel_ms"].items())[:14]})
PY
  done
done
