#!/bin/bash
# A/B of environment switches on the headline bench: tools/ab.sh "VAR=a VAR=b ..." [workload]
mkdir -p gpurun_out
W=${2:-C}
for S in $1; do
  env $S timeout 600 python bench.py --workload $W --steps 30 --warmup 5 --no-sweep --no-cpu --no-md > gpurun_out/ab_$S.json 2>gpurun_out/ab_$S.err || tail -5 gpurun_out/ab_$S.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/ab_$S.json").read().strip().splitlines()[-1])
print("$W $S", d["ms_per_step"], "ms", {k: round(v,4) for k,v in list(d["kernel_ms"].items())[:12]})
PY
done
