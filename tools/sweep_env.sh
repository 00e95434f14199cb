#!/bin/bash
# Step time of config C under NNP_* tuning switches (one line per setting).
run() {
  env "$@" python bench.py --workload C --steps 20 --warmup 5 --no-sweep --no-cpu --no-md 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
k = d['kernel_ms']
print('$*', d['ms_per_step'], {n: round(k[n], 4) for n in ('k_edge_message_bwd', 'k_edge_message', 'k_embed_edge') if n in k})"
}
run NNP_NONE=1
run NNP_CPL_BWD=2
run NNP_BWD_BLOCK=64
run NNP_CPL_BWD=2 NNP_BWD_BLOCK=64
run NNP_CPL_FWD=2
run NNP_FWD_BLOCK=64
run NNP_FWD_BLOCK=256
run NNP_CPL_EMB=2
run NNP_EMB_BLOCK=64
run NNP_EMB_BLOCK=256
