#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_tensornet.py -x -q --timeout 300 -p no:cacheprovider -k "gemm or small_open or config_a or triclinic" 2>&1 | tail -2
run() { env "$@" timeout 200 python tools_tune.py $WL 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['wl'], d['graph_ms'], d['E'], {k:v for k,v in list(d['top'].items())[:8]})"; }
for WL in A; do export WL; run NNP_X=1; done
