#!/bin/bash
timeout 200 python -m pytest tests/test_gpu_tensornet.py -q -x -k "gemm or periodic_triclinic or config_a" --timeout 150 -p no:cacheprovider 2>&1 | tail -3
for DBG in 0 512; do
  NNP_GEMM_DBG=$DBG NNP_GEMM_MODE=4 timeout 200 python tools_tune.py C 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['wl'], d['graph_ms'], 'gemm_mix', d['top'].get('gemm_mix'), 'dense', d['top'].get('gemm_dense'))"
done
