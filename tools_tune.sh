#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_tensornet.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -5
for G in 1 2; do
  NNP_GEMM_MODE=$G timeout 200 python tools_tune.py C 2>&1 | tail -1
done
NNP_GEMM_MODE=2 timeout 200 python tools_tune.py A 2>&1 | tail -1
NNP_GEMM_MODE=2 timeout 200 python tools_tune.py D 2>&1 | tail -1
