#!/bin/bash
timeout 120 python -m pytest tests/test_gpu_tensornet.py -q -x -k "gemm" --timeout 100 -p no:cacheprovider 2>&1 | tail -8
timeout 400 python -m pytest tests/test_gpu_tensornet.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -5
for G in 2 3; do
  NNP_GEMM_MODE=$G timeout 200 python tools_tune.py C 2>&1 | tail -1
done
NNP_BWD_BLOCK=256 timeout 200 python tools_tune.py C 2>&1 | tail -1
NNP_CPL_BWD=2 timeout 200 python tools_tune.py C 2>&1 | tail -1
timeout 200 python tools_tune.py A 2>&1 | tail -1
timeout 200 python tools_tune.py D 2>&1 | tail -1
