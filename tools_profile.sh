#!/bin/bash
mkdir -p gpurun_out
NNP_GEMM_MODE=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_wstat -s 4 -c 1 \
      -f -o gpurun_out/prof3_wstat python tools_tune.py C > gpurun_out/prof3_wstat.log 2>&1
ls -la gpurun_out | tail -3
