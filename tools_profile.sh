#!/bin/bash
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu"
for K in gemm_nt_tc5 k_edge_message_bwd k_embed_edge_bwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 2 \
      -f -o gpurun_out/prof2_$K $BENCH > gpurun_out/prof2_$K.log 2>&1
done
timeout 300 python tools_tune.py C 2>&1 | tail -1
ls -la gpurun_out | tail -8
