#!/bin/bash
# Round-1 profiling pass (run under gpurun): launch list + full captures of the top kernels.
set -x
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 130 -c 260 --csv \
    --log-file gpurun_out/launches.csv $BENCH > gpurun_out/launches_bench.log 2>&1
for K in k_edge_message_bwd k_edge_message gemm_nt_kernel k_rows k_embed_edge_bwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 2 \
      -f -o gpurun_out/prof_$K $BENCH > gpurun_out/prof_$K.log 2>&1
done
ls -la gpurun_out
