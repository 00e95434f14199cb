#!/bin/bash
# ncu --set full of selected kernels of the second eager config-C step
mkdir -p gpurun_out
PAT=${1:-"k_edge_message|k_embed_edge|gemm_nt_tc5"}
NAME=${2:-prof_edges}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$PAT" -s ${3:-14} -c ${4:-14} \
      -f -o gpurun_out/$NAME python tools/ncu.py C > gpurun_out/$NAME.log 2>&1
tail -3 gpurun_out/$NAME.log
ls -la gpurun_out | tail -3
