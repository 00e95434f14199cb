#!/bin/bash
# One GPU call: parity tests, smoke, bench (all workloads), ncu launch list.  $1 = extra pytest args
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider $1 > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
bash tools/bench.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/ncu_bench.log | cut -c1-300
# whole-step traffic: DRAM / L2 / L2->L1 bytes of every launch of two eager config-C steps
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file gpurun_out/step_traffic.csv python tools/ncu.py C > gpurun_out/step_traffic.log 2>&1
tail -1 gpurun_out/step_traffic.log
