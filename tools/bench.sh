#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 10 > gpurun_out/bench_C.json 2>gpurun_out/bench_C.err
tail -c 600 gpurun_out/bench_C.err
for W in A D E; do
  timeout 600 python bench.py --workload $W --steps 30 --warmup 5 --no-sweep --no-cpu > gpurun_out/bench_$W.json 2>gpurun_out/bench_$W.err
  tail -c 300 gpurun_out/bench_$W.err
done
python - <<'PY'
import json
for w in "CADE":
    try:
        d=json.loads(open(f"gpurun_out/bench_{w}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(w, "FAILED", e); continue
    print(w, d["value"], d["unit"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "step_frac", d["step_roofline"]["frac"], "launches", d["launches_per_step"], d["clocks"])
    print("   roofline", d["roofline"])
    print("   kernels", list(d["kernel_ms"].items())[:8])
    if "cpu_baseline" in d: print("   cpu", d["cpu_baseline"]["value"])
    for r in d.get("neighbor_sweep", []): print("   ", r)
PY
