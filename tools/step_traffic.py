"""Whole-step traffic from the ncu metric list of two eager config-C steps (tools/round.sh):
python tools/step_traffic.py gpurun_out/step_traffic.csv  ->  per-kernel and total DRAM / L2 / L2->L1 bytes
of the SECOND step, as JSON (profiles/r2_step_traffic.json)."""
import csv, json, sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
launches = OrderedDict()
for r in rows:
    if len(r) != len(hdr) or not r[ii].isdigit():
        continue
    d = launches.setdefault(int(r[ii]), {"kernel": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
ids = sorted(launches)
names = [launches[i]["kernel"] for i in ids]
# the second step starts at the last k_f32_to_f64 / k_sample_ptr launch
starts = [n for n, k in enumerate(names) if "k_sample_ptr" in k]
first = starts[-1] - (1 if starts[-1] > 0 and "k_f32_to_f64" in names[starts[-1] - 1] else 0)
step = [launches[i] for i in ids[first:]]
short = lambda k: k.split("(")[0].replace("void ", "").replace("<unnamed>::", "").strip()
per = OrderedDict()
tot = {"dram_bytes": 0.0, "l2_bytes": 0.0, "l2_to_l1_bytes": 0.0, "time_us": 0.0, "launches": 0}
for d in step:
    k = short(d["kernel"])
    e = per.setdefault(k, {"launches": 0, "dram_bytes": 0.0, "l2_bytes": 0.0, "l2_to_l1_bytes": 0.0, "time_us": 0.0})
    dram = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    for target in (e, tot):
        target["launches"] += 1
        target["dram_bytes"] += dram
        target["l2_bytes"] += d.get("lts__t_bytes.sum", 0.0)
        target["l2_to_l1_bytes"] += d.get("l1tex__m_xbar2l1tex_read_bytes.sum", 0.0)
        target["time_us"] += d.get("gpu__time_duration.sum", 0.0) / 1e3
out = {"what": "second eager step of tools/ncu.py C under ncu --clock-control none (cold-cache, serialised launches)",
       "total": {k: (round(v / 1e9, 3) if k.endswith("bytes") else round(v, 1)) for k, v in tot.items()},
       "units": {"bytes": "GB", "time_us": "us"},
       "per_kernel": {k: {kk: (round(vv / 1e6, 1) if kk.endswith("bytes") else round(vv, 1)) for kk, vv in v.items()} for k, v in per.items()},
       "per_kernel_units": {"bytes": "MB"}}
print(json.dumps(out, indent=1))
