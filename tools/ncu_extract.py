"""Per-kernel extract of an ncu --set full report as CSV rows (appended to profiles/rN_ncu_kernels.csv):
python tools/ncu_extract.py gpurun_out/prof.ncu-rep capture_label >> profiles/r2_ncu_kernels.csv"""
import csv, io, subprocess, sys
rep, label = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "lts__t_sectors_srcunit_tex.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "sm__cycles_elapsed.max",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
ki = hdr.index("Kernel Name")
w = csv.writer(sys.stdout)
if len(sys.argv) > 3:
    w.writerow(["capture", "kernel"] + want)
for r in data:
    w.writerow([label, r[ki]] + [(r[hdr.index(m)] + " " + units[hdr.index(m)]).strip() if m in hdr else "" for m in want])
