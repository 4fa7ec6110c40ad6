"""Print the key raw metrics and the hottest source lines of an ncu report (run here, no GPU)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.max.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
        "sm__cycles_active.max", "sm__cycles_active.min"]
for k in KEYS:
    if k in hdr:
        i = hdr.index(k)
        print(f"{k:70s} {vals[i]:>16s} {units[i]}")
if "--source" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(src)))
    h = r[1]
    ix = {x: i for i, x in enumerate(h)}
    data = r[2:]
    top = sorted(data, key=lambda x: -float(x[ix["Warp Stall Sampling (All Samples)"]] or 0))[:25]
    for x in top:
        print(x[ix["Address"]][-5:], x[ix["Source"]][:55].ljust(55), x[ix["Warp Stall Sampling (All Samples)"]],
              x[ix["Instructions Executed"]], x[ix["Avg. Threads Executed"]])
