"""Print key metrics of an ncu report (raw page) per kernel."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.avg.per_cycle_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_barrier", 
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg"]
extra = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
for row in rows[2:]:
    d = dict(zip(h, row))
    print("=" * 100)
    for w in want:
        if w in d:
            print(f"  {w:70s} {d[w]}")
    st = sorted(((float(d[c].replace(',', '') or 0), c) for c in extra if d.get(c, '').replace(',', '').replace('.', '').isdigit()), reverse=True)[:10]
    for v, c in st:
        print(f"  {c:70s} {v}")
