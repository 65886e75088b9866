"""Summarise an ncu report (raw page + SASS source page) per kernel, as text.

  python scripts/ncu_report.py gpurun_out/prof.ncu-rep [kernel-regex] > profiles/rNN/xxx.txt

Prints, per profiled launch: duration, DRAM bytes read/written, DRAM / FMA / LSU / issue
utilisation, registers, warps active, the top stall reasons, and (for the first launch of
each kernel) the SASS instructions holding the most stall samples.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    h, units = raw[0], raw[1]
    un = dict(zip(h, units))
    seen = set()
    for row in raw[2:]:
        d = dict(zip(h, row))
        name = d.get("Kernel Name", "?")
        if kre and kre not in name:
            continue
        print("=" * 100)
        print(name[:140])
        for k in KEYS:
            if k in d:
                print(f"  {k:66s} {d[k]:>18s} {un.get(k, '')}")
        st = []
        for c in h:
            if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued"):
                try:
                    st.append((float(d[c].replace(",", "")), c))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        for v, c in sorted(st, reverse=True)[:8]:
            print(f"  stall {c[len('smsp__pcsamp_warps_issue_stalled_'):]:30s} {100 * v / tot:5.1f}%")
        short = name.split("(")[0]
        if short in seen:
            continue
        seen.add(short)
        src = ncu(["-i", rep, "--page", "source", "--csv", "-k", "regex:" + short.split("::")[-1].split("<")[0]])
        rows = list(csv.reader(io.StringIO(src)))
        if len(rows) < 3:
            continue
        data = []
        for n, r in enumerate(rows[2:]):
            try:
                data.append((int(r[2] or 0), n, r[1].strip()))
            except (ValueError, IndexError):
                pass
        tot = sum(x[0] for x in data) or 1
        print(f"  top SASS stall sites ({tot} samples):")
        for s, n, ins in sorted(data, reverse=True)[:12]:
            print(f"    {100 * s / tot:5.1f}%  #{n:5d}  {ins[:90]}")


if __name__ == "__main__":
    main()
