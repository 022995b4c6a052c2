"""Summarise an ncu report: key raw metrics + stall samples per source region.
usage: python scripts/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
for r in rows[2:]:
    print("kernel:", r[h.index("Kernel Name")][:80])
    for n in WANT:
        if n in h:
            i = h.index(n)
            print(f"  {n:70s} {r[i]:>16s} {units[i]}")
    st = [(n, r[i]) for i, n in enumerate(h)
          if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
    st = sorted(st, key=lambda x: -float(x[1] or 0))[:8]
    print("  top stalls (warps per issue):", ", ".join(f"{n[34:-23]}={float(v):.2f}" for n, v in st))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if len(srows) > 3:
    hh = srows[1]
    i_s = hh.index("Warp Stall Sampling (All Samples)")

    def _num(x):
        try:
            float(x or 0)
            return True
        except ValueError:
            return False

    data = [r for r in srows[2:] if len(r) > i_s and _num(r[i_s])]  # one kernel's rows
    i_src = hh.index("Source")
    tot = sum(float(r[i_s] or 0) for r in data) or 1
    top = sorted(range(len(data)), key=lambda i: -float(data[i][i_s] or 0))[:25]
    print("top SASS by stall samples:")
    for i in sorted(top):
        print(f"  {i:5d} {float(data[i][i_s]) / tot * 100:5.1f}%  {data[i][i_src][:70]}")
