"""Instruction/stall share per line range of one source file.
usage: python scripts/ncu_ranges.py report.ncu-rep file.cu name:lo-hi ..."""
import csv, io, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    n, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((n, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
f = None; hdr = None; res = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            res.append((f, int(r[0]), float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0),
                        float(r[hdr.index("Instructions Executed")] or 0)))
        except ValueError:
            pass
ts = sum(x[2] for x in res) or 1; te = sum(x[3] for x in res) or 1
acc = {n: [0, 0] for n, _, _ in ranges}
other = [0, 0]
for ff, l, s, e in res:
    for n, lo, hi in ranges:
        if ff == fname and lo <= l <= hi:
            acc[n][0] += s; acc[n][1] += e; break
    else:
        other[0] += s; other[1] += e
for n, _, _ in ranges:
    print(f"{n:12s} stall {acc[n][0] / ts * 100:5.1f}%  inst {acc[n][1] / te * 100:5.1f}%  ({acc[n][1]:.0f})")
print(f"{'other':12s} stall {other[0] / ts * 100:5.1f}%  inst {other[1] / te * 100:5.1f}%  ({other[1]:.0f})")
