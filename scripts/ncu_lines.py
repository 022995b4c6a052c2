"""Per-CUDA-source-line instruction and stall totals from an ncu report.
usage: python scripts/ncu_lines.py report.ncu-rep [top] [kernel-regex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kf = ["--kernel-name", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
f = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_e = hdr.index("Instructions Executed")
        try:
            res.append((f, int(r[0]), r[1].strip()[:70], float(r[i_s] or 0), float(r[i_e] or 0)))
        except ValueError:
            pass
ts = sum(x[3] for x in res) or 1
te = sum(x[4] for x in res) or 1
print(f"total samples {ts:.0f} inst {te:.0f}")
for x in sorted(res, key=lambda x: -(x[3] / ts + x[4] / te))[:top]:
    print(f"{x[0]:>12s}:{x[1]:<5d} stall {x[3] / ts * 100:5.1f}%  inst {x[4] / te * 100:5.1f}%  {x[2]}")
