"""Per-source-line totals from `ncu -i X --page source --csv --print-source sass,cuda`:
instructions executed, stall samples, shared wavefronts. Usage:
  python scripts/ncu_lines.py src.csv [top_n]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
fname, hdr, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    def g(name):
        try:
            return float(r[hdr.index(name)])
        except (ValueError, IndexError):
            return 0.0
    out.append((fname, ln, r[1].strip()[:70], g("Instructions Executed"), g("Warp Stall Sampling (All Samples)"),
                g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Ideal")))
ti = sum(o[3] for o in out) or 1
ts = sum(o[4] for o in out) or 1
tw = sum(o[5] for o in out) or 1
print(f"total inst {ti:.3e}  stall samples {ts:.0f}  smem wavefronts {tw:.3e}")
for key, lab in ((3, "instructions"), (4, "stall samples"), (5, "smem wavefronts")):
    print(f"--- top by {lab}")
    for o in sorted(out, key=lambda o: -o[key])[:top]:
        print(f"{o[0]}:{o[1]:<5} inst {o[3]/ti*100:5.1f}%  stall {o[4]/ts*100:5.1f}%  smem {o[5]/tw*100:5.1f}% (ideal {o[6]/max(o[5],1):.2f})  {o[2]}")
