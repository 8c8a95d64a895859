"""Per-CUDA-line totals from `ncu --page source --csv --print-source=cuda,sass`
(lines whose Address is '-' carry the line aggregates): executed
warp-instructions, stall samples and shared-memory excess wavefronts (bank
conflicts), sorted by a chosen column.
    python tools/ncu_src_lines.py SOURCE.csv [N] [sort: inst|stall|conf]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(r for r in rows if r and r[0] == "Line No")
ix = {k: i for i, k in enumerate(h)}
def col(r, k):
    try:
        return float(r[ix[k]].replace(",", "") or 0)
    except (ValueError, KeyError, IndexError):
        return 0.0
out = []
for r in rows[rows.index(h) + 1:]:
    if len(r) < len(h) or r[2] != "-":
        continue
    out.append((col(r, "Instructions Executed"), col(r, "Warp Stall Sampling (All Samples)"),
                col(r, "L1 Wavefronts Shared Excessive"), col(r, "L1 Wavefronts Shared"), r[0], r[1]))
ti = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
tc = sum(o[2] for o in out) or 1
tw = sum(o[3] for o in out) or 1
print(f"warp-inst {ti:.0f}  stall samples {ts:.0f}  smem wavefronts {tw:.0f}  excessive {tc:.0f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = {"inst": 0, "stall": 1, "conf": 2}[sys.argv[3] if len(sys.argv) > 3 else "inst"]
for o in sorted(out, key=lambda x: -x[key])[:n]:
    print(f"inst {o[0]/ti:6.1%} stall {o[1]/ts:6.1%} conf {o[2]/tc:6.1%} ({o[2]:9.0f}/{o[3]:9.0f}) L{o[4]:>5} {o[5].strip()[:70]}")
