"""Per-source-line totals from `ncu --page source --print-source=cuda,sass --csv`:
executed warp-instructions and stall samples (lines with a '-' address are
the line aggregates)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[2]
out = []
for r in rows[3:]:
    if len(r) < 8 or r[2] != "-":
        continue
    try:
        ex = float(r[7].replace(",", "") or 0)
        sm = float(r[4].replace(",", "") or 0)
        thr = float(r[10].replace(",", "") or 0)
    except ValueError:
        continue
    out.append((ex, sm, thr, r[0], r[1]))
tot = sum(o[0] for o in out)
tots = sum(o[1] for o in out) or 1
print(f"total warp-instructions {tot:.0f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for o in sorted(out, key=lambda x: -x[0])[:n]:
    print(f"{o[0]/tot:6.1%} stall {o[1]/tots:6.1%} thr {o[2]:5.1f} L{o[3]:>4} {o[4].strip()[:80]}")
