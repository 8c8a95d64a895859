"""Summarise an ncu `--page source --print-source=sass --csv` dump: hottest
SASS instructions by stall samples and by executed warp-instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
recs = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    def f(k):
        try:
            return float(r[idx[k]].replace(",", "") or 0)
        except ValueError:
            return 0.0
    recs.append((r[idx["Address"]], r[idx["Source"]], f("Warp Stall Sampling (All Samples)"),
                 f("Instructions Executed"), f("Avg. Threads Executed"),
                 {k: f(k) for k in h if k.startswith("stall_") and "Not Issued" not in k}))
tot_s = sum(x[2] for x in recs)
tot_i = sum(x[3] for x in recs)
print(f"total samples {tot_s:.0f}  total warp-instructions {tot_i:.0f}")
stalls = {}
for x in recs:
    for k, v in x[5].items():
        stalls[k] = stalls.get(k, 0) + v
print("stall mix:", ", ".join(f"{k[6:]}={v/tot_s:.1%}" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("--- by samples")
for x in sorted(recs, key=lambda x: -x[2])[:n]:
    top = max(x[5].items(), key=lambda kv: kv[1])[0][6:] if x[5] else ""
    print(f"{x[0]:>6} {x[2]/tot_s:6.1%} ex={x[3]:9.0f} thr={x[4]:5.1f} {top:12s} {x[1][:70]}")
