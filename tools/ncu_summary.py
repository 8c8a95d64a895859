"""Summaries of the ncu captures kept under profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv
    python tools/ncu_summary.py full gpurun_out/prof_k2.ncu-rep [records]

`launches`: per-kernel launch counts and device times from the
`--metrics gpu__time_duration.sum` pass (cold-cache, serialised: compare
shares, not absolutes). K2 launches are split into full-batch launches and
the e2e loader's per-chunk launches.
`full`: the metrics the roofline and the optimisation log cite, from one
`--set full` capture of K2 (dram bytes, issue utilisation, stall mix, smem /
L2-RED traffic, instructions per record).
"""
import collections
import csv
import io
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
            t = float(r[vi].replace(",", ""))
            if name.startswith("k2") and t > 3e5:
                name += " [full batch]"
            elif name.startswith("k2"):
                name += " [e2e chunk]"
            agg[name].append(t)
    print(f"{'launches':>8} {'avg_us':>10} {'total_us':>10}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / 1e3:10.1f}  {k}")


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__bytes.sum.per_second", "dram throughput"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps/scheduler"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 RED sectors"),
    ("lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed", "L2 RED % of peak"),
    ("sass__inst_executed_local_loads", "local loads"),
]


def full(path, records=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel: {name[:100]}")
        d = dict(zip(h, v))
        for k, label in KEYS:
            if k in d:
                print(f"  {label:28s} {d[k]:>18s} {u[h.index(k)]}")
        stalls = {k.split("stalled_")[1].replace("_per_issue_active.ratio", ""): float(d[k])
                  for k in h if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:7]
        print("  stall mix (cycles/issue):  " + ", ".join(f"{k}={x:.2f}" for k, x in top)
              + f"  (total {tot:.1f})")
        if records and "smsp__inst_executed.sum" in d:
            wi = float(d["smsp__inst_executed.sum"].replace(",", ""))
            print(f"  warp-instructions/record     {wi / records:18.2f}")
            rd = float(d["dram__bytes_read.sum"].replace(",", ""))
            unit = u[h.index("dram__bytes_read.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            print(f"  dram read bytes/record       {rd * scale / records:18.2f}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else None)
