"""Rebuild profiles/ncu_traffic.json (bench.py's `traffic` / `ncu` fields) from one GPU round:
per-launch dram bytes of K1 and the line kernels from the `ncu --set full` captures, and the
whole sweep's dram bytes from the launch list of the bench command (ncu --metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum), averaged over its sweeps.

    python tools/update_traffic.py <tag>      (reads gpurun_out/<tag>_*)"""
import collections
import csv
import json
import os
import subprocess
import sys

tag = sys.argv[1]
O = "gpurun_out"
WANT = {"dram__bytes_read.sum": "rd", "dram__bytes_write.sum": "wr",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
        "launch__registers_per_thread": "regs", "gpu__time_duration.sum": "time"}


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for i, n in enumerate(h):
        if n in WANT:
            x = float(v[i].replace(",", ""))
            unit = u[i]
            if WANT[n] in ("rd", "wr"):
                x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d[WANT[n]] = x
    return d


res = {"source": f"ncu --set full --clock-control none (gpurun_out/{tag}_prof_*.ncu-rep, copied to profiles/r02/), "
                 f"dram__bytes_read.sum + dram__bytes_write.sum per launch; c5:sweep from the launch list of "
                 f"`bench.py --steps 2 --warmup 1` (dram bytes of the sweep's kernels / sweeps)",
       "counters": {}}
for key, rep in (("c5:k1", "k1"), ("c5:line_x", "row"), ("c5:line_y_nl", "colnl")):
    path = os.path.join(O, f"{tag}_prof_{rep}.ncu-rep")
    if not os.path.exists(path):
        continue
    d = full(path)
    res[key] = d["rd"] + d["wr"]
    res["counters"][key] = {k: d[k] for k in ("dram_pct", "fp64_pipe_pct", "issue_active_pct", "occupancy_pct", "regs")}
# whole sweep: K1 launches = sweeps; sum the dram bytes of the sweep kernels
rows = list(csv.reader(open(os.path.join(O, f"{tag}_launches.csv"))))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
ui = h.index("Metric Unit") if "Metric Unit" in h else None
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) > vi:
        x = float(r[vi].replace(",", ""))
        if ui is not None and "bytes" in r[mi]:
            x *= SCALE.get(r[ui], 1)
        per[r[ii]][r[mi]] = x
        per[r[ii]]["name"] = r[ki]
tot, sweeps = 0.0, 0
sweep_kernels = ("k_time_ring", "k_time_wp", "k_time_tma", "k_line<2048, 0, 0", "k_line<2048, 1, 1", "k_stage3p", "k_reduce_rows")
first_k1 = None
for lid in sorted(per, key=int):
    d = per[lid]
    if any(s in d["name"] for s in ("k_time_ring", "k_time_wp", "k_time_tma")):
        sweeps += 1
        first_k1 = first_k1 or int(lid)
for lid in sorted(per, key=int):
    d = per[lid]
    if first_k1 is not None and int(lid) < first_k1 - 200:
        continue
    if any(s in d["name"] for s in sweep_kernels):
        tot += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
res["c5:sweep"] = tot / max(sweeps, 1)
res["c5:sweep_note"] = f"{sweeps} sweeps in the launch list; {tot / 1e9:.1f} GB over them"
json.dump(res, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(res, indent=1))
