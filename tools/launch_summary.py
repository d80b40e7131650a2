"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*.sum --csv,
--cache-control all) of one bench command against its per-cell CUDA-event times.
One graph replay of the step = the first n_cells consecutive libss launches that
start with a kernel matching FIRST (the first cell's kernel), in cell order.
Usage: python tools/launch_summary.py launches.csv cells.json out.md FIRST [traffic.json]"""
import csv
import json
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
launch = {}
order = []
for r in rows:
    k = int(r[ix["ID"]])
    if k not in launch:
        launch[k] = {"name": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]]}
        order.append(k)
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    launch[k][r[ix["Metric Name"]]] = v * scale.get(unit, 1)
cells = json.load(open(sys.argv[2]))
cl = cells["cells"]
ours = [k for k in order if " ss::" in launch[k]["name"]]
i0 = next(i for i, k in enumerate(ours) if re.search(sys.argv[4], launch[k]["name"]))
step = [launch[k] for k in ours[i0:i0 + len(cl)]]
tot_ncu = sum(s["gpu__time_duration.sum"] for s in step)
tot_ev = sum(c["avg_ms"] * 1e3 for c in cl)
lines = ["| cell | kernel | grid | ncu us (cold, serialised) | ncu share | CUDA-event us (graph, 2 buffer sets) | event share |"
         " DRAM rd MB | DRAM wr MB | algorithmic MB |", "|---|---|---|---|---|---|---|---|---|---|"]
traffic = {}
for c, s in zip(cl, step):
    t = s["gpu__time_duration.sum"]
    rd, wr = s.get("dram__bytes_read.sum", 0), s.get("dram__bytes_write.sum", 0)
    traffic[c["cell"]] = int(rd + wr)
    name = s["name"].split("(")[0].replace("void ", "").replace("ss::", "")
    lines.append(f"| {c['cell']} | `{name[:60]}` | {s['grid']} | {t:.1f} | {t / tot_ncu:.4f} | {c['avg_ms'] * 1e3:.1f} | "
                 f"{c['avg_ms'] * 1e3 / tot_ev:.4f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {c['bytes'] / 1e6:.1f} |")
lines.append(f"\nSum: ncu {tot_ncu:.1f} us, CUDA events {tot_ev:.1f} us (bench step {cells.get('step_ms', 0) * 1e3:.1f} us).")
open(sys.argv[3], "w").write("\n".join(lines) + "\n")
if len(sys.argv) > 5:
    traffic["_about"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --cache-control all launch list "
                         "(cold L2 at kernel start; output lines still dirty in L2 at kernel end are not counted)")
    json.dump(traffic, open(sys.argv[5], "w"), indent=1)
print("\n".join(lines))
