"""Rewrite DESIGN.md's suite results paragraph + per-cell table from profiles/r01_cells.json
(the block from 'Suite: **' to the line before 'History:')."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = dict(json.load(open(os.path.join(ROOT, "profiles", "r01_cells.json"))))
line = d["line"]
rows = []
for c in d["cells"]:
    extra = ("TC %.4f" % c["tc_frac"]) if "tc_frac" in c else (("%.4f" % c["fma_frac"]) if "fma_frac" in c else "")
    rows.append(f"| {c['cell']} | {c['avg_ms'] * 1000:.1f} | {c['gelem_s']:.0f} | {c['gbs']:.0f} | "
                f"{c['frac_hbm']:.3f} | {c['frac_8tbs']:.3f} | {extra} |")
hb = line["hbm_gbs"]
text = (f"Suite: **{line['value']:.1f} GElem/s**, {line['ms_per_step']:.3f} ms/step, {hb:.0f} GB/s algorithmic "
        f"({hb / 6556.2 * 100:.1f}% of measured HBM,\n{hb / 8000 * 100:.0f}% of 8 TB/s); e2e {line['e2e']['value']:.1f} "
        f"GElem/s ({line['e2e']['ms_per_step']:.1f} ms/step, PCIe-bound); CPU oracle\n"
        f"{line['cpu_baseline']['value']:.4f} GElem/s ({line['cpu_baseline']['cores']} core); CUDA-graph replay "
        f"of the step: {line['config'].get('cuda_graph')}. Per kernel, from the "
        "instrumented eager pass (each cell also pays for the L2 write-back of\nthe previous cell's output and for the "
        "event pair around it, so isolated numbers are higher -- e.g. cfg4 2x2\nruns at 6.0 TB/s alone under ncu):\n\n"
        "| cell | us | GElem/s | GB/s | of 6549 | of 8 TB/s | FP32 FMA / TC frac |\n|---|---|---|---|---|---|---|\n"
        + "\n".join(rows) + "\n\n")
p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
a = s.index("Suite: **")
b = s.index("History:", a)
s = s[:a] + text + s[b:]
open(p, "w").write(s)
print(line["value"])
