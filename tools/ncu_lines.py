"""Top CUDA source lines by warp-stall samples in an ncu report (needs -lineinfo
and --import-source).  Usage: python tools/ncu_lines.py report.ncu-rep [launch] [n]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                               "--launch-skip", str(k), "--launch-count", "1"], stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r[:2] == ["Line No", "Source"])
hdr = rows[hi]
key = hdr.index("Warp Stall Sampling (All Samples)")
per_line = defaultdict(float)
text = {}
for r in rows[hi + 1:]:
    if len(r) != len(hdr) or not r[0].isdigit():
        continue
    try:
        per_line[int(r[0])] += float(r[key] or 0)
    except ValueError:
        continue
    text[int(r[0])] = r[1]
tot = sum(per_line.values()) or 1
for ln, v in sorted(per_line.items(), key=lambda t: -t[1])[:n]:
    print(f"{v:8.0f} {100 * v / tot:5.1f}%  L{ln:<5d} {text[ln].strip()[:100]}")
