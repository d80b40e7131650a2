"""Per-instruction view of one kernel in an ncu report (SASS source page):
instruction mix, smem excessive wavefronts, top stall lines.
Usage: python tools/ncu_source.py report.ncu-rep <launch-index>"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, k = sys.argv[1], int(sys.argv[2])
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(k),
                               "--launch-count", "1", "--print-source", "sass"], stderr=subprocess.DEVNULL).decode()
rows = [r for r in csv.reader(io.StringIO(raw))]
print(rows[0][:2])
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}


def v(r, c):
    try:
        return int(float(r[ix[c]] or 0))
    except (ValueError, KeyError):
        return 0


print("samples", sum(v(r, "# Samples") for r in data), "warp-instructions", sum(v(r, "Instructions Executed") for r in data))
mix = Counter()
for r in data:
    s = r[ix["Source"]].strip().split()
    if not s:
        continue
    op = s[1] if s[0].startswith("@") else s[0]
    mix[op.split(".")[0]] += v(r, "Instructions Executed")
print("mix", mix.most_common(20))
ex = sorted(data, key=lambda r: -v(r, "L1 Wavefronts Shared Excessive"))[:8]
for r in ex:
    if v(r, "L1 Wavefronts Shared Excessive"):
        print("smem-excess", v(r, "L1 Wavefronts Shared Excessive"), v(r, "L1 Wavefronts Shared"), r[ix["Source"]].strip()[:70])
for r in sorted(data, key=lambda r: -v(r, "# Samples"))[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
    print("stall", v(r, "# Samples"), r[ix["Address"]][-5:], r[ix["Source"]].strip()[:90])
