"""Copy a round's GPU artefacts from gpurun_out/ into profiles/ (tracked) and
derive profiles/traffic.json (DRAM bytes per launch of each bench cell, from
the ncu --set full capture, which profiles one bench step's kernels in cell
order).  Usage: python tools/make_profiles.py TAG ROUND"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

tag, rnd = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
g = os.path.join(root, "gpurun_out")
prof = os.path.join(root, "profiles")
os.makedirs(prof, exist_ok=True)
for src, dst in ((f"bench_full_{tag}.json", f"{rnd}_bench.json"), (f"cells_full_{tag}.json", f"{rnd}_cells.json"),
                 (f"bench_ref_{tag}.json", f"{rnd}_bench_reference.json"), (f"launches_{tag}.csv", f"{rnd}_launches.csv"),
                 (f"smi_{tag}.csv", f"{rnd}_nvidia_smi.csv")):
    if os.path.exists(os.path.join(g, src)):
        shutil.copy(os.path.join(g, src), os.path.join(prof, dst))
rep = os.path.join(g, f"prof_full_{tag}.ncu-rep")
if os.path.exists(rep):
    subprocess.check_call([sys.executable, os.path.join(root, "tools", "ncu_summary.py"), rep,
                           os.path.join(prof, f"{rnd}_ncu_full_summary.md")], stdout=subprocess.DEVNULL)
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def val(row, name):
        i = hdr.index(name)
        return float(row[i].replace(",", "")) * scale.get(units[i], 1)
    cells = json.load(open(os.path.join(prof, f"{rnd}_cells.json")))["cells"]
    traffic = {}
    for c, row in zip(cells, data):
        traffic[c["cell"]] = int(val(row, "dram__bytes_read.sum") + val(row, "dram__bytes_write.sum"))
    traffic["_about"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch from ncu --set full "
                         f"({rnd}, one bench step, cold/serialised launches; writes still in L2 at kernel "
                         f"end are not counted)")
    json.dump(traffic, open(os.path.join(prof, "traffic.json"), "w"), indent=1)
print("profiles updated")
