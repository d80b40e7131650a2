"""Summarise an ncu --set full report (raw page CSV) per kernel launch: duration,
DRAM bytes/throughput, issue activity, pipe use, smem conflicts and the top
stall reasons.  Usage: python tools/ncu_summary.py report.ncu-rep [out.md]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def g(row, name, default=""):
    i = ix.get(name)
    return row[i] if i is not None else default


SCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def f(row, name, to_base=False):
    """Value of a metric; with to_base, times -> us and bytes -> MB."""
    try:
        v = float(g(row, name).replace(",", ""))
    except ValueError:
        return float("nan")
    if to_base:
        v *= SCALE.get(units[ix[name]], 1.0)
    return v


stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
out = ["| # | kernel | grid x block | regs | dur us | DRAM rd MB | DRAM wr MB | DRAM %pk | issue % | FMA pipe % | LSU % | smem ld conflicts | top stalls (warps/issue) |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for n, row in enumerate(data):
    name = g(row, "Kernel Name")
    short = name.split("(")[0].replace("void ", "")
    if "<" in short:
        short = short[:short.index("<")] + "<" + name.split("<", 1)[1].split(">")[0][:60] + ">"
    stalls = sorted(((f(row, c), c.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")) for c in stall_cols), reverse=True)[:3]
    out.append("| {} | `{}` | {} x {} | {} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.0f} | {} |".format(
        n, short, g(row, "launch__grid_size"), g(row, "launch__block_size"), g(row, "launch__registers_per_thread"),
        f(row, "gpu__time_duration.sum", True),
        f(row, "dram__bytes_read.sum", True), f(row, "dram__bytes_write.sum", True),
        f(row, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        f(row, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        f(row, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        f(row, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        f(row, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
        ", ".join(f"{s} {v:.2f}" for v, s in stalls)))
txt = "\n".join(out)
print(txt)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(txt + "\n")
