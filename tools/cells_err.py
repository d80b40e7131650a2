"""Print (cell, avg_ms, frac_hbm, tc_frac) from a bench stderr log (the per-cell JSON it writes there)."""
import re
import sys

t = open(sys.argv[1]).read()
for m in re.finditer(r'\{"cell": "([^"]+)", "avg_ms": ([0-9.]+)[^}]*?"frac_hbm": ([0-9.]+)[^}]*?\}', t):
    tc = re.search(r'"tc_frac": ([0-9.]+)', m.group(0))
    print(f"{m.group(1):34s} {float(m.group(2)) * 1e3:9.2f} us  hbm {m.group(3)}  tc {tc.group(1) if tc else '-'}")
