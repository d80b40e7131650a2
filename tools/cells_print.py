"""Print a bench --cells-out file as a table (line summary + per-cell times)."""
import json
import sys

d = json.load(open(sys.argv[1]))
ln = d["line"]
print(f"value {ln['value']} GElem/s  hbm {ln['hbm_gbs']} GB/s  ms/step {ln['ms_per_step']}  "
      f"cells_sum/step {d.get('cells_sum_over_step')}  clocks {ln.get('clocks', {}).get('sm_mhz')} "
      f"{ln.get('clocks', {}).get('reasons')}")
for c in d["cells"]:
    extra = c.get("tc_frac", c.get("fma_frac", ""))
    print(f"{c['cell']:28s} {c['avg_ms'] * 1e3:8.1f} us {c['gelem_s']:8.1f} GE/s {c['gbs']:7.0f} GB/s "
          f"frac {c['frac_hbm']:.3f} /8T {c['frac_8tbs']:.3f} {extra}")
if ln.get("cfg5"):
    c5 = ln["cfg5"]
    print("cfg5:", c5["value"], "GElem/s", c5["ms_per_step"], "ms/step", c5["hbm_gbs"], "GB/s", c5["cells"],
          c5.get("clocks", {}).get("sm_mhz"), c5.get("clocks", {}).get("reasons"))
for k in ("e2e", "cpu_baseline", "verify", "roofline"):
    if ln.get(k):
        print(k, json.dumps(ln[k])[:400])
