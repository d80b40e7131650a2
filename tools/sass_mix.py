"""Opcode histogram of one kernel's SASS: python tools/sass_mix.py lib.so <name-regex>"""
import re
import subprocess
import sys
from collections import Counter

out = subprocess.check_output(["cuobjdump", "-sass", sys.argv[1]], stderr=subprocess.DEVNULL).decode()
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if not re.search(sys.argv[2], name):
        continue
    c = Counter()
    n = 0
    for line in f.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
        if not m:
            continue
        ins = m.group(1).strip()
        if ins.startswith("@"):
            ins = ins.split(None, 1)[1]
        op = ins.split()[0].split(".")[0]
        c[op] += 1
        n += 1
    print(name[:90], "total", n)
    print("  ", ", ".join(f"{k}:{v}" for k, v in c.most_common(22)))
