"""Sustained tensor-core conv (config 3, k = 63) for ~3 s while nvidia-smi samples the SM clock."""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2305_16513_b200 as ss  # noqa: E402
import synth  # noqa: E402

x = torch.empty(64, 1 << 20, device="cuda")
synth.fill_device(x, "normal", 3)
k = int(os.environ.get("K", "63"))
f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
y = torch.empty(64, (1 << 20) - k + 1, device="cuda")
for _ in range(5):
    ss.conv1d(x, f, out=y)
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                        "--format=csv,noheader", "-lms", "50"], stdout=subprocess.PIPE, text=True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
a.record()
n = 0
while time.time() - t0 < 3.0:
    for _ in range(50):
        ss.conv1d(x, f, out=y)
    n += 50
    torch.cuda.synchronize()
b.record()
torch.cuda.synchronize()
smi.terminate()
out = smi.communicate()[0].strip().splitlines()
print(f"k={k}: {a.elapsed_time(b) / n * 1e3:.1f} us/call over {n} calls")
print("smi samples (clock, power, reasons):", out[len(out) // 2 - 3: len(out) // 2 + 3])
