#!/usr/bin/env python
"""Benchmark of the sliding-window-sum hot path (arXiv 2305.16513) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload suite|cfg1..cfg5|...]
                    [--impl ours|reference] [--no-e2e] [--no-cpu-baseline] [--cells-out F]
                    [--graph | --no-graph] [--cell-timing separate|inline]

One STEP = one pass of the whole hot path over one batch of the workload's
synthetic inputs (BASELINE.json configs, seeded, generated on the device by
synth/ -- the same counter-based stream the oracle side regenerates on the
host).  Default workload "suite" = every BASELINE.json cell measured at one
GPU except the oracle-sized config 1 and the 16 GiB config 5 (run those with
--workload cfg1 / cfg5):
    cfg2: int32 N=2^26 sliding sum and max, w in {3,16,64,256}      (8 launches)
    cfg3: fp32 64 x 2^20 conv1d, k in {3,5,7,15,31,63}               (6 launches)
    cfg4: fp32 NCHW 32x64x112x112 max/avg pool 3x3 s1 and 2x2 s2     (4 launches)
Metric (BASELINE.json): output GElem/s (whole job, all ranks) plus achieved
HBM GB/s = (input bytes + output bytes) / time.

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
cuda.synchronize on both sides, timed with CUDA events on the launch stream,
max over ranks.  On one GPU the step is captured once as a CUDA graph and
replayed (--no-graph: eager launches; multi-GPU is always eager: the halo
exchange is not captured).  Per-kernel durations (-> the dominant kernel's
roofline) come from CUDA events around every launch on the same stream, in an
eager pass of K more steps right after the timed ones (--cell-timing
separate, default: an event pair between every two kernels costs ~7% of the
step), or inside the timed eager steps (--cell-timing inline).  L2: every
cell's input is larger than L2 (126 MB) or, for cfg4, each cell reads its own
copy of the input, so no cell starts with its input L2-resident.

Multi-GPU (torchrun, one rank per GPU, NCCL): cfg2 / cfg5 are sequence-
sharded with a (w_max-1)-element halo exchanged by NCCL send/recv and
overlapped with the interior kernels; cfg3 / cfg4 are batch-sharded with no
collective; cfg1 runs as replicas.  Default --scaling weak: the global problem
is the BASELINE.json shape times N (N x the rows / images / sequence length),
so every rank processes one config-sized share ("scaling":"weak");
--scaling strong keeps the BASELINE.json shape and splits it.

--impl reference: the CPU oracle (oracle/, plain C, 1 thread) timed on a
bounded sample of the same workload (rank 0 only) -- the tier's reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "output GElem/s and achieved HBM GB/s (% of ~8 TB/s) for sliding pool/conv1d"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback if MEASURED_PEAKS.json is absent
FP32_FMA_PEAK = 148 * 128 * 1.965e9  # FMA/s: SMs x FP32 lanes x max SM clock
# Tensor-core conv1d (csrc/conv_tc.cu): 33 <= k <= 64 at stride 1, dilation 1; over the K = 192
# Toeplitz depth every output costs one TF32 product (xh fh, 384 flop) and one bf16 correction
# product of depth 2K (768 flop at twice the TF32 rate): 768 TF32-equivalent flop per output
# (the 3xTF32 mode, SS_CONV_TC_MIXED=0, executes 1152).
TC_CONV_K = (33, 64)
TC_FLOP_PER_OUT = 3 * 192 * 2 if os.environ.get("SS_CONV_TC_MIXED", "1") == "0" else 2 * 192 * 2


BWD_OPS = ("conv_bwd_in", "conv_bwd_f", "sum_bwd", "max_bwd", "pool2d_bwd", "conv2d_bwd_in", "conv2d_bwd_f")


def conv_on_tensor_cores(c) -> bool:
    # forward conv, and the stride-1 input gradient (forward kernels on padded dy); dilated
    # filters whose extent (k-1)d+1 <= 64 also run on the tensor cores
    if c.op not in ("conv", "conv_bwd_in") or c.stride != 1:
        return False
    if c.dilation == 1:
        return TC_CONV_K[0] <= c.w <= TC_CONV_K[1]
    return (c.w - 1) * c.dilation + 1 <= TC_CONV_K[1]


def tf32_peak_tflops():
    """Dense TF32 peak: the measured bf16 number (MEASURED_PEAKS.json) x the nominal tf32/bf16 ratio 1/2."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]) / 2
    except Exception:  # noqa: BLE001
        return 2250.0 / 2


# ============================================================== workload cells
class Cell:
    """One kernel launch of the workload."""

    def __init__(self, cfg, name, op, *, w=None, f=None, kh=None, kw=None, sh=None, sw=None,
                 mode=None, inp=None, inp2=None, stride=1, dilation=1, pads=(0, 0), pad_mode="zeros"):
        self.cfg, self.name, self.op = cfg, name, op
        self.inp2 = inp2  # second input (affine: v), None otherwise
        self.stride, self.dilation, self.pads, self.pad_mode = stride, dilation, pads, pad_mode
        self.w, self.f, self.kh, self.kw, self.sh, self.sw, self.mode = w, f, kh, kw, sh, sw, mode
        self.f_flat = None if f is None else [float(v) for v in f.reshape(-1)]  # host taps for 2-D calls
        self.inp = inp  # key of the input tensor it reads
        self.n_out = 0
        self.bytes = 0
        self.flops = 0
        self.times = []

    def inputs(self):
        return [self.inp] + ([self.inp2] if self.inp2 else [])


def cfg_cells(workload: str):
    """(inputs spec, cells) for a workload; inputs spec: key -> dict(shape, dist, seed, kw, shard)."""
    import synth
    inputs, cells = {}, []
    if workload in ("suite", "cfg2"):
        inputs["x2"] = dict(n=1 << 26, dtype="int32", dist="int", seed=2, kw=dict(lo=-1000, hi=1000),
                            shard="seq", w_max=256)
        for w in (3, 16, 64, 256):
            for op in ("sum", "max"):
                cells.append(Cell("cfg2", f"cfg2_{op}_w{w}", op, w=w, inp="x2"))
    if workload in ("suite", "cfg3"):
        inputs["x3"] = dict(rows=64, n=1 << 20, dtype="float32", dist="normal", seed=3, kw={},
                            shard="batch")
        for k in (3, 5, 7, 15, 31, 63):
            f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
            cells.append(Cell("cfg3", f"cfg3_conv_k{k}", "conv", w=k, f=f, inp="x3"))
    if workload in ("suite", "cfg4"):
        spec = dict(images=32, C=64, H=112, W=112, dtype="float32", dist="u01", seed=5, kw={},
                    shard="image")
        for i, (mode, kk, ss_) in enumerate((("max", 3, 1), ("avg", 3, 1), ("max", 2, 2), ("avg", 2, 2))):
            key = f"x4_{i}"  # one copy per cell: no cell starts with its input in L2
            inputs[key] = dict(spec)
            cells.append(Cell("cfg4", f"cfg4_{mode}_{kk}x{kk}_s{ss_}", "pool2d", kh=kk, kw=kk, sh=ss_,
                              sw=ss_, mode=mode, inp=key))
    if workload == "cfg1":
        inputs["x1"] = dict(n=65536, dtype="float32", dist="upm1", seed=0, kw={}, shard="replica")
        cells.append(Cell("cfg1", "cfg1_sum_w8", "sum", w=8, inp="x1"))
        cells.append(Cell("cfg1", "cfg1_max_w8", "max", w=8, inp="x1"))
        cells.append(Cell("cfg1", "cfg1_conv_k8", "conv", w=8, f=synth.uniform_pm1(1, 8), inp="x1"))
    if workload == "cfg5":
        inputs["x5"] = dict(n=1 << 32, dtype="float32", dist="normal", seed=6, kw={}, shard="seq", w_max=64)
        cells.append(Cell("cfg5", "cfg5_conv_k31", "conv", w=31,
                          f=synth.normal(7, 31, sigma=synth.cfg_sigma_filter(31)), inp="x5"))
        cells.append(Cell("cfg5", "cfg5_max_w64", "max", w=64, inp="x5"))
    if workload == "stride":  # row a4 (strided 1-D windows); not a BASELINE.json config
        inputs["xs"] = dict(rows=64, n=1 << 20, dtype="float32", dist="normal", seed=3, kw={},
                            shard="batch")
        cells.append(Cell("stride", "stride_max_w3_s2", "max", w=3, stride=2, inp="xs"))
        cells.append(Cell("stride", "stride_sum_w2_s2", "sum", w=2, stride=2, inp="xs"))
        cells.append(Cell("stride", "stride_sum_w4_s4", "sum", w=4, stride=4, inp="xs"))
        cells.append(Cell("stride", "stride_conv_k7_s2", "conv", w=7, stride=2,
                          f=synth.normal(4, 7, sigma=synth.cfg_sigma_filter(7)), inp="xs"))
    if workload == "winspec":  # zero padding + dilation; not a BASELINE config
        inputs["xw"] = dict(rows=64, n=1 << 20, dtype="float32", dist="normal", seed=3, kw={},
                            shard="batch")
        for k, d, pad in ((7, 1, 3), (31, 1, 15), (7, 4, 12), (15, 8, 0)):
            cells.append(Cell("winspec", f"winspec_conv_k{k}_d{d}_p{pad}", "conv", w=k, dilation=d, pads=(pad, pad),
                              f=synth.normal(4, k, sigma=synth.cfg_sigma_filter(k)), inp="xw"))
        cells.append(Cell("winspec", "winspec_max_w3_p1", "max", w=3, pads=(1, 1), inp="xw"))
        cells.append(Cell("winspec", "winspec_sum_w8_d2", "sum", w=8, dilation=2, inp="xw"))
        # padding modes ("mirroring, or periodicity") and the sliding min (l.136)
        cells.append(Cell("winspec", "winspec_conv_k7_p3_reflect", "conv", w=7, pads=(3, 3), pad_mode="reflect",
                          f=synth.normal(4, 7, sigma=synth.cfg_sigma_filter(7)), inp="xw"))
        cells.append(Cell("winspec", "winspec_min_w16_p8_circular", "min", w=16, pads=(8, 7), pad_mode="circular",
                          inp="xw"))
    if workload == "affine":  # sliding window of gamma pairs; not a BASELINE config
        inputs["xa_u"] = dict(rows=8, n=1 << 24, dtype="float32", dist="uab", seed=31,
                              kw=dict(lo=0.5, hi=1.0), shard="batch")
        inputs["xa_v"] = dict(rows=8, n=1 << 24, dtype="float32", dist="normal", seed=32, kw={},
                              shard="batch")
        for w in (8, 64, 1024):
            cells.append(Cell("affine", f"affine_w{w}", "affine", w=w, inp="xa_u", inp2="xa_v"))
    if workload == "conv2d":  # 2-D sliding dot product on the config-4 tensor
        for i, (kk, st) in enumerate(((3, 1), (5, 1), (7, 1), (3, 2))):
            inputs[f"x2d_{i}"] = dict(images=32, C=64, H=112, W=112, dtype="float32", dist="u01", seed=5, kw={},
                                      shard="image")
            f = synth.normal(70 + kk, kk * kk, sigma=1.0 / kk).reshape(kk, kk)
            cells.append(Cell("conv2d", f"conv2d_{kk}x{kk}_s{st}", "conv2d", kh=kk, kw=kk, sh=st, sw=st, f=f,
                              inp=f"x2d_{i}"))
    if workload == "mc":  # multi-channel conv1d, channels-last bf16 (tensor cores)
        for cin, cout, k in ((64, 64, 3), (128, 128, 3), (64, 64, 9)):
            key = f"xmc{cin}"
            inputs[key] = dict(rows=16, n=65536 * cin, dtype="bfloat16", dist="normal", seed=96, kw={},
                               shard="batch")
            wf = synth.normal(97, cout * cin * k, sigma=(cin * k) ** -0.5).reshape(cout, cin, k)
            cells.append(Cell("mc", f"mc_c{cin}x{cout}_k{k}", "conv_mc", w=k, f=wf, inp=key, kh=cin, kw=cout))
    if workload == "backward":  # backward passes on config-3 / config-4 shapes; not a BJ config
        inputs["xb"] = dict(rows=64, n=1 << 20, dtype="float32", dist="normal", seed=3, kw={}, shard="batch")
        for k in (7, 31, 63):
            inputs[f"gb{k}"] = dict(rows=64, n=(1 << 20) - k + 1, dtype="float32", dist="normal", seed=33, kw={},
                                    shard="batch")
            f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
            cells.append(Cell("backward", f"bwd_conv_input_k{k}", "conv_bwd_in", w=k, f=f, inp=f"gb{k}"))
            cells.append(Cell("backward", f"bwd_conv_filter_k{k}", "conv_bwd_f", w=k, f=f, inp="xb", inp2=f"gb{k}"))
        inputs["gb16"] = dict(rows=64, n=(1 << 20) - 15, dtype="float32", dist="normal", seed=33, kw={}, shard="batch")
        cells.append(Cell("backward", "bwd_sum_w16", "sum_bwd", w=16, inp="gb16"))
        cells.append(Cell("backward", "bwd_max_w16", "max_bwd", w=16, inp="xb", inp2="gb16"))
        inputs["x4b"] = dict(images=32, C=64, H=112, W=112, dtype="float32", dist="u01", seed=5, kw={}, shard="image")
        for kk, st in ((3, 1), (2, 2)):
            oh = (112 - kk) // st + 1
            inputs[f"g4_{kk}"] = dict(images=32, C=64, H=oh, W=oh, dtype="float32", dist="normal", seed=34, kw={},
                                      shard="image")
            for mode in ("max", "avg"):
                cells.append(Cell("backward", f"bwd_pool2d_{mode}_{kk}x{kk}_s{st}", "pool2d_bwd", kh=kk, kw=kk, sh=st,
                                  sw=st, mode=mode, inp="x4b", inp2=f"g4_{kk}"))
        for kk in (3, 7):  # 2-D conv gradients (reading R21) on the config-4 planes
            oh = 112 - kk + 1
            if f"g4_{kk}" not in inputs:
                inputs[f"g4_{kk}"] = dict(images=32, C=64, H=oh, W=oh, dtype="float32", dist="normal", seed=34,
                                          kw={}, shard="image")
            f = synth.normal(70 + kk, kk * kk, sigma=1.0 / kk).reshape(kk, kk)
            cells.append(Cell("backward", f"bwd_conv2d_input_{kk}x{kk}", "conv2d_bwd_in", kh=kk, kw=kk, sh=1, sw=1,
                              f=f, inp=f"g4_{kk}", inp2="x4b"))
            cells.append(Cell("backward", f"bwd_conv2d_filter_{kk}x{kk}", "conv2d_bwd_f", kh=kk, kw=kk, sh=1, sw=1,
                              f=f, inp="x4b", inp2=f"g4_{kk}"))
    if not cells:
        raise SystemExit(f"unknown workload {workload}")
    return inputs, cells


# ============================================================== clocks (NVML)
class ClockSampler:
    """Samples SM clock and throttle reasons DURING the timed region with
    `nvidia-smi -lms 20` in a subprocess (the GPU selected by UUID, so
    CUDA_VISIBLE_DEVICES remapping is respected); falls back to NVML polling."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            import torch
            u = str(torch.cuda.get_device_properties(self.dev).uuid)
            uid = u if u.startswith("GPU-") else "GPU-" + u
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                                          "-lms", "20", "-i", uid], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the sampler start before the timed region
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons, pw = [], None, set(), []
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                pw.append(float(f[6]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": getattr(self, "err", "no nvidia-smi samples")}
        busy = [c for c, p in zip(sm, pw) if p > 200] or sm  # samples under load
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ============================================================== helpers
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_)"
        except Exception:  # noqa: BLE001
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ============================================================== our arm
def scale_inputs(inputs, factor: int):
    """Weak scaling: the global problem is `factor` x each sharded dimension
    (rows, images, sequence length); replicas are unchanged."""
    for sp in inputs.values():
        if sp.get("shard") == "batch":
            sp["rows"] *= factor
        elif sp.get("shard") == "image":
            sp["images"] *= factor
        elif sp.get("shard") == "seq":
            sp["n"] *= factor
    return inputs


class Runner:
    def __init__(self, workload, world, rank, device, weak=False):
        import torch

        import paper_2305_16513_b200 as ss
        import synth
        from paper_2305_16513_b200 import dist as ssd
        self.torch, self.ss, self.synth, self.ssd = torch, ss, synth, ssd
        self.world, self.rank, self.device = world, rank, device
        self.inputs_spec, self.cells = cfg_cells(workload)
        if weak and world > 1:
            scale_inputs(self.inputs_spec, world)
        self.stream = torch.cuda.current_stream()
        self.x = {}      # device inputs (local shard, incl. halo slots)
        self.meta = {}   # per-input sharding geometry
        self.y = {}      # device outputs per cell
        self._alloc()

    # ---- inputs / outputs
    def _alloc(self):
        torch, synth, ssd = self.torch, self.synth, self.ssd
        for key, sp in self.inputs_spec.items():
            dt = torch.int32 if sp["dtype"] == "int32" else torch.float32
            if sp["shard"] == "seq":
                sh = ssd.SeqShard(sp["n"], self.world, self.rank, sp["w_max"])
                t = torch.zeros(sh.size + sh.halo, dtype=dt, device=self.device)
                synth.fill_device(t[:sh.size], sp["dist"], sp["seed"], start=sh.start, **sp["kw"])
                self.meta[key] = ("seq", sh)
            elif sp["shard"] == "batch":
                r0, r1 = ssd.even_split(sp["rows"], self.world, self.rank)
                t = torch.empty((r1 - r0, sp["n"]), dtype=dt, device=self.device)
                synth.fill_device(t, sp["dist"], sp["seed"], start=r0 * sp["n"], **sp["kw"])
                if sp["dtype"] == "bfloat16":  # generated in fp32, rounded once (untimed)
                    t = t.to(torch.bfloat16)
                self.meta[key] = ("batch", (r1 - r0, sp["n"]))
            elif sp["shard"] == "image":
                i0, i1 = ssd.even_split(sp["images"], self.world, self.rank)
                per = sp["C"] * sp["H"] * sp["W"]
                t = torch.empty((i1 - i0, sp["C"], sp["H"], sp["W"]), dtype=dt, device=self.device)
                synth.fill_device(t, sp["dist"], sp["seed"], start=i0 * per, **sp["kw"])
                self.meta[key] = ("image", (i1 - i0, sp["C"], sp["H"], sp["W"]))
            else:  # replica
                t = torch.empty(sp["n"], dtype=dt, device=self.device)
                synth.fill_device(t, sp["dist"], sp["seed"], start=0, **sp["kw"])
                self.meta[key] = ("replica", sp["n"])
            self.x[key] = t
        for c in self.cells:
            kind, geo = self.meta[c.inp]
            x = self.x[c.inp]
            es = x.element_size()
            if c.op in BWD_OPS:
                self._alloc_bwd(c)
                continue
            if c.op == "conv_mc":
                rows, n = geo
                cin, cout, k = c.kh, c.kw, c.w
                N = n // cin
                L = N - k + 1
                self.y[c.name] = torch.empty((rows, L, cout), dtype=torch.float32, device=self.device)
                self.wmc = getattr(self, "wmc", {})
                self.wmc[c.name] = torch.from_numpy(c.f).to(self.device).to(torch.bfloat16).contiguous()
                c.n_out = rows * L * cout
                c.bytes = rows * N * cin * 2 + c.n_out * 4 + cout * cin * k * 2
                c.flops = 2 * k * cin * c.n_out
                continue
            if c.op in ("pool2d", "conv2d"):
                B, C, H, W = geo
                OH, OW = (H - c.kh) // c.sh + 1, (W - c.kw) // c.sw + 1
                self.y[c.name] = torch.empty((B, C, OH, OW), dtype=x.dtype, device=self.device)
                c.n_out = B * C * OH * OW
                c.bytes = (B * C * H * W + c.n_out) * es
            elif kind == "seq":
                sh = geo
                c.n_out = sh.n_outputs(c.w)
                self.y[c.name] = torch.empty(max(c.n_out, 1), dtype=x.dtype, device=self.device)
                c.bytes = (sh.size + c.n_out) * es
            elif kind == "batch" and c.op == "affine":  # y = [U; V]
                rows, n = geo
                L = (n - c.w) // c.stride + 1
                self.y[c.name] = torch.empty((2, rows, L), dtype=x.dtype, device=self.device)
                c.n_out = rows * L
                c.bytes = 2 * (rows * n + c.n_out) * es
            elif kind == "batch":
                rows, n = geo
                L = (n + sum(c.pads) - ((c.w - 1) * c.dilation + 1)) // c.stride + 1
                self.y[c.name] = torch.empty((rows, L), dtype=x.dtype, device=self.device)
                c.n_out = rows * L
                c.bytes = (rows * n + c.n_out) * es
            else:
                n = geo
                L = n - c.w + 1
                self.y[c.name] = torch.empty(L, dtype=x.dtype, device=self.device)
                c.n_out = L
                c.bytes = (n + L) * es
            c.flops = 2 * c.w * c.n_out if c.op == "conv" else (2 * c.kh * c.kw * c.n_out if c.op == "conv2d" else 0)

    def _alloc_bwd(self, c):
        """Backward cells: dx (or df + workspace) and the algorithmic bytes / unit counts.
        n_out = gradient elements written (dx), or for the filter gradient the
        rows x L products it reduces."""
        torch = self.torch
        x = self.x[c.inp]
        if c.op == "pool2d_bwd":
            g = self.x[c.inp2]
            self.y[c.name] = torch.empty_like(x)
            c.n_out = x.numel()
            c.bytes = 4 * (x.numel() * (2 if c.mode == "max" else 1) + g.numel())
            return
        if c.op == "conv2d_bwd_in":  # inp = dy [B, C, OH, OW], inp2 = x (shape only)
            g, xs = x, self.x[c.inp2]
            self.y[c.name] = torch.empty_like(xs)
            c.n_out = xs.numel()
            c.bytes = 4 * (g.numel() + xs.numel())
            c.flops = 2 * c.kh * c.kw * g.numel()
            return
        if c.op == "conv2d_bwd_f":  # inp = x [B, C, H, W], inp2 = dy
            g = self.x[c.inp2]
            self.y[c.name] = torch.empty((c.kh, c.kw), dtype=torch.float32, device=self.device)
            self.ws = getattr(self, "ws", {})
            self.ws[c.name] = torch.empty(self.ss.ss_conv2d_backward_filter_workspace(c.kh, c.kw), dtype=torch.uint8,
                                          device=self.device)
            c.n_out = g.numel()
            c.bytes = 4 * (x.numel() + g.numel())
            c.flops = 2 * c.kh * c.kw * g.numel()
            return
        if c.op in ("conv_bwd_in", "sum_bwd"):  # inp = dy [rows, L]
            rows, L = x.shape
            N = L + c.w - 1
            self.y[c.name] = torch.empty((rows, N), dtype=x.dtype, device=self.device)
            c.n_out = rows * N
            c.bytes = 4 * (rows * L + rows * N)
            c.flops = 2 * c.w * rows * L if c.op == "conv_bwd_in" else 0
            return
        rows, N = x.shape                          # inp = x [rows, N], inp2 = dy [rows, L]
        L = self.x[c.inp2].shape[1]
        if c.op == "max_bwd":
            self.y[c.name] = torch.empty((rows, N), dtype=x.dtype, device=self.device)
            c.n_out = rows * N
            c.bytes = 4 * (2 * rows * N + rows * L)
        else:  # conv_bwd_f
            self.y[c.name] = torch.empty(c.w, dtype=torch.float32, device=self.device)
            self.ws = getattr(self, "ws", {})
            self.ws[c.name] = torch.empty(self.ss.ss_conv1d_backward_filter_workspace(c.w), dtype=torch.uint8,
                                          device=self.device)
            c.n_out = rows * L
            c.bytes = 4 * (rows * N + rows * L + c.w)
            c.flops = 2 * c.w * rows * L

    def _launch_bwd(self, c):
        ss, st = self.ss, self.stream.cuda_stream
        x, y = self.x[c.inp], self.y[c.name]
        if c.op == "pool2d_bwd":
            B, C, H, W = x.shape
            g = self.x[c.inp2]
            ss.check(ss.ss_pool2d_backward(x.data_ptr(), g.data_ptr(), y.data_ptr(), B * C, H, W, c.kh, c.kw, c.sh,
                                           c.sw, ss.SS_POOL_MAX if c.mode == "max" else ss.SS_POOL_AVG,
                                           ss.SS_F32, st))
        elif c.op == "conv2d_bwd_in":
            B, C, H, W = y.shape
            ss.check(ss.ss_conv2d_backward_input(x.data_ptr(), y.data_ptr(), B * C, H, W, c.f_flat, c.kh, c.kw, 1, 1,
                                                 ss.SS_F32, st))
        elif c.op == "conv2d_bwd_f":
            B, C, H, W = x.shape
            ws = self.ws[c.name]
            ss.check(ss.ss_conv2d_backward_filter(x.data_ptr(), self.x[c.inp2].data_ptr(), y.data_ptr(), B * C, H, W,
                                                  c.kh, c.kw, 1, 1, ws.data_ptr(), ws.numel(), st))
        elif c.op == "conv_bwd_in":
            rows, L = x.shape
            ss.check(ss.ss_conv1d_backward_input(x.data_ptr(), y.data_ptr(), L + c.w - 1, rows, c.f, c.w, 1,
                                                 ss.SS_F32, st))
        elif c.op == "sum_bwd":
            rows, L = x.shape
            ss.check(ss.ss_pool_sum_backward(x.data_ptr(), y.data_ptr(), L + c.w - 1, rows, c.w, 1, ss.SS_F32, st))
        elif c.op == "max_bwd":
            rows, N = x.shape
            ss.check(ss.ss_pool_max_backward(x.data_ptr(), self.x[c.inp2].data_ptr(), y.data_ptr(), N, rows, c.w, 1,
                                             ss.SS_F32, st))
        else:
            rows, N = x.shape
            ws = self.ws[c.name]
            ss.check(ss.ss_conv1d_backward_filter(x.data_ptr(), self.x[c.inp2].data_ptr(), y.data_ptr(), N, rows,
                                                  c.w, 1, ws.data_ptr(), ws.numel(), st))

    # ---- one launch
    def _launch_1d(self, c, x, y):
        ss = self.ss
        s = self.stream.cuda_stream
        code = ss.SS_I32 if x.dtype == self.torch.int32 else ss.SS_F32
        if x.dim() == 1:
            N, B = x.shape[0], 1
        else:
            B, N = x.shape
        win = (c.stride, c.dilation, c.pads[0], c.pads[1], ss.PAD_MODES[c.pad_mode], code, s)
        if c.op == "affine":
            v = self.x[c.inp2]
            st = ss.ss_affine_window(x.data_ptr(), v.data_ptr(), y[0].data_ptr(), y[1].data_ptr(), N, B, c.w,
                                     c.stride, s)
        elif c.op == "conv":
            st = ss.ss_conv1d_ex(x.data_ptr(), y.data_ptr(), N, B, c.f, c.w, *win)
        elif c.op == "sum":
            st = ss.ss_pool_sum_ex(x.data_ptr(), y.data_ptr(), N, B, c.w, *win)
        elif c.op == "min":
            st = ss.ss_pool_min_ex(x.data_ptr(), y.data_ptr(), N, B, c.w, *win)
        else:
            st = ss.ss_pool_max_ex(x.data_ptr(), y.data_ptr(), N, B, c.w, *win)
        ss.check(st)

    def _launch_cell(self, c, events=None):
        kind, geo = self.meta[c.inp]
        x, y = self.x[c.inp], self.y[c.name]
        if c.op in BWD_OPS:
            ev0 = self._ev(events)
            self._launch_bwd(c)
            self._ev_end(events, c, ev0)
        elif c.op == "conv_mc":
            rows, n = geo
            ev0 = self._ev(events)
            self.ss.check(self.ss.ss_conv1d_mc(x.data_ptr(), self.wmc[c.name].data_ptr(), y.data_ptr(), rows,
                                               n // c.kh, c.kh, c.kw, c.w, self.stream.cuda_stream))
            self._ev_end(events, c, ev0)
        elif c.op == "conv2d":
            B, C, H, W = geo
            ev0 = self._ev(events)
            self.ss.check(self.ss.ss_conv2d(x.data_ptr(), y.data_ptr(), B * C, H, W, c.f.reshape(-1).tolist(), c.kh,
                                            c.kw, c.sh, c.sw, self.ss.SS_F32, self.stream.cuda_stream))
            self._ev_end(events, c, ev0)
        elif c.op == "pool2d":
            B, C, H, W = geo
            ev0 = self._ev(events)
            self.ss.check(self.ss.ss_pool2d(x.data_ptr(), y.data_ptr(), B * C, H, W, c.kh, c.kw, c.sh, c.sw,
                                            self.ss.SS_POOL_MAX if c.mode == "max" else self.ss.SS_POOL_AVG,
                                            self.ss.SS_F32, self.stream.cuda_stream))
            self._ev_end(events, c, ev0)
        elif kind == "seq":
            ev0 = self._ev(events)
            self.ssd.run_interior(x, geo, c.w, lambda xv, yv: self._launch_1d(c, xv, yv), y)
            self._ev_end(events, c, ev0)
        else:
            ev0 = self._ev(events)
            self._launch_1d(c, x, y)
            self._ev_end(events, c, ev0)

    def _ev(self, events):
        if events is None:
            return None
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def _ev_end(self, events, c, ev0):
        if events is None:
            return
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        events.append((c, ev0, e))

    def step(self, events=None, before=None, after=None):
        """One pass of the hot path over the workload (this rank's share).
        before(c)/after(c): optional hooks around each cell's launches (the
        end-to-end loop uses them to chain copies on other streams)."""
        works = {}
        for key, (kind, geo) in self.meta.items():  # post halo exchanges first
            if kind == "seq" and self.world > 1:
                works[key] = self.ssd.halo_start(self.x[key], geo)
        for c in self.cells:  # interiors / whole cells
            if before:
                before(c)
            self._launch_cell(c, events)
            if after and not (self.meta[c.inp][0] == "seq" and works):
                after(c)
        for key, wk in works.items():
            self.ssd.wait_all(wk)
        if works:
            for c in self.cells:  # tails
                kind, geo = self.meta[c.inp]
                if kind == "seq":
                    self.ssd.run_tail(self.x[c.inp], geo, c.w,
                                      lambda xv, yv, c=c: self._launch_1d(c, xv, yv), self.y[c.name])
                    if after:
                        after(c)

    # ---- end to end: pinned host buffers -> device -> kernels -> host
    def setup_e2e(self):
        """Pinned host buffers for every input and output, and the streams /
        events of the overlapped end-to-end loop."""
        torch = self.torch
        self.hx = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in self.x.items()}
        for k, v in self.x.items():
            self.hx[k].copy_(v)
        # cfg4 cells read distinct device copies in the kernel-only loop; end to end,
        # every cell gets its own H2D copy too (same bytes).
        self.hy = {c.name: torch.empty(self.y[c.name].shape, dtype=self.y[c.name].dtype, pin_memory=True)
                   for c in self.cells}
        torch.cuda.synchronize()
        self.h2d_bytes = sum(v.numel() * v.element_size() for v in self.hx.values())
        self.d2h_bytes = sum(v.numel() * v.element_size() for v in self.hy.values())
        self.s_h2d = torch.cuda.Stream(device=self.device)
        self.s_d2h = torch.cuda.Stream(device=self.device)
        ev = lambda: torch.cuda.Event()  # noqa: E731
        self.ev_in_ready = {k: ev() for k in self.x}
        self.ev_in_free = {k: ev() for k in self.x}
        self.ev_out_ready = {c.name: ev() for c in self.cells}
        self.ev_out_free = {c.name: ev() for c in self.cells}
        for e in list(self.ev_in_free.values()) + list(self.ev_out_free.values()):
            e.record(self.stream)
        self.last_reader = {k: c.name for c in self.cells for k in c.inputs()}  # last reader of each input

    def step_e2e(self):
        """One end-to-end step through the public C ABI: H2D of every input from
        pinned memory (copy stream), the kernels (compute stream), D2H of every
        output to pinned memory (second copy stream).  Copies of one cell overlap
        kernels of the next; an input is overwritten only after its last reader
        of the previous step, an output only after its previous D2H."""
        torch = self.torch
        for k in self.x:
            self.s_h2d.wait_event(self.ev_in_free[k])
            with torch.cuda.stream(self.s_h2d):
                self.x[k].copy_(self.hx[k], non_blocking=True)
            self.ev_in_ready[k].record(self.s_h2d)

        def before(c):
            for k in c.inputs():
                self.stream.wait_event(self.ev_in_ready[k])
            self.stream.wait_event(self.ev_out_free[c.name])

        def after(c):
            self.ev_out_ready[c.name].record(self.stream)
            for k in c.inputs():
                if self.last_reader[k] == c.name:
                    self.ev_in_free[k].record(self.stream)
            self.s_d2h.wait_event(self.ev_out_ready[c.name])
            with torch.cuda.stream(self.s_d2h):
                self.hy[c.name].copy_(self.y[c.name], non_blocking=True)
            self.ev_out_free[c.name].record(self.s_d2h)

        self.step(before=before, after=after)

    def e2e_fence(self):
        """Make the compute stream wait for every outstanding copy."""
        done = self.torch.cuda.Event()
        done.record(self.s_d2h)
        self.stream.wait_event(done)
        done2 = self.torch.cuda.Event()
        done2.record(self.s_h2d)
        self.stream.wait_event(done2)


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local % torch.cuda.device_count())
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # test mode: several ranks may share a GPU; host-staged halo
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    device = torch.device("cuda", torch.cuda.current_device())
    import paper_2305_16513_b200 as ss
    weak = args.scaling == "weak"
    if args.graph is None:  # default: replay the step as a CUDA graph on one GPU (halo exchange is not captured)
        args.graph = world == 1
    if args.graph:  # graphs are captured on a non-default stream: run everything there
        torch.cuda.set_stream(torch.cuda.Stream())
    R = Runner(args.workload, world, rank, device, weak=weak)
    torch.cuda.synchronize()

    coll_dev = device if args.dist_backend == "nccl" else torch.device("cpu")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            if args.dist_backend == "nccl":
                dist.barrier(device_ids=[torch.cuda.current_device()])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        R.step()
    barrier()
    events = []
    graph = None
    if args.graph:
        # capture one step in a CUDA graph and replay it (no host launch gaps between kernels);
        # per-kernel durations come from one eager pass with events (below)
        if world > 1:
            raise SystemExit("--graph is single-GPU only (the halo exchange is not captured)")
        n_cap0 = ss.ss_launch_count()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=R.stream):
            R.step()
        launches_per_step = ss.ss_launch_count() - n_cap0
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
    n_launch0 = ss.ss_launch_count()
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        barrier()
        t0.record(R.stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                R.step(events if args.cell_timing == "inline" else None)
        t1.record(R.stream)
        torch.cuda.synchronize()
        barrier()
    launches = ss.ss_launch_count() - n_launch0
    if graph is not None:
        launches = launches_per_step * args.steps
    if graph is not None or args.cell_timing == "separate":
        for _ in range(args.steps):  # instrumented eager pass: the per-kernel event durations
            R.step(events)
        torch.cuda.synchronize()
    ms_local = t0.elapsed_time(t1)
    ms = max_over_ranks(ms_local)
    for c, a, b in events:
        c.times.append(a.elapsed_time(b))
    out_local = sum(c.n_out for c in R.cells) * args.steps
    bytes_local = sum(c.bytes for c in R.cells) * args.steps
    tot = torch.tensor([out_local, bytes_local], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(tot)
    out_total, bytes_total = float(tot[0]), float(tot[1])
    value = out_total / (ms * 1e-3) / 1e9
    hbm_gbs = bytes_total / (ms * 1e-3) / 1e9

    # per-kernel (cell) stats and the dominant kernel
    peak_hbm, peak_src = measured_peaks()
    cells = []
    for c in R.cells:
        avg_ms = sum(c.times) / len(c.times)
        gbs = c.bytes / (avg_ms * 1e-3) / 1e9
        d = {"cell": c.name, "avg_ms": round(avg_ms, 5), "n_out": c.n_out, "bytes": c.bytes,
             "gelem_s": round(c.n_out / (avg_ms * 1e-3) / 1e9, 2), "gbs": round(gbs, 1),
             "frac_hbm": round(gbs / peak_hbm, 4), "frac_8tbs": round(gbs / 8000.0, 4),
             "share": 0.0}
        if c.op == "conv_mc":
            d["tc_frac"] = round(c.flops / (avg_ms * 1e-3) / 1e12 / (2 * tf32_peak_tflops()), 4)  # bf16 peak
        elif conv_on_tensor_cores(c):
            d["tc_frac"] = round(c.n_out * TC_FLOP_PER_OUT / (avg_ms * 1e-3) / 1e12 / tf32_peak_tflops(), 4)
        elif c.op in ("conv", "conv_bwd_in", "conv_bwd_f", "conv2d", "conv2d_bwd_in", "conv2d_bwd_f"):
            fma_s = c.flops / 2 / (avg_ms * 1e-3)
            d["fma_frac"] = round(fma_s / FP32_FMA_PEAK, 4)
        cells.append(d)
    tot_k = sum(d["avg_ms"] for d in cells)
    for d in cells:
        d["share"] = round(d["avg_ms"] / tot_k, 4)
    dom = max(cells, key=lambda d: d["avg_ms"])
    dom_cell = next(c for c in R.cells if c.name == dom["cell"])
    if dom_cell.op in ("conv", "conv_bwd_in", "conv_bwd_f", "conv2d", "conv2d_bwd_in", "conv2d_bwd_f") and dom.get("fma_frac", 0) > dom["frac_hbm"]:
        achieved = dom_cell.flops / (dom["avg_ms"] * 1e-3) / 1e12
        roofline = {"bound": "alu", "kernel": dom["cell"], "achieved": round(achieved, 2),
                    "peak": round(2 * FP32_FMA_PEAK / 1e12, 2), "unit": "TFLOP/s",
                    "frac": round(achieved / (2 * FP32_FMA_PEAK / 1e12), 4),
                    "peak_source": "148 SM x 128 FP32 FMA/clk x 1965 MHz (DESIGN.md)",
                    "hbm_gbs": dom["gbs"], "hbm_frac": dom["frac_hbm"], "traffic": None}
    else:
        roofline = {"bound": "hbm", "kernel": dom["cell"], "achieved": dom["gbs"], "peak": peak_hbm,
                    "unit": "GB/s", "frac": dom["frac_hbm"], "peak_source": peak_src, "traffic": None}
        if "tc_frac" in dom and dom_cell.op == "conv_mc":
            roofline["tensor_frac"] = dom["tc_frac"]
            roofline["tensor_peak_tflops"] = round(2 * tf32_peak_tflops(), 1)
            roofline["tensor_note"] = "bf16 MMA work (2 k Cin flop/output) / measured dense bf16 peak"
        elif "tc_frac" in dom:  # tensor-core conv: HBM is the roofline (its TC ceiling is higher)
            roofline["tensor_frac"] = dom["tc_frac"]
            roofline["tensor_peak_tflops"] = round(tf32_peak_tflops(), 1)
            roofline["tensor_note"] = (f"executed MMA work ({TC_FLOP_PER_OUT} TF32-equivalent flop/output: "
                                       "xh*fh in TF32 + one bf16 correction product at half weight) / dense "
                                       "TF32 peak (measured bf16 / 2)")
    roofline["share_of_step"] = dom["share"]
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):  # dram bytes per launch from a committed `ncu --set full` capture
        try:
            roofline["traffic"] = json.load(open(tf)).get(dom["cell"])
        except Exception:  # noqa: BLE001
            pass

    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        R.setup_e2e()
        for _ in range(2):
            R.step_e2e()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        n_e2e = max(2, min(args.steps, args.e2e_steps))
        R.e2e_fence()
        e0.record(R.stream)
        R.s_h2d.wait_stream(R.stream)
        for _ in range(n_e2e):
            R.step_e2e()
        R.e2e_fence()
        e1.record(R.stream)
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": round(out_total / args.steps * n_e2e / (ems * 1e-3) / 1e9, 3), "unit": "GElem/s",
               "h2d_bytes_per_step": int(R.h2d_bytes), "d2h_bytes_per_step": int(R.d2h_bytes),
               "ms_per_step": round(ems / n_e2e, 3), "steps": n_e2e,
               "path": "pinned host -> cudaMemcpyAsync (copy stream) -> ss_* C ABI (compute stream) -> "
                       "cudaMemcpyAsync (2nd copy stream) -> pinned host, overlapped across cells"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.workload, budget_s=args.cpu_budget)

    if rank == 0:
        cfg = {"workload": args.workload, "cells": [c.name for c in R.cells], "cuda_graph": bool(args.graph),
               "cell_timing": ("per-launch CUDA events in the timed steps" if args.cell_timing == "inline" and not
                               args.graph else "per-launch CUDA events in an eager pass of the same steps right "
                               "after the timed ones (the timed steps carry no per-launch events)"),
               "parallelism": f"{'seq+batch' if args.workload == 'suite' else 'shard'} x{world}",
               "l2": "inputs > L2 (126 MB) per cell; cfg4 cells read distinct input copies",
               "inputs": {k: {kk: vv for kk, vv in v.items() if kk != "kw"} for k, v in R.inputs_spec.items()}}
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GElem/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
                "higher_is_better": True, "scaling": args.scaling,
                "vs_baseline": None, "dtype": "f32/i32" if args.workload == "suite" else
                ("i32" if args.workload == "cfg2" else "f32"),
                "data": "synthetic (splitmix64 counter-based, BASELINE.json seeds/distributions)",
                "config": cfg, "hbm_gbs": round(hbm_gbs, 1), "hbm_frac_8tbs": round(hbm_gbs / 8000.0, 4),
                "hbm_frac_measured": round(hbm_gbs / peak_hbm, 4),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk.summary(), "impl": "ours"}
        print(json.dumps(line), flush=True)
        if args.cells_out:
            with open(args.cells_out, "w") as fh:
                json.dump({"line": line, "cells": cells}, fh, indent=1)
        else:
            print(json.dumps({"cells": cells}), file=sys.stderr)
    if world > 1:
        dist.destroy_process_group()


# ============================================================== oracle arm
def oracle_sample_plan(workload: str, frac: float):
    """Bounded sample of every cell: the same cells, a `frac` share of each
    (leading rows / images / output range).  Returns [(cell, fn)] where fn()
    runs the oracle on its sample and returns the number of outputs."""
    import oracle
    import synth
    _, cells = cfg_cells(workload)
    plan = []
    for c in cells:
        if c.cfg == "cfg2" or c.cfg == "cfg1" or c.cfg == "cfg5":
            n_total = {"cfg2": 1 << 26, "cfg1": 65536, "cfg5": 1 << 32}[c.cfg]
            n_out = max(1, int((n_total - c.w + 1) * frac))
            if c.cfg == "cfg2":
                x = synth.randint(2, n_out + c.w - 1, -1000, 1000)
            elif c.cfg == "cfg1":
                x = synth.uniform_pm1(0, n_out + c.w - 1)
            else:
                x = synth.normal(6, n_out + c.w - 1)
            if c.op == "sum":
                plan.append((c, lambda x=x, c=c: (oracle.pool_sum(x, c.w), x.size - c.w + 1)[1]))
            elif c.op == "max":
                plan.append((c, lambda x=x, c=c: (oracle.pool_max(x, c.w), x.size - c.w + 1)[1]))
            else:
                plan.append((c, lambda x=x, c=c: (oracle.conv1d(x, c.f), x.size - c.w + 1)[1]))
        elif c.cfg == "cfg3":
            rows = max(1, int(round(64 * frac)))
            n = 1 << 20
            if rows * n > 64 * n * frac * 1.5:  # frac below one row: shorten the row instead
                n = max(c.w, int(64 * (1 << 20) * frac))
                rows = 1
            x = synth.normal(3, rows * n).reshape(rows, n)
            plan.append((c, lambda x=x, c=c: (oracle.conv1d(x, c.f), x.shape[0] * (x.shape[1] - c.w + 1))[1]))
        elif c.cfg == "mc":
            cin, cout, k = c.kh, c.kw, c.w
            n = max(k + 1, int(16 * 65536 * frac))
            xb = oracle.to_bf16_bits(synth.normal(96, n * cin).reshape(1, n, cin))
            wb = oracle.to_bf16_bits(c.f)
            plan.append((c, lambda xb=xb, wb=wb, c=c, n=n: (oracle.conv1d_mc(xb, wb), (n - c.w + 1) * c.kw)[1]))
        elif c.cfg == "conv2d":
            planes = max(1, int(round(32 * 64 * frac)))
            x = synth.uniform01(5, planes * 112 * 112).reshape(planes, 112, 112)
            oh = (112 - c.kh) // c.sh + 1
            plan.append((c, lambda x=x, c=c, oh=oh: (oracle.conv2d(x, c.f, c.sh, c.sw), x.shape[0] * oh * oh)[1]))
        elif c.cfg == "backward" and c.op == "pool2d_bwd":
            planes = max(1, int(round(32 * 64 * frac)))
            oh = (112 - c.kh) // c.sh + 1
            x = synth.uniform01(5, planes * 112 * 112).reshape(planes, 112, 112)
            g = synth.normal(34, planes * oh * oh).reshape(planes, oh, oh)
            m = oracle.POOL2D_MAX if c.mode == "max" else oracle.POOL2D_AVG
            plan.append((c, lambda x=x, g=g, c=c, m=m: (oracle.pool2d_backward(x, g, 112, 112, c.kh, c.kw, c.sh,
                                                                               c.sw, m), x.size)[1]))
        elif c.cfg == "backward" and c.op in ("conv2d_bwd_in", "conv2d_bwd_f"):
            planes = max(1, int(round(32 * 64 * frac)))
            oh = 112 - c.kh + 1
            x = synth.uniform01(5, planes * 112 * 112).reshape(planes, 112, 112)
            g = synth.normal(34, planes * oh * oh).reshape(planes, oh, oh)
            if c.op == "conv2d_bwd_in":
                fn = (lambda g=g, c=c: (oracle.conv2d_backward_input(g, c.f, 112, 112), planes * 112 * 112)[1])
            else:
                fn = (lambda x=x, g=g, c=c: (oracle.conv2d_backward_filter(x, g, c.kh, c.kw), g.size)[1])
            plan.append((c, fn))
        elif c.cfg == "backward":
            rows = max(1, int(round(64 * frac)))
            n = 1 << 20
            if rows * n > 64 * n * frac * 1.5:  # frac below one row: shorten the row instead
                n = max(c.w + 1, int(64 * (1 << 20) * frac))
                rows = 1
            L = n - c.w + 1
            x = synth.normal(3, rows * n).reshape(rows, n)
            g = synth.normal(33, rows * L).reshape(rows, L)
            if c.op == "conv_bwd_in":
                fn = (lambda g=g, c=c, n=n: (oracle.conv1d_backward_input(g, c.f, n), g.shape[0] * n)[1])
            elif c.op == "conv_bwd_f":
                fn = (lambda x=x, g=g, c=c: (oracle.conv1d_backward_filter(x, g, c.w), g.size)[1])
            elif c.op == "sum_bwd":
                fn = (lambda g=g, c=c, n=n: (oracle.pool_sum_backward(g, n, c.w), g.shape[0] * n)[1])
            else:
                fn = (lambda x=x, g=g, c=c: (oracle.pool_max_backward(x, g, c.w), x.size)[1])
            plan.append((c, fn))
        elif c.cfg in ("stride", "winspec"):
            rows, n = 1, max(4 * (c.w - 1) * c.dilation + 8, int(64 * (1 << 20) * frac))
            x = synth.normal(3, rows * n).reshape(rows, n)
            kw = dict(s=c.stride, d=c.dilation, pl=c.pads[0], pr=c.pads[1], mode=c.pad_mode)
            L = oracle.out_len_ex(n, c.w, c.stride, c.dilation, c.pads[0], c.pads[1])
            fn = {"sum": lambda x=x, c=c, kw=kw: oracle.pool_sum_ex(x, c.w, **kw),
                  "max": lambda x=x, c=c, kw=kw: oracle.pool_max_ex(x, c.w, **kw),
                  "min": lambda x=x, c=c, kw=kw: oracle.pool_min_ex(x, c.w, **kw),
                  "conv": lambda x=x, c=c, kw=kw: oracle.conv1d_ex(x, c.f, **kw)}[c.op]
            plan.append((c, lambda fn=fn, L=L: (fn(), L)[1]))
        elif c.cfg == "affine":
            n = max(c.w, int(8 * (1 << 24) * frac))
            u = synth.uab(31, n, 0.5, 1.0)
            v = synth.normal(32, n)
            plan.append((c, lambda u=u, v=v, c=c: (oracle.affine_window(u, v, c.w), u.size - c.w + 1)[1]))
        else:  # cfg4
            planes = max(1, int(round(32 * 64 * frac)))
            x = synth.uniform01(5, planes * 112 * 112).reshape(planes, 112, 112)
            m = oracle.POOL2D_MAX if c.mode == "max" else oracle.POOL2D_AVG
            oh = (112 - c.kh) // c.sh + 1
            plan.append((c, lambda x=x, c=c, m=m, oh=oh: (oracle.pool2d(x, c.kh, c.kw, c.sh, c.sw, m),
                                                          x.shape[0] * oh * oh)[1]))
    return plan


def cpu_baseline(workload: str, budget_s: float = 20.0):
    """Time the oracle (as it stands, 1 thread) on a bounded sample of the workload."""
    # calibrate: a tiny fraction first, then scale the fraction to the budget
    frac = 1.0 / 4096 if workload != "cfg1" else 1.0
    plan = oracle_sample_plan(workload, frac)
    t0 = time.perf_counter()
    outs = sum(fn() for _, fn in plan)
    dt = time.perf_counter() - t0
    if workload != "cfg1" and dt > 0:
        frac = min(1.0, frac * max(1.0, budget_s / dt))
        plan = oracle_sample_plan(workload, frac)
        t0 = time.perf_counter()
        outs = sum(fn() for _, fn in plan)
        dt = time.perf_counter() - t0
    return {"value": round(outs / dt / 1e9, 6), "unit": "GElem/s", "cores": 1, "kind": "oracle",
            "sample": f"every cell of workload '{workload}', leading {frac:.3%} of its outputs/rows/images "
                      f"({outs} outputs, {dt:.1f} s, single-threaded C oracle -O2)",
            "seconds": round(dt, 2)}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference; the others exit 0 without work
    import oracle
    oracle.build()
    frac = 1.0 / 2048 if args.workload != "cfg1" else 1.0
    plan = oracle_sample_plan(args.workload, frac)
    for _ in range(args.warmup):
        for _, fn in plan:
            fn()
    times = []
    outs = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        outs = sum(fn() for _, fn in plan)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = outs * args.steps / tot / 1e9
    line = {"metric": METRIC, "value": round(value, 6), "unit": "GElem/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64/i64 accumulate", "data": "synthetic (same generator and seeds)",
            "config": {"workload": args.workload, "sample_fraction": frac},
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 6), "unit": "GElem/s", "cores": 1, "kind": "oracle",
                             "sample": f"leading {frac:.4%} of every cell of '{args.workload}' per step"},
            "e2e": {"value": round(value, 6), "unit": "GElem/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="suite", choices=["suite", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "stride", "winspec", "affine", "backward", "conv2d", "mc"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="multi-GPU: weak = N x the BASELINE shape (config-sized share per rank), strong = split it")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", dest="graph", action="store_true", default=None,
                    help="replay each timed step as a captured CUDA graph (default on 1 GPU)")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="launch every timed step eagerly")
    ap.add_argument("--cell-timing", choices=("inline", "separate"), default="separate",
                    help="per-kernel CUDA events inside the timed steps (inline) or in a second pass of the "
                         "same steps right after them (separate: the timed steps carry no events)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cells-out", default=None)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo = test mode (ranks may share one GPU, host-staged halo)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
