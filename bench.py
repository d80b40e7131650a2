#!/usr/bin/env python
"""Benchmark of the sliding-window-sum hot path (arXiv 2305.16513) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload suite|cfg1..cfg5|...]
                    [--impl ours|reference] [--no-e2e] [--no-cpu-baseline] [--no-cfg5]
                    [--verify] [--cells-out F] [--dist-backend nccl|gloo]

One STEP = one pass of the whole hot path over one batch of the workload's
synthetic inputs (BASELINE.json configs, seeded, generated on the device by
synth/ -- the same counter-based stream the oracle side regenerates on the
host).  Default workload "suite" = BASELINE.json configs 2-4 (config 1 is the
oracle-sized case: --workload cfg1):
    cfg2: int32 N=2^26 sliding sum and max, w in {3,16,64,256}      (8 launches)
    cfg3: fp32 64 x 2^20 conv1d, k in {3,5,7,15,31,63}               (6 launches)
    cfg4: fp32 NCHW 32x64x112x112 max/avg pool 3x3 s1 and 2x2 s2     (4 launches)
plus, as a sub-record ("cfg5" in the JSON line), config 5: one fp32 sequence
of 2^32 elements, conv k=31 + max w=64, split over the N ranks (strong).
Metric (BASELINE.json): output GElem/s (whole job, all ranks) plus achieved
HBM GB/s = (input bytes + output bytes) / time.

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
cuda.synchronize on both sides, timed with CUDA events on the launch stream,
max over ranks.  At every N the kernels of a step are two captured CUDA graphs:
A = every interior (all of a batch-sharded cell), B = the sequence-shard tails;
the NCCL halo is posted eagerly before A and waited before B.  Per-kernel
durations (-> the dominant kernel's roofline) time each cell alone as a graph
of --cell-reps launches alternating over two input/output buffer sets (no
launch starts with its input in L2, every launch pays its own write-back);
their sum is reported against the step time.  L2: every cell's input is larger
than L2 (126 MB) or, for cfg4, each cell reads its own copy of the input.

Multi-GPU (one process per GPU, NCCL): `--gpus N` without WORLD_SIZE re-runs
this command under torch.distributed.run with N ranks (rank 0 prints the
line).  cfg2 / cfg5 are sequence-sharded with a (w_max-1)-element halo
exchanged by NCCL send/recv and overlapped with the interior kernels; cfg3 /
cfg4 are batch-sharded with no collective; cfg1 runs as replicas.  Default
--scaling weak: the global problem is the BASELINE.json shape times N, so every
rank processes one config-sized share ("scaling":"weak"); the cfg5 sub-record
is always strong.  --verify compares every rank's outputs with one unsharded
call on the regenerated global slice, bit for bit.

--impl reference: the CPU oracle (oracle/, plain C, as it stands) timed on a
bounded sample of the same workload on every host core (rank 0 only) -- the
tier's reference arm.
"""
from __future__ import annotations

import argparse
import copy
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


def cfg_cells(workload: str, cfg5_log2n: int = 32):
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
        inputs["x5"] = dict(n=1 << cfg5_log2n, dtype="float32", dist="normal", seed=6, kw={}, shard="seq", w_max=64)
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
        # its input gradient (reading R23): dy [16][65536-k+1][cout] bf16 -> dx [16][65536][cin] fp32
        for cin, cout, k in ((64, 64, 3), (128, 128, 3)):
            key = f"gmc{cout}_k{k}"
            inputs[key] = dict(rows=16, n=(65536 - k + 1) * cout, dtype="bfloat16", dist="normal", seed=98, kw={},
                               shard="batch")
            wf = synth.normal(97, cout * cin * k, sigma=(cin * k) ** -0.5).reshape(cout, cin, k)
            cells.append(Cell("mc", f"mc_dx_c{cin}x{cout}_k{k}", "conv_mc_bwd_in", w=k, f=wf, inp=key, kh=cin,
                              kw=cout))
        # its filter gradient (reading R25): dy [16][65536-k+1][cout] and x [16][65536][cin] -> dw
        for cin, cout, k in ((64, 64, 3), (64, 128, 2)):
            key = f"gmcf{cout}_k{k}"
            inputs[key] = dict(rows=16, n=(65536 - k + 1) * cout, dtype="bfloat16", dist="normal", seed=99, kw={},
                               shard="batch")
            cells.append(Cell("mc", f"mc_dw_c{cin}x{cout}_k{k}", "conv_mc_bwd_f", w=k, inp=key, inp2=f"xmc{cin}",
                              kh=cin, kw=cout))
        # multi-channel 2-D convolution (reading R22), NHWC bf16, ResNet-like layers; the image
        # shard's (C, H, W) slots hold (H, W, Cin) of the NHWC tensor
        for hw, cin, cout in ((56, 64, 64), (56, 64, 128)):
            key = f"x2mc{hw}"
            inputs[key] = dict(images=128, C=hw, H=hw, W=cin, dtype="bfloat16", dist="normal", seed=102, kw={},
                               shard="image")
            wf = synth.normal(103, cout * cin * 9, sigma=(cin * 9) ** -0.5).reshape(cout, cin, 3, 3)
            cells.append(Cell("mc", f"mc2d_{hw}x{hw}_c{cin}x{cout}_3x3", "conv2d_mc", kh=3, kw=3, f=wf, inp=key))
        # its input gradient (reading R26): dy [128][54][54][64] bf16 -> dx [128][56][56][64] fp32
        inputs["g2mc56"] = dict(images=128, C=54, H=54, W=64, dtype="bfloat16", dist="normal", seed=104, kw={},
                                shard="image")
        wf = synth.normal(103, 64 * 64 * 9, sigma=(64 * 9) ** -0.5).reshape(64, 64, 3, 3)
        cells.append(Cell("mc", "mc2d_dx_56x56_c64x64_3x3", "conv2d_mc_bwd_in", kh=3, kw=3, f=wf, inp="g2mc56"))
        # and its filter gradient (reading R27): dy [128][54][54][64] and x [128][56][56][64] -> dw [64][64][3][3]
        cells.append(Cell("mc", "mc2d_dw_56x56_c64x64_3x3", "conv2d_mc_bwd_f", kh=3, kw=3, inp="g2mc56",
                          inp2="x2mc56"))
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
    """One rank's share of a workload: inputs (nsets independent copies of every
    input and output, so a cell can be timed over distinct buffers), the launch
    of every cell through the public C ABI, and the multi-GPU halo plumbing."""

    def __init__(self, workload, world, rank, device, weak=False, nsets=1, cfg5_log2n=32):
        import torch

        import paper_2305_16513_b200 as ss
        import synth
        from paper_2305_16513_b200 import dist as ssd
        self.torch, self.ss, self.synth, self.ssd = torch, ss, synth, ssd
        self.world, self.rank, self.device = world, rank, device
        self.inputs_spec, self.cells = cfg_cells(workload, cfg5_log2n)
        if weak and world > 1:
            scale_inputs(self.inputs_spec, world)
        self.stream = torch.cuda.current_stream()
        self.meta = {}   # per-input sharding geometry
        self.xs = []     # [set] -> {key: device input (local shard, incl. halo slots)}
        self.ys = []     # [set] -> {cell name: device output}
        self.ws = {}     # workspaces (shared by the sets: launches on one stream are ordered)
        self.wmc = {}    # multi-channel conv weights
        for _ in range(nsets):
            self._alloc_set()

    @property
    def x(self):
        return self.xs[0]

    @property
    def y(self):
        return self.ys[0]

    # ---- inputs / outputs
    def _gen(self, sp, start, shape, dt):
        t = self.torch.empty(shape, dtype=self.torch.float32 if sp["dtype"] == "bfloat16" else dt,
                             device=self.device)
        self.synth.fill_device(t, sp["dist"], sp["seed"], start=start, **sp["kw"])
        if sp["dtype"] == "bfloat16":  # generated in fp32, rounded once (untimed)
            t = t.to(self.torch.bfloat16)
        return t

    def _alloc_set(self):
        torch, ssd = self.torch, self.ssd
        xd, yd = {}, {}
        for key, sp in self.inputs_spec.items():
            dt = torch.int32 if sp["dtype"] == "int32" else torch.float32
            if sp["shard"] == "seq":
                sh = ssd.SeqShard(sp["n"], self.world, self.rank, sp["w_max"])
                t = torch.zeros(sh.size + sh.halo, dtype=dt, device=self.device)
                self.synth.fill_device(t[:sh.size], sp["dist"], sp["seed"], start=sh.start, **sp["kw"])
                self.meta[key] = ("seq", sh)
            elif sp["shard"] == "batch":
                r0, r1 = ssd.even_split(sp["rows"], self.world, self.rank)
                t = self._gen(sp, r0 * sp["n"], (r1 - r0, sp["n"]), dt)
                self.meta[key] = ("batch", (r1 - r0, sp["n"]))
            elif sp["shard"] == "image":
                i0, i1 = ssd.even_split(sp["images"], self.world, self.rank)
                t = self._gen(sp, i0 * sp["C"] * sp["H"] * sp["W"], (i1 - i0, sp["C"], sp["H"], sp["W"]), dt)
                self.meta[key] = ("image", (i1 - i0, sp["C"], sp["H"], sp["W"]))
            else:  # replica
                t = self._gen(sp, 0, (sp["n"],), dt)
                self.meta[key] = ("replica", sp["n"])
            xd[key] = t
        for c in self.cells:
            yd[c.name] = self._alloc_out(c, xd)
        self.xs.append(xd)
        self.ys.append(yd)

    def _alloc_out(self, c, xd):
        """Output of cell c (and, on the first set, its unit counts / algorithmic bytes)."""
        torch = self.torch
        kind, geo = self.meta[c.inp]
        x = xd[c.inp]
        es = x.element_size()
        if c.op in BWD_OPS:
            return self._alloc_bwd(c, xd)
        if c.op == "conv_mc":
            rows, n = geo
            cin, cout, k = c.kh, c.kw, c.w
            N = n // cin
            L = N - k + 1
            if c.name not in self.wmc:
                self.wmc[c.name] = torch.from_numpy(c.f).to(self.device).to(torch.bfloat16).contiguous()
            c.n_out = rows * L * cout
            c.bytes = rows * N * cin * 2 + c.n_out * 4 + cout * cin * k * 2
            c.flops = 2 * k * cin * c.n_out
            return torch.empty((rows, L, cout), dtype=torch.float32, device=self.device)
        if c.op == "conv_mc_bwd_f":
            rows, n = geo
            cin, cout, k = c.kh, c.kw, c.w
            L = n // cout
            N = L + k - 1
            need = self.ss.ss_conv1d_mc_backward_filter_workspace(cin, cout, k)
            if c.name not in self.ws:
                self.ws[c.name] = torch.empty(max(need, 8), dtype=torch.uint8, device=self.device)
            c.n_out = rows * L * cout  # dy elements consumed (one window position each)
            c.bytes = rows * L * cout * 2 + rows * N * cin * 2 + cout * cin * k * 4
            c.flops = 2 * k * cin * cout * rows * L
            return torch.empty((cout, cin, k), dtype=torch.float32, device=self.device)
        if c.op == "conv_mc_bwd_in":
            rows, n = geo
            cin, cout, k = c.kh, c.kw, c.w
            L = n // cout
            N = L + k - 1
            if c.name not in self.wmc:
                self.wmc[c.name] = torch.from_numpy(c.f).to(self.device).to(torch.bfloat16).contiguous()
            c.n_out = rows * N * cin
            c.bytes = rows * L * cout * 2 + c.n_out * 4 + cout * cin * k * 2
            c.flops = 2 * k * cout * c.n_out
            return torch.empty((rows, N, cin), dtype=torch.float32, device=self.device)
        if c.op == "conv2d_mc_bwd_f":
            B, OH, OW, cout = geo
            H, W = OH + c.kh - 1, OW + c.kw - 1
            cin = 64
            need = self.ss.ss_conv2d_mc_backward_filter_workspace(cin, cout, c.kh, c.kw)
            if c.name not in self.ws:
                self.ws[c.name] = torch.empty(max(need, 8), dtype=torch.uint8, device=self.device)
            c.n_out = B * OH * OW * cout  # dy elements consumed
            c.bytes = B * OH * OW * cout * 2 + B * H * W * cin * 2 + cout * cin * c.kh * c.kw * 4
            c.flops = 2 * c.kh * c.kw * cin * cout * B * OH * OW
            return torch.empty((cout, cin, c.kh, c.kw), dtype=torch.float32, device=self.device)
        if c.op == "conv2d_mc_bwd_in":
            B, OH, OW, cout = geo
            cin = c.f.shape[1]
            H, W = OH + c.kh - 1, OW + c.kw - 1
            if c.name not in self.wmc:
                self.wmc[c.name] = torch.from_numpy(c.f).to(self.device).to(torch.bfloat16).contiguous()
            c.n_out = B * H * W * cin
            c.bytes = B * OH * OW * cout * 2 + c.n_out * 4 + cout * cin * c.kh * c.kw * 2
            c.flops = 2 * c.kh * c.kw * cout * c.n_out
            return torch.empty((B, H, W, cin), dtype=torch.float32, device=self.device)
        if c.op == "conv2d_mc":
            B, H, W, cin = geo
            cout = c.f.shape[0]
            OH, OW = H - c.kh + 1, W - c.kw + 1
            if c.name not in self.wmc:
                self.wmc[c.name] = torch.from_numpy(c.f).to(self.device).to(torch.bfloat16).contiguous()
            c.n_out = B * OH * OW * cout
            c.bytes = B * H * W * cin * 2 + c.n_out * 4 + cout * cin * c.kh * c.kw * 2
            c.flops = 2 * c.kh * c.kw * cin * c.n_out
            return torch.empty((B, OH, OW, cout), dtype=torch.float32, device=self.device)
        if c.op in ("pool2d", "conv2d"):
            B, C, H, W = geo
            OH, OW = (H - c.kh) // c.sh + 1, (W - c.kw) // c.sw + 1
            y = torch.empty((B, C, OH, OW), dtype=x.dtype, device=self.device)
            c.n_out = B * C * OH * OW
            c.bytes = (B * C * H * W + c.n_out) * es
        elif kind == "seq":
            sh = geo
            c.n_out = sh.n_outputs(c.w)
            y = torch.empty(max(c.n_out, 1), dtype=x.dtype, device=self.device)
            c.bytes = (sh.size + c.n_out) * es
        elif kind == "batch" and c.op == "affine":  # y = [U; V]
            rows, n = geo
            L = (n - c.w) // c.stride + 1
            y = torch.empty((2, rows, L), dtype=x.dtype, device=self.device)
            c.n_out = rows * L
            c.bytes = 2 * (rows * n + c.n_out) * es
        elif kind == "batch":
            rows, n = geo
            L = (n + sum(c.pads) - ((c.w - 1) * c.dilation + 1)) // c.stride + 1
            y = torch.empty((rows, L), dtype=x.dtype, device=self.device)
            c.n_out = rows * L
            c.bytes = (rows * n + c.n_out) * es
        else:
            n = geo
            L = n - c.w + 1
            y = torch.empty(L, dtype=x.dtype, device=self.device)
            c.n_out = L
            c.bytes = (n + L) * es
        c.flops = 2 * c.w * c.n_out if c.op == "conv" else (2 * c.kh * c.kw * c.n_out if c.op == "conv2d" else 0)
        return y

    def _alloc_bwd(self, c, xd):
        """Backward cells: dx (or df + workspace) and the algorithmic bytes / unit counts.
        n_out = gradient elements written (dx), or for the filter gradient the
        rows x L products it reduces."""
        torch = self.torch
        x = xd[c.inp]
        if c.op == "pool2d_bwd":
            g = xd[c.inp2]
            c.n_out = x.numel()
            c.bytes = 4 * (x.numel() * (2 if c.mode == "max" else 1) + g.numel())
            return torch.empty_like(x)
        if c.op == "conv2d_bwd_in":  # inp = dy [B, C, OH, OW], inp2 = x (shape only)
            g, xs = x, xd[c.inp2]
            c.n_out = xs.numel()
            c.bytes = 4 * (g.numel() + xs.numel())
            c.flops = 2 * c.kh * c.kw * g.numel()
            return torch.empty_like(xs)
        if c.op == "conv2d_bwd_f":  # inp = x [B, C, H, W], inp2 = dy
            g = xd[c.inp2]
            if c.name not in self.ws:
                self.ws[c.name] = torch.empty(max(8, self.ss.ss_conv2d_backward_filter_workspace(c.kh, c.kw)),
                                              dtype=torch.uint8, device=self.device)
            c.n_out = g.numel()
            c.bytes = 4 * (x.numel() + g.numel())
            c.flops = 2 * c.kh * c.kw * g.numel()
            return torch.empty((c.kh, c.kw), dtype=torch.float32, device=self.device)
        if c.op in ("conv_bwd_in", "sum_bwd"):  # inp = dy [rows, L]
            rows, L = x.shape
            N = L + c.w - 1
            c.n_out = rows * N
            c.bytes = 4 * (rows * L + rows * N)
            c.flops = 2 * c.w * rows * L if c.op == "conv_bwd_in" else 0
            return torch.empty((rows, N), dtype=x.dtype, device=self.device)
        rows, N = x.shape                          # inp = x [rows, N], inp2 = dy [rows, L]
        L = xd[c.inp2].shape[1]
        if c.op == "max_bwd":
            c.n_out = rows * N
            c.bytes = 4 * (2 * rows * N + rows * L)
            return torch.empty((rows, N), dtype=x.dtype, device=self.device)
        if c.name not in self.ws:  # conv_bwd_f
            self.ws[c.name] = torch.empty(max(8, self.ss.ss_conv1d_backward_filter_workspace(c.w)),
                                          dtype=torch.uint8, device=self.device)
        c.n_out = rows * L
        c.bytes = 4 * (rows * N + rows * L + c.w)
        c.flops = 2 * c.w * rows * L
        return torch.empty(c.w, dtype=torch.float32, device=self.device)

    # ---- launches (every step of the path runs in libss through the C ABI)
    def _launch_bwd(self, c, xd, y):
        ss, st = self.ss, self.stream.cuda_stream
        x = xd[c.inp]
        if c.op == "pool2d_bwd":
            B, C, H, W = x.shape
            g = xd[c.inp2]
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
            ss.check(ss.ss_conv2d_backward_filter(x.data_ptr(), xd[c.inp2].data_ptr(), y.data_ptr(), B * C, H, W,
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
            ss.check(ss.ss_pool_max_backward(x.data_ptr(), xd[c.inp2].data_ptr(), y.data_ptr(), N, rows, c.w, 1,
                                             ss.SS_F32, st))
        else:
            rows, N = x.shape
            ws = self.ws[c.name]
            ss.check(ss.ss_conv1d_backward_filter(x.data_ptr(), xd[c.inp2].data_ptr(), y.data_ptr(), N, rows,
                                                  c.w, 1, ws.data_ptr(), ws.numel(), st))

    def launch_1d(self, c, x, y, v=None):
        ss = self.ss
        s = self.stream.cuda_stream
        code = ss.SS_I32 if x.dtype == self.torch.int32 else ss.SS_F32
        if x.dim() == 1:
            N, B = x.shape[0], 1
        else:
            B, N = x.shape
        win = (c.stride, c.dilation, c.pads[0], c.pads[1], ss.PAD_MODES[c.pad_mode], code, s)
        if c.op == "affine":
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

    def launch_cell(self, c, si=0, part="whole"):
        """part: 'whole' (interior + tail), 'interior' (needs no halo) or 'tail'
        (sequence-sharded cells only: the windows reaching into the halo)."""
        ss = self.ss
        kind, geo = self.meta[c.inp]
        xd, y = self.xs[si], self.ys[si][c.name]
        x = xd[c.inp]
        if kind == "seq":
            fn = (lambda xv, yv, c=c: self.launch_1d(c, xv, yv))
            if part in ("whole", "interior"):
                self.ssd.run_interior(x, geo, c.w, fn, y)
            if part in ("whole", "tail"):
                self.ssd.run_tail(x, geo, c.w, fn, y)
            return
        if part == "tail":
            return
        if c.op in BWD_OPS:
            self._launch_bwd(c, xd, y)
        elif c.op == "conv_mc":
            rows, n = geo
            ss.check(ss.ss_conv1d_mc(x.data_ptr(), self.wmc[c.name].data_ptr(), y.data_ptr(), rows,
                                     n // c.kh, c.kh, c.kw, c.w, self.stream.cuda_stream))
        elif c.op == "conv_mc_bwd_f":
            rows, n = geo
            L = n // c.kw
            xm = xd[c.inp2]
            need = ss.ss_conv1d_mc_backward_filter_workspace(c.kh, c.kw, c.w)
            ss.check(ss.ss_conv1d_mc_backward_filter(x.data_ptr(), xm.data_ptr(), y.data_ptr(), rows, L + c.w - 1,
                                                     c.kh, c.kw, c.w, self.ws[c.name].data_ptr(), need,
                                                     self.stream.cuda_stream))
        elif c.op == "conv_mc_bwd_in":
            rows, n = geo
            L = n // c.kw
            ss.check(ss.ss_conv1d_mc_backward_input(x.data_ptr(), self.wmc[c.name].data_ptr(), y.data_ptr(), rows,
                                                    L + c.w - 1, c.kh, c.kw, c.w, self.stream.cuda_stream))
        elif c.op == "conv2d_mc_bwd_f":
            B, OH, OW, cout = geo
            xm = xd[c.inp2]
            need = ss.ss_conv2d_mc_backward_filter_workspace(64, cout, c.kh, c.kw)
            ss.check(ss.ss_conv2d_mc_backward_filter(x.data_ptr(), xm.data_ptr(), y.data_ptr(), B, OH + c.kh - 1,
                                                     OW + c.kw - 1, 64, cout, c.kh, c.kw,
                                                     self.ws[c.name].data_ptr(), need, self.stream.cuda_stream))
        elif c.op == "conv2d_mc_bwd_in":
            B, OH, OW, cout = geo
            ss.check(ss.ss_conv2d_mc_backward_input(x.data_ptr(), self.wmc[c.name].data_ptr(), y.data_ptr(), B,
                                                    OH + c.kh - 1, OW + c.kw - 1, c.f.shape[1], cout, c.kh, c.kw,
                                                    self.stream.cuda_stream))
        elif c.op == "conv2d_mc":
            B, H, W, cin = geo
            ss.check(ss.ss_conv2d_mc(x.data_ptr(), self.wmc[c.name].data_ptr(), y.data_ptr(), B, H, W, cin,
                                     c.f.shape[0], c.kh, c.kw, self.stream.cuda_stream))
        elif c.op == "conv2d":
            B, C, H, W = geo
            ss.check(ss.ss_conv2d(x.data_ptr(), y.data_ptr(), B * C, H, W, c.f_flat, c.kh, c.kw, c.sh, c.sw,
                                  ss.SS_F32, self.stream.cuda_stream))
        elif c.op == "pool2d":
            B, C, H, W = geo
            ss.check(ss.ss_pool2d(x.data_ptr(), y.data_ptr(), B * C, H, W, c.kh, c.kw, c.sh, c.sw,
                                  ss.SS_POOL_MAX if c.mode == "max" else ss.SS_POOL_AVG, ss.SS_F32,
                                  self.stream.cuda_stream))
        else:
            self.launch_1d(c, x, y, xd.get(c.inp2) if c.inp2 else None)

    def seq_keys(self):
        return [k for k, (kind, _) in self.meta.items() if kind == "seq"]

    def post_halos(self, si=0):
        """Post every sequence input's halo exchange (one NCCL send/recv pair per
        neighbour); returns the work handles."""
        works = []
        if self.world > 1:
            for key in self.seq_keys():
                works += self.ssd.halo_start(self.xs[si][key], self.meta[key][1])
        return works

    def launch_interiors(self, si=0):
        for c in self.cells:
            self.launch_cell(c, si, "interior")

    def launch_tails(self, si=0):
        for c in self.cells:
            if self.meta[c.inp][0] == "seq":
                self.launch_cell(c, si, "tail")

    def step_eager(self, si=0):
        works = self.post_halos(si)
        self.launch_interiors(si)
        self.ssd.wait_all(works)
        self.launch_tails(si)

    # ---- CUDA graphs: the same launch mode at every N
    def capture(self, si=0):
        """Capture the step's kernels as two CUDA graphs (thread-local capture mode, so the NCCL
        watchdog thread's event queries stay legal during capture): A = every cell's interior
        (all of it for batch-sharded cells), B = the sequence-sharded tails (empty
        at N = 1).  The NCCL halo is posted eagerly before A and waited before B.
        Returns (graph A, graph B or None, libss launches per step)."""
        torch, ss = self.torch, self.ss
        n0 = ss.ss_launch_count()
        ga = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ga, stream=self.stream, capture_error_mode="thread_local"):
            self.launch_interiors(si)
        gb = None
        if self.world > 1 and self.seq_keys():
            gb = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gb, stream=self.stream, capture_error_mode="thread_local"):
                self.launch_tails(si)
        return ga, gb, ss.ss_launch_count() - n0

    def step_graph(self, graphs, si=0):
        ga, gb, _ = graphs
        works = self.post_halos(si)
        ga.replay()
        self.ssd.wait_all(works)
        if gb is not None:
            gb.replay()

    def cell_times(self, reps: int, replays: int):
        """Per-cell kernel time: each cell captured alone as a graph of `reps`
        launches alternating over the buffer sets (so no launch finds its input
        in L2 and every launch pays its own output write-back), replayed
        `replays` times after one warm replay; CUDA events on the launch stream.
        Returns {cell name: ms per launch}."""
        torch = self.torch
        out = {}
        nsets = len(self.xs)
        for c in self.cells:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream, capture_error_mode="thread_local"):
                for r in range(reps):
                    self.launch_cell(c, r % nsets, "whole")
            g.replay()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            for _ in range(replays):
                g.replay()
            e1.record(self.stream)
            torch.cuda.synchronize()
            out[c.name] = e0.elapsed_time(e1) / (reps * replays)
            del g
        return out

    # ---- sharded == unsharded (the library against itself, on regenerated global slices)
    def verify(self, seg: int = 8192):
        """Recompute sampled outputs from the GLOBAL input regenerated locally
        (synth is counter-based) with one unsharded call, and compare them with
        this rank's outputs bit for bit: windows at both ends of every sequence
        shard (the halo windows) and in its middle, the first and last local row
        / image of batch-sharded inputs.  Returns (outputs compared, mismatch list)."""
        torch, synth = self.torch, self.synth
        n_cmp, bad = 0, []
        for c in self.cells:
            kind, geo = self.meta[c.inp]
            sp = self.inputs_spec[c.inp]
            y = self.y[c.name]
            dt = self.x[c.inp].dtype
            if kind == "seq":
                sh = geo
                n_out = sh.n_outputs(c.w)
                if n_out == 0:
                    continue
                lo, hi = sh.start, sh.start + n_out
                mid = (lo + hi) // 2
                for o0, o1 in ((lo, lo + seg), (hi - seg, hi), (mid - seg // 2, mid + seg // 2)):
                    o0, o1 = max(o0, lo), min(o1, hi)
                    if o1 <= o0:
                        continue
                    xg = torch.empty(o1 - o0 + c.w - 1, dtype=dt, device=self.device)
                    synth.fill_device(xg, sp["dist"], sp["seed"], start=o0, **sp["kw"])
                    ref = torch.empty(o1 - o0, dtype=dt, device=self.device)
                    self.launch_1d(c, xg, ref)
                    torch.cuda.synchronize()
                    n_cmp += o1 - o0
                    if not torch.equal(ref, y[o0 - lo:o1 - lo]):
                        bad.append(f"{c.name} outputs [{o0}, {o1})")
            elif kind in ("batch", "image") and c.op in ("conv", "sum", "max", "min", "pool2d", "conv2d"):
                rows = geo[0]
                g0 = self.ssd.even_split(sp["rows"] if kind == "batch" else sp["images"], self.world, self.rank)[0]
                per = geo[1] if kind == "batch" else geo[1] * geo[2] * geo[3]
                for r in sorted({0, rows - 1}):
                    shape = (1, geo[1]) if kind == "batch" else (1,) + tuple(geo[1:])
                    xg = torch.empty(shape, dtype=dt, device=self.device)
                    synth.fill_device(xg, sp["dist"], sp["seed"], start=(g0 + r) * per, **sp["kw"])
                    ref = torch.empty((1,) + tuple(y.shape[1:]), dtype=y.dtype, device=self.device)
                    if c.op == "pool2d":
                        self.ss.pool2d(xg, (c.kh, c.kw), (c.sh, c.sw), c.mode, out=ref)
                    elif c.op == "conv2d":
                        self.ss.conv2d(xg, c.f, (c.sh, c.sw), out=ref)
                    else:
                        self.launch_1d(c, xg, ref)
                    torch.cuda.synchronize()
                    n_cmp += ref.numel()
                    if conv_on_tensor_cores(c):
                        # the tensor-core conv rounds by position in the staged view (a row's
                        # array tail runs on the FFMA path): equal within twice the BJ bound,
                        # the magnitudes sum|x||f| from the same library on |x|, |f|
                        mag = torch.empty_like(ref)
                        cabs = copy.copy(c)
                        cabs.f = np.abs(c.f)
                        self.launch_1d(cabs, xg.abs(), mag)
                        torch.cuda.synchronize()
                        ok = bool(((ref[0].double() - y[r].double()).abs() <=
                                   2 * (1e-5 * mag[0].double() + 1e-6)).all())
                    else:
                        ok = torch.equal(ref[0], y[r])
                    if not ok:
                        bad.append(f"{c.name} local row {r} (global {g0 + r})")
        return n_cmp, bad

    # ---- end to end: pinned host buffers -> device -> kernels -> host
    def setup_e2e(self):
        """Pinned host buffers for every input (a sequence shard WITHOUT its halo
        slots: those are filled by the exchange, never from the host) and every
        output, and the streams / events of the overlapped end-to-end loop."""
        torch = self.torch
        self.own = {k: (self.meta[k][1].size if self.meta[k][0] == "seq" else v.numel()) for k, v in self.x.items()}
        self.hx = {k: torch.empty(self.own[k], dtype=v.dtype, pin_memory=True) for k, v in self.x.items()}
        for k, v in self.x.items():
            self.hx[k].copy_(v.reshape(-1)[:self.own[k]])
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
        of the previous step, an output only after its previous D2H.  Sequence
        shards: the compute stream waits for the shard's H2D BEFORE the halo is
        posted (NCCL orders against the compute stream), and the H2D never
        touches the halo slots the exchange fills."""
        torch = self.torch
        for k in self.x:
            self.s_h2d.wait_event(self.ev_in_free[k])
            with torch.cuda.stream(self.s_h2d):
                self.x[k].view(-1)[:self.own[k]].copy_(self.hx[k], non_blocking=True)
            self.ev_in_ready[k].record(self.s_h2d)
        for k in self.seq_keys():
            self.stream.wait_event(self.ev_in_ready[k])
        works = self.post_halos(0)
        seq = {c.name for c in self.cells if self.meta[c.inp][0] == "seq"}

        def after(c):
            self.ev_out_ready[c.name].record(self.stream)
            for k in c.inputs():
                if self.last_reader[k] == c.name:
                    self.ev_in_free[k].record(self.stream)
            self.s_d2h.wait_event(self.ev_out_ready[c.name])
            with torch.cuda.stream(self.s_d2h):
                self.hy[c.name].copy_(self.y[c.name], non_blocking=True)
            self.ev_out_free[c.name].record(self.s_d2h)

        for c in self.cells:
            for k in c.inputs():
                self.stream.wait_event(self.ev_in_ready[k])
            self.stream.wait_event(self.ev_out_free[c.name])
            self.launch_cell(c, 0, "interior")
            if c.name not in seq or self.world == 1:
                after(c)
        self.ssd.wait_all(works)
        if self.world > 1:
            for c in self.cells:
                if c.name in seq:
                    self.launch_cell(c, 0, "tail")
                    after(c)

    def e2e_fence(self):
        """Make the compute stream wait for every outstanding copy."""
        for s in (self.s_d2h, self.s_h2d):
            done = self.torch.cuda.Event()
            done.record(s)
            self.stream.wait_event(done)


def _dtype_label(cells):
    """The arithmetic type(s) the timed path computes in, with the tensor-core conv's split precision."""
    dts = []
    if any(c.cfg == "cfg2" for c in cells):
        dts.append("i32")
    if any(c.cfg not in ("cfg2", "mc") for c in cells):
        dts.append("f32")
    if any(c.cfg == "mc" for c in cells):
        dts.append("bf16 x bf16 -> f32 accumulate (tensor cores, kind::f16)")
    lab = "/".join(dts)
    tc = [c for c in cells if conv_on_tensor_cores(c)]
    if tc:
        mode = ("3xTF32" if os.environ.get("SS_CONV_TC_MIXED", "1") == "0"
                else "TF32 hi*hi + one bf16 correction MMA")
        lab += f" ({', '.join(c.name for c in tc)}: tensor cores, {mode}, fp32 accumulate)"
    return lab


def run_cfg5(args, world, rank, device, barrier, max_over_ranks, coll):
    """BASELINE.json config 5 as a sub-record: one fp32 sequence of 2^32 elements
    (16 GiB), conv k=31 + sliding max w=64, STRONG-scaled (the one sequence split
    contiguously over the N ranks, (w_max-1)-element NCCL halo), timed like the
    suite (graphs A / B around the eagerly posted halo, max over ranks)."""
    import torch
    R = Runner("cfg5", world, rank, device, weak=False, nsets=1, cfg5_log2n=args.cfg5_log2n)
    R.step_eager()
    graphs = R.capture()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, args.cfg5_steps))
    for _ in range(3):
        R.step_graph(graphs)
    with ClockSampler(torch.cuda.current_device()) as clk:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(R.stream)
        for _ in range(steps):
            R.step_graph(graphs)
        t1.record(R.stream)
        torch.cuda.synchronize()
        barrier()
    ms = max_over_ranks(t0.elapsed_time(t1))
    cell_ms = R.cell_times(reps=2, replays=max(1, steps // 4))
    tot = torch.tensor([float(sum(c.n_out for c in R.cells)), float(sum(c.bytes for c in R.cells))],
                       dtype=torch.float64, device=coll)
    if world > 1:
        torch.distributed.all_reduce(tot)
    n_out, nbytes = float(tot[0]), float(tot[1])
    rec = {"workload": f"cfg5: fp32 N=2^{args.cfg5_log2n}, conv k=31 + max w=64, seq-sharded x{world} (strong)",
           "value": round(n_out * steps / (ms * 1e-3) / 1e9, 3), "unit": "GElem/s",
           "ms_per_step": round(ms / steps, 4), "steps": steps, "n_gpus": world, "scaling": "strong",
           "hbm_gbs": round(nbytes * steps / (ms * 1e-3) / 1e9, 1),
           "cells": {k: round(v, 4) for k, v in cell_ms.items()},
           "gpu_launches_per_step": int(graphs[2]), "clocks": clk.summary(),
           "parity": "tests/test_configs_gpu.py::test_cfg5_full_size_and_shard_emulation (oracle, sampled + shard "
                     "boundaries); --verify: sharded == unsharded"}
    if args.verify:
        n_cmp, bad = R.verify()
        t = torch.tensor([float(n_cmp), float(len(bad))], dtype=torch.float64, device=coll)
        if world > 1:
            torch.distributed.all_reduce(t)
        rec["verify"] = {"compared": int(t[0]), "mismatches": int(t[1]), "first": bad[:4]}
    del R, graphs
    torch.cuda.empty_cache()
    return rec


_T0 = time.perf_counter()


def _phase(name: str) -> None:
    """Wall-clock progress of the bench phases on stderr (never part of the JSON line)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f} s] {name}", file=sys.stderr, flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local % torch.cuda.device_count())
        if args.dist_backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")   # keep the communicator init lines in the log
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        else:  # test mode: several ranks may share a GPU; host-staged halo
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    device = torch.device("cuda", torch.cuda.current_device())
    import paper_2305_16513_b200 as ss
    torch.cuda.set_stream(torch.cuda.Stream())  # graphs are captured on a non-default stream: run everything there
    coll = device if args.dist_backend == "nccl" else torch.device("cpu")

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
        t = torch.tensor([v], dtype=torch.float64, device=coll)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    _phase("init")
    R = Runner(args.workload, world, rank, device, weak=args.scaling == "weak", nsets=2,
               cfg5_log2n=args.cfg5_log2n)
    torch.cuda.synchronize()
    for _ in range(args.warmup):  # eager warm-up (kernel attributes, tensor maps)
        R.step_eager()
    barrier()
    _phase("capture")
    graphs = R.capture()
    launches_per_step = graphs[2]
    for _ in range(args.warmup):
        R.step_graph(graphs)
    barrier()
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        barrier()
        t0.record(R.stream)
        for _ in range(args.steps):
            R.step_graph(graphs)
        t1.record(R.stream)
        torch.cuda.synchronize()
        barrier()
    ms_local = t0.elapsed_time(t1)
    ms = max_over_ranks(ms_local)
    out_local = sum(c.n_out for c in R.cells) * args.steps
    bytes_local = sum(c.bytes for c in R.cells) * args.steps
    tot = torch.tensor([out_local, bytes_local], dtype=torch.float64, device=coll)
    if world > 1:
        dist.all_reduce(tot)
    out_total, bytes_total = float(tot[0]), float(tot[1])
    value = out_total / (ms * 1e-3) / 1e9
    hbm_gbs = bytes_total / (ms * 1e-3) / 1e9

    _phase("cell timing")
    # per-kernel (cell) times: each cell alone as a graph over 2 buffer sets
    reps = 2 * max(2, args.cell_reps // 2)
    cell_ms = R.cell_times(reps=reps, replays=max(1, args.steps // reps))
    peak_hbm, peak_src = measured_peaks()
    cells = []
    for c in R.cells:
        avg_ms = cell_ms[c.name]
        gbs = c.bytes / (avg_ms * 1e-3) / 1e9
        d = {"cell": c.name, "avg_ms": round(avg_ms, 5), "n_out": c.n_out, "bytes": c.bytes,
             "gelem_s": round(c.n_out / (avg_ms * 1e-3) / 1e9, 2), "gbs": round(gbs, 1),
             "frac_hbm": round(gbs / peak_hbm, 4), "frac_8tbs": round(gbs / 8000.0, 4), "share": 0.0}
        if c.op in ("conv_mc", "conv2d_mc", "conv_mc_bwd_in", "conv_mc_bwd_f", "conv2d_mc_bwd_in",
                    "conv2d_mc_bwd_f"):
            d["tc_frac"] = round(c.flops / (avg_ms * 1e-3) / 1e12 / (2 * tf32_peak_tflops()), 4)  # bf16 peak
        elif conv_on_tensor_cores(c):
            d["tc_frac"] = round(c.n_out * TC_FLOP_PER_OUT / (avg_ms * 1e-3) / 1e12 / tf32_peak_tflops(), 4)
        elif c.op in ("conv", "conv_bwd_in", "conv_bwd_f", "conv2d", "conv2d_bwd_in", "conv2d_bwd_f"):
            d["fma_frac"] = round(c.flops / 2 / (avg_ms * 1e-3) / FP32_FMA_PEAK, 4)
        cells.append(d)
    step_ms = ms / args.steps
    tot_k = sum(d["avg_ms"] for d in cells)
    for d in cells:
        d["share"] = round(d["avg_ms"] / tot_k, 4)
    dom = max(cells, key=lambda d: d["avg_ms"])
    dom_cell = next(c for c in R.cells if c.name == dom["cell"])
    if dom_cell.op in ("conv", "conv_bwd_in", "conv_bwd_f", "conv2d", "conv2d_bwd_in", "conv2d_bwd_f") and \
            dom.get("fma_frac", 0) > dom["frac_hbm"]:
        achieved = dom_cell.flops / (dom["avg_ms"] * 1e-3) / 1e12
        roofline = {"bound": "alu", "kernel": dom["cell"], "achieved": round(achieved, 2),
                    "peak": round(2 * FP32_FMA_PEAK / 1e12, 2), "unit": "TFLOP/s",
                    "frac": round(achieved / (2 * FP32_FMA_PEAK / 1e12), 4),
                    "peak_source": "148 SM x 128 FP32 FMA/clk x 1965 MHz (DESIGN.md)",
                    "hbm_gbs": dom["gbs"], "hbm_frac": dom["frac_hbm"], "traffic": None}
    else:
        roofline = {"bound": "hbm", "kernel": dom["cell"], "achieved": dom["gbs"], "peak": peak_hbm,
                    "unit": "GB/s", "frac": dom["frac_hbm"], "peak_source": peak_src, "traffic": None,
                    "frac_8tbs": dom["frac_8tbs"]}
        if "tc_frac" in dom and dom_cell.op in ("conv_mc", "conv2d_mc", "conv_mc_bwd_in", "conv_mc_bwd_f",
                                                "conv2d_mc_bwd_in", "conv2d_mc_bwd_f"):
            roofline["tensor_frac"] = dom["tc_frac"]
            roofline["tensor_peak_tflops"] = round(2 * tf32_peak_tflops(), 1)
            roofline["tensor_note"] = "bf16 MMA work (2 k Cin flop/output) / measured dense bf16 peak"
        elif "tc_frac" in dom:  # tensor-core conv: HBM is the roofline (its TC ceiling is higher)
            roofline["tensor_frac"] = dom["tc_frac"]
            roofline["tensor_peak_tflops"] = round(tf32_peak_tflops(), 1)
            roofline["tensor_note"] = (f"executed MMA work ({TC_FLOP_PER_OUT} TF32-equivalent flop/output: "
                                       "xh*fh in TF32 + one bf16 correction product at half weight) / dense "
                                       "TF32 peak (measured bf16 / 2)")
    roofline["algorithmic_bytes_per_launch"] = dom_cell.bytes
    roofline["avg_launch_ms"] = dom["avg_ms"]
    roofline["share_of_step"] = round(dom["avg_ms"] / step_ms, 4)
    roofline["timing"] = (f"the kernel alone, captured as a CUDA graph of {reps} launches alternating over 2 "
                          "input/output buffer sets, CUDA events on its stream")
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):  # dram bytes per launch from a committed `ncu --set full` capture
        try:
            roofline["traffic"] = json.load(open(tf)).get(dom["cell"])
        except Exception:  # noqa: BLE001
            pass

    verify = None
    if args.verify:
        n_cmp, bad = R.verify()
        t = torch.tensor([float(n_cmp), float(len(bad))], dtype=torch.float64, device=coll)
        if world > 1:
            dist.all_reduce(t)
        verify = {"compared": int(t[0]), "mismatches": int(t[1]), "first": bad[:4],
                  "what": "sharded outputs == one unsharded call on the regenerated global slice, bitwise "
                          "(tensor-core conv cells: within twice the BASELINE.json bound)"}

    _phase("e2e")
    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        R.setup_e2e()
        for _ in range(2):
            R.step_e2e()
        R.e2e_fence()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        n_e2e = max(2, min(args.steps, args.e2e_steps))
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
    cells_info = {"cells": cells, "cells_sum_ms": round(tot_k, 4), "step_ms": round(step_ms, 4),
                  "cells_sum_over_step": round(tot_k / step_ms, 4)}
    names = [c.name for c in R.cells]
    inputs_spec = {k: {kk: vv for kk, vv in v.items() if kk != "kw"} for k, v in R.inputs_spec.items()}
    dtype = _dtype_label(R.cells)
    del R, graphs
    torch.cuda.empty_cache()

    cfg5 = None
    if args.workload == "suite" and not args.no_cfg5:
        _phase("cfg5")
        cfg5 = run_cfg5(args, world, rank, device, barrier, max_over_ranks, coll)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        _phase("cpu baseline")
        cpu = cpu_baseline(args.workload, budget_s=args.cpu_budget)
    _phase("done")

    if rank == 0:
        cfg = {"workload": args.workload, "cells": names,
               "launch_mode": "CUDA graphs at every N: A = interiors + batch-sharded cells, B = sequence tails "
                              "(N > 1), NCCL halo posted eagerly between them",
               "parallelism": f"{'seq+batch' if args.workload == 'suite' else 'shard'} x{world}",
               "l2": "step: every cell's input > L2 (126 MB) or, for cfg4, a distinct input copy per cell; "
                     "per-cell timing alternates 2 buffer sets",
               "inputs": inputs_spec}
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GElem/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4),
                "higher_is_better": True, "scaling": args.scaling,
                "vs_baseline": None, "dtype": dtype,
                "data": "synthetic: splitmix64 counter-based generator (synth/), BASELINE.json seeds; "
                        "U[0,1), U[-1,1), U{-1000..1000} exact; 'N(0,1)' = Irwin-Hall(12) stand-in "
                        "(mean 0, var 1, support [-6,6), DESIGN.md R12)",
                "config": cfg, "hbm_gbs": round(hbm_gbs, 1), "hbm_frac_8tbs": round(hbm_gbs / 8000.0, 4),
                "hbm_frac_measured": round(hbm_gbs / peak_hbm, 4),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches_per_step * args.steps),
                "clocks": clk.summary(), "cfg5": cfg5, "verify": verify,
                "cells_sum_over_step": cells_info["cells_sum_over_step"], "impl": "ours"}
        print(json.dumps(line), flush=True)
        if args.cells_out:
            with open(args.cells_out, "w") as fh:
                json.dump({"line": line, **cells_info}, fh, indent=1)
        else:
            print(json.dumps(cells_info), file=sys.stderr)
    if world > 1:
        dist.destroy_process_group()


# ============================================================== oracle arm
def _seq_task(x, w, fn):
    """A 1-D sample x whose len(x) - w + 1 windows can be split into output
    ranges: run(i, parts) evaluates part i (input x[a : b + w - 1] for outputs
    [a, b)) and returns its output count."""
    n_out = x.size - w + 1

    def run(i=0, parts=1):
        a, b = n_out * i // parts, n_out * (i + 1) // parts
        if b <= a:
            return 0
        fn(x[a:b + w - 1])
        return b - a
    return run


def _rows_task(x, fn, outs_per_row):
    """A sample of independent rows / planes (leading axis), split by rows."""
    def run(i=0, parts=1):
        r0, r1 = x.shape[0] * i // parts, x.shape[0] * (i + 1) // parts
        if r1 <= r0:
            return 0
        fn(x[r0:r1])
        return (r1 - r0) * outs_per_row
    return run


def _whole_task(fn):
    """A sample that is not split: part 0 runs it all."""
    return lambda i=0, parts=1: fn() if i == 0 else 0


def oracle_sample_plan(workload: str, frac: float):
    """Bounded sample of every cell: the same cells, a `frac` share of each
    (leading rows / images / output range).  Returns [(cell, run)] where
    run(i, parts) evaluates part i of `parts` of the sample with the oracle and
    returns its output count (run() = the whole sample)."""
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
            fn = {"sum": lambda xv, c=c: oracle.pool_sum(xv, c.w), "max": lambda xv, c=c: oracle.pool_max(xv, c.w),
                  "conv": lambda xv, c=c: oracle.conv1d(xv, c.f)}[c.op]
            plan.append((c, _seq_task(x, c.w, fn)))
        elif c.cfg == "cfg3":
            rows = max(1, int(round(64 * frac)))
            n = 1 << 20
            if rows * n > 64 * n * frac * 1.5:  # frac below one row: shorten the row instead
                n = max(c.w, int(64 * (1 << 20) * frac))
                rows = 1
            x = synth.normal(3, rows * n).reshape(rows, n)
            if rows == 1:
                plan.append((c, _seq_task(x[0], c.w, lambda xv, c=c: oracle.conv1d(xv, c.f))))
            else:
                plan.append((c, _rows_task(x, lambda xr, c=c: oracle.conv1d(xr, c.f), n - c.w + 1)))
        elif c.cfg == "mc" and c.op == "conv2d_mc":
            hw, cin = int(c.name.split("_")[1].split("x")[0]), c.f.shape[1]
            imgs = max(1, int(round(128 * frac)))
            xb = oracle.to_bf16_bits(synth.normal(102, imgs * hw * hw * cin).reshape(imgs, hw, hw, cin))
            wb = oracle.to_bf16_bits(c.f)
            plan.append((c, _rows_task(xb, lambda xi, wb=wb: oracle.conv2d_mc(xi, wb),
                                       (hw - 2) * (hw - 2) * c.f.shape[0])))
        elif c.cfg == "mc" and c.op == "conv2d_mc_bwd_f":
            imgs = max(1, int(round(128 * frac)))
            gb = oracle.to_bf16_bits(synth.normal(104, imgs * 54 * 54 * 64).reshape(imgs, 54, 54, 64))
            xb = oracle.to_bf16_bits(synth.normal(102, imgs * 56 * 56 * 64).reshape(imgs, 56, 56, 64))
            plan.append((c, _whole_task(lambda gb=gb, xb=xb, imgs=imgs: (
                oracle.conv2d_mc_backward_filter(gb, xb, 3, 3), imgs * 54 * 54 * 64)[1])))
        elif c.cfg == "mc" and c.op == "conv2d_mc_bwd_in":
            imgs = max(1, int(round(128 * frac)))
            gb = oracle.to_bf16_bits(synth.normal(104, imgs * 54 * 54 * 64).reshape(imgs, 54, 54, 64))
            wb = oracle.to_bf16_bits(c.f)
            plan.append((c, _rows_task(gb, lambda gi, wb=wb: oracle.conv2d_mc_backward_input(gi, wb, 56, 56),
                                       56 * 56 * 64)))
        elif c.cfg == "mc" and c.op == "conv_mc_bwd_f":
            cin, cout, k = c.kh, c.kw, c.w
            N = max(k + 1, int(16 * 65536 * frac))
            gb = oracle.to_bf16_bits(synth.normal(99, (N - k + 1) * cout).reshape(1, N - k + 1, cout))
            xb = oracle.to_bf16_bits(synth.normal(96, N * cin).reshape(1, N, cin))
            plan.append((c, _whole_task(lambda gb=gb, xb=xb, k=k, N=N, cout=cout: (
                oracle.conv1d_mc_backward_filter(gb, xb, k), (N - k + 1) * cout)[1])))
        elif c.cfg == "mc" and c.op == "conv_mc_bwd_in":
            cin, cout, k = c.kh, c.kw, c.w
            N = max(k + 1, int(16 * 65536 * frac))
            gb = oracle.to_bf16_bits(synth.normal(98, (N - k + 1) * cout).reshape(1, N - k + 1, cout))
            wb = oracle.to_bf16_bits(c.f)
            plan.append((c, _whole_task(lambda gb=gb, wb=wb, N=N, cin=cin: (
                oracle.conv1d_mc_backward_input(gb, wb, N), N * cin)[1])))
        elif c.cfg == "mc":
            cin, cout, k = c.kh, c.kw, c.w
            n = max(k + 1, int(16 * 65536 * frac))
            xb = oracle.to_bf16_bits(synth.normal(96, n * cin).reshape(1, n, cin))
            wb = oracle.to_bf16_bits(c.f)
            plan.append((c, _whole_task(lambda xb=xb, wb=wb, c=c, n=n: (oracle.conv1d_mc(xb, wb),
                                                                          (n - c.w + 1) * c.kw)[1])))
        elif c.cfg == "conv2d":
            planes = max(1, int(round(32 * 64 * frac)))
            x = synth.uniform01(5, planes * 112 * 112).reshape(planes, 112, 112)
            oh = (112 - c.kh) // c.sh + 1
            plan.append((c, _rows_task(x, lambda xp, c=c: oracle.conv2d(xp, c.f, c.sh, c.sw), oh * oh)))
        elif c.cfg == "backward" and c.op == "pool2d_bwd":
            planes = max(1, int(round(32 * 64 * frac)))
            oh = (112 - c.kh) // c.sh + 1
            x = synth.uniform01(5, planes * 112 * 112).reshape(planes, 112, 112)
            g = synth.normal(34, planes * oh * oh).reshape(planes, oh, oh)
            m = oracle.POOL2D_MAX if c.mode == "max" else oracle.POOL2D_AVG
            plan.append((c, _whole_task(lambda x=x, g=g, c=c, m=m: (oracle.pool2d_backward(
                x, g, 112, 112, c.kh, c.kw, c.sh, c.sw, m), x.size)[1])))
        elif c.cfg == "backward" and c.op in ("conv2d_bwd_in", "conv2d_bwd_f"):
            planes = max(1, int(round(32 * 64 * frac)))
            oh = 112 - c.kh + 1
            x = synth.uniform01(5, planes * 112 * 112).reshape(planes, 112, 112)
            g = synth.normal(34, planes * oh * oh).reshape(planes, oh, oh)
            if c.op == "conv2d_bwd_in":
                fn = (lambda g=g, c=c: (oracle.conv2d_backward_input(g, c.f, 112, 112), planes * 112 * 112)[1])
            else:
                fn = (lambda x=x, g=g, c=c: (oracle.conv2d_backward_filter(x, g, c.kh, c.kw), g.size)[1])
            plan.append((c, _whole_task(fn)))
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
            plan.append((c, _whole_task(fn)))
        elif c.cfg in ("stride", "winspec"):
            rows, n = 1, max(4 * (c.w - 1) * c.dilation + 8, int(64 * (1 << 20) * frac))
            x = synth.normal(3, rows * n).reshape(rows, n)
            kw = dict(s=c.stride, d=c.dilation, pl=c.pads[0], pr=c.pads[1], mode=c.pad_mode)
            L = oracle.out_len_ex(n, c.w, c.stride, c.dilation, c.pads[0], c.pads[1])
            fn = {"sum": lambda x=x, c=c, kw=kw: oracle.pool_sum_ex(x, c.w, **kw),
                  "max": lambda x=x, c=c, kw=kw: oracle.pool_max_ex(x, c.w, **kw),
                  "min": lambda x=x, c=c, kw=kw: oracle.pool_min_ex(x, c.w, **kw),
                  "conv": lambda x=x, c=c, kw=kw: oracle.conv1d_ex(x, c.f, **kw)}[c.op]
            plan.append((c, _whole_task(lambda fn=fn, L=L: (fn(), L)[1])))
        elif c.cfg == "affine":
            n = max(c.w, int(8 * (1 << 24) * frac))
            u = synth.uab(31, n, 0.5, 1.0)
            v = synth.normal(32, n)
            plan.append((c, _whole_task(lambda u=u, v=v, c=c: (oracle.affine_window(u, v, c.w),
                                                                u.size - c.w + 1)[1])))
        else:  # cfg4
            planes = max(1, int(round(32 * 64 * frac)))
            x = synth.uniform01(5, planes * 112 * 112).reshape(planes, 112, 112)
            m = oracle.POOL2D_MAX if c.mode == "max" else oracle.POOL2D_AVG
            oh = (112 - c.kh) // c.sh + 1
            ow = (112 - c.kw) // c.sw + 1
            plan.append((c, _rows_task(x, lambda xp, c=c, m=m: oracle.pool2d(xp, c.kh, c.kw, c.sh, c.sw, m),
                                       oh * ow)))
    return plan


def _run_parts(plan, parts: int = 1):
    """Run the plan's samples split into `parts` disjoint pieces, one thread per
    piece (ctypes releases the GIL inside every oracle call, so the threads run
    on separate cores).  Returns (outputs, seconds)."""
    from concurrent.futures import ThreadPoolExecutor
    t0 = time.perf_counter()
    if parts == 1:
        outs = sum(run() for _, run in plan)
    else:
        with ThreadPoolExecutor(parts) as ex:
            outs = sum(ex.map(lambda i: sum(run(i, parts) for _, run in plan), range(parts)))
    return outs, time.perf_counter() - t0


def cpu_baseline(workload: str, budget_s: float = 10.0):
    """Time the oracle as it stands (plain C, -O2) on a bounded sample of the
    workload: on one thread, then on every host core (os.cpu_count() threads,
    the sample split into disjoint output ranges / rows / planes)."""
    import oracle
    oracle.build()
    frac = 1.0 / 4096 if workload != "cfg1" else 1.0
    outs, dt = _run_parts(oracle_sample_plan(workload, frac))  # calibrate
    if workload != "cfg1" and dt > 0:
        frac = min(1.0, frac * max(1.0, budget_s / dt))
    plan = oracle_sample_plan(workload, frac)
    outs, dt = _run_parts(plan)
    cores = os.cpu_count() or 1
    outs_all, dt_all = _run_parts(plan, cores)
    return {"value": round(outs_all / dt_all / 1e9, 6), "unit": "GElem/s", "cores": cores, "kind": "oracle",
            "sample": f"every cell of workload '{workload}', {frac:.3%} of its outputs/rows/images ({outs_all} "
                      f"outputs), split over {cores} threads into disjoint output ranges / rows / planes; plain C "
                      f"oracle -O2, {dt_all:.1f} s",
            "host_cpu_count": cores,
            "single_thread": {"value": round(outs / dt / 1e9, 6), "unit": "GElem/s", "cores": 1, "outputs": outs,
                              "seconds": round(dt, 2)},
            "seconds": round(dt_all, 2)}


def run_reference(args):
    """The tier's reference arm: the CPU oracle (plain C, as it stands) on every
    host core, each step a bounded sample of every cell of the workload."""
    world, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference; the others exit 0 without work
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1
    frac = 1.0 / 32 if args.workload != "cfg1" else 1.0
    plan = oracle_sample_plan(args.workload, frac)
    for _ in range(args.warmup):
        _run_parts(plan, cores)
    times, outs = [], 0
    for _ in range(args.steps):
        outs, dt = _run_parts(plan, cores)
        times.append(dt)
    tot = sum(times)
    value = outs * args.steps / tot / 1e9
    sample = (f"{frac:.4%} of every cell of '{args.workload}' per step, split over {cores} threads into disjoint "
              "output ranges / rows / planes (plain C oracle -O2)")
    line = {"metric": METRIC, "value": round(value, 6), "unit": "GElem/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64/i64 accumulate", "data": "synthetic (same generator and seeds)",
            "config": {"workload": args.workload, "sample_fraction": frac, "threads": cores},
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 6), "unit": "GElem/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 6), "unit": "GElem/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="suite", choices=["suite", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "stride",
                                                             "winspec", "affine", "backward", "conv2d", "mc"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="multi-GPU: weak = N x the BASELINE shape (config-sized share per rank), strong = split it")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cell-reps", type=int, default=20, help="launches per per-cell timing graph (even)")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the config-5 sub-record of the suite")
    ap.add_argument("--cfg5-log2n", type=int, default=32, help="config 5 sequence length (2^32 in BASELINE.json)")
    ap.add_argument("--cfg5-steps", type=int, default=20)
    ap.add_argument("--verify", action="store_true",
                    help="check sharded outputs against one unsharded call on regenerated global slices (bitwise)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--cells-out", default=None)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo = test mode (ranks may share one GPU, host-staged halo)")
    args = ap.parse_args()
    world = os.environ.get("WORLD_SIZE")
    if args.impl == "ours" and args.gpus > 1 and world is None:
        # one process per GPU: re-launch this command under torchrun, rank 0 prints the line
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world is not None and args.impl == "ours" and int(world) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
