#!/usr/bin/env python
"""bench.py — PSCWin layer latency on B200 (BASELINE.json metric: "PSCWin encoder-layer latency ms/image").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload 1024|2048|4096] [--impl ours|reference]

A step is one pass of the whole hot path over one batch of synthetic input: at the default workload
(configs[1], 1024^2 input) the three layers of HRSAM stage 1 under the global-alternation reading
(Q8): plain window attention (P), padded-shift window attention (S, LEARNABLE pad) and the
cycle-scan module + plain attention (CS+P), ViT-B (C=768, 12 heads, w=16, shift 8, N=32, E=2), bf16,
B=1 image per rank. Under torchrun each rank processes its own image (weak scaling; no data-path
collective). Inputs are resident in HBM before timing; L2 is flushed (256 MiB write) before every
timed step, and each step is timed with CUDA events on the launching stream; max over ranks.

Also reported: e2e (same metric through the public API with pinned-host input/output copies in the timed
region), the dominant kernel's roofline (per-kernel CUDA-event timing inside the library), the fp64 CPU
oracle as cpu_baseline (rank 0, N=1), clocks sampled by nvidia-smi during the timed region, and the number
of library kernel launches inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

F32_KEYS = {"ln1_g", "ln1_b", "b_qkv", "b_o", "lns_g", "lns_b", "conv_w", "conv_b", "w_dt", "b_dt", "a_log",
            "d_skip", "ln2_g", "ln2_b", "b_fc1", "b_fc2"}
METRIC = "PSCWin encoder-layer latency ms/image"


FFN_HIDDEN = 0   # set by --ffn: 3072 = 768 x 4, the FFN sub-layer after every attention sub-layer


def workload(name: str):
    """(label, B per rank, [LayerConfig per layer])."""
    if name == "1024":
        side, B, n_layers = 64, 1, 3
        label = "1024^2 (64x64 tokens) HRSAM stage 1: P, S(pad learnable), CS+P; ViT-B bf16"
    elif name == "2048":
        side, B, n_layers = 128, 8, 12
        label = "2048^2 (128x128 tokens) full 12-layer PSCWin stack (6 P, 6 S, 4 CS); ViT-B bf16"
    elif name == "4096":
        side, B, n_layers = 256, 1, 12
        label = "4096^2 (256x256 tokens) full 12-layer PSCWin stack, one image per GPU; ViT-B bf16"
    else:
        raise SystemExit(f"unknown workload {name}")
    cfgs = []
    for i in range(n_layers):
        shifted, cs = synth.stack_layer_kind(i)
        cfgs.append(synth.vitb(side, B=B, shift_x=8 if shifted else 0, shift_y=8 if shifted else 0,
                               cycle_scan=int(cs), mlp_hidden=FFN_HIDDEN))
    if FFN_HIDDEN:
        label += f" + FFN {FFN_HIDDEN}"
    return label, B, cfgs


OVERVIEW = 32   # HRSAM++ overview image 512^2 -> 32 x 32 tokens
MS_SCALES = [(64, 64), (128, 128), (256, 256)]   # config 5: 1024^2 + 2048^2 + 4096^2 token grids per sample


def ms_workload():
    """configs[4] (HRSAM++ multi-scale): per sample the 64^2 + 128^2 + 256^2 token grids
    packed into one sequence of 86016 tokens; the 12-layer global-alternation stack with a single-scale
    cycle-scan module before layers 2, 5, 8, 11 and a multi-scale cycle-scan module closing each stage
    (after layers 2, 5, 8, 11; Fig. 4). B = 2 samples per GPU (config 5: batch 16 over 8 GPUs).
    Returns (label, B, [(cfg, attention, cs_mode, weight_seed)])."""
    B = 2
    specs = []
    for i in range(12):
        shifted, cs = synth.stack_layer_kind(i)
        cfg = synth.vitb(64, B=B, shift_x=8 if shifted else 0, shift_y=8 if shifted else 0, mlp_hidden=FFN_HIDDEN)
        specs.append((cfg, 1, 1 if cs else 0, i))
        if cs:
            specs.append((synth.vitb(64, B=B, shift_x=0, shift_y=0), 0, 2, 100 + i))
    label = ("HRSAM++ multi-scale: 64^2+128^2+256^2 token grids packed per sample (86016 tokens), 12-layer stack "
             "+ 4 single-scale and 4 multi-scale cycle-scan modules; ViT-B bf16")
    if FFN_HIDDEN:
        label += f" + FFN {FFN_HIDDEN}"
    return label, B, specs


def layer_metas(args):
    """Per-layer shapes for the roofline accounting: T tokens, widths, whether attention / cycle scan run."""
    if args.workload == "ms":
        _, B, specs = ms_workload()
        T = B * sum(h * w for h, w in MS_SCALES)
        return [dict(T=T, B=B, C=c.C, D=c.D, N=c.N, R=c.R, attn=a, cs=int(cs > 0), Hd=c.mlp_hidden * a, pad=0,
                     Hp=0, Wp=0, chunks=-(-T // (256 * B))) for c, a, cs, _ in specs]
    _, _, cfgs = workload(args.workload)
    out = []
    for c in cfgs:
        sh = c.shift_x or c.shift_y
        pt, pl_ = (c.window - c.shift_y) % c.window, (c.window - c.shift_x) % c.window
        Hp = -(-(c.H + pt) // c.window) * c.window
        Wp = -(-(c.W + pl_) // c.window) * c.window
        out.append(dict(T=c.B * c.H * c.W, B=c.B, C=c.C, D=c.D, N=c.N, R=c.R, attn=1, cs=int(c.cycle_scan),
                        Hd=c.mlp_hidden, pad=int(bool(sh) and c.pad_mode == synth.PAD_LEARNABLE), Hp=Hp, Wp=Wp,
                        chunks=scan_chunks(c)))
    return out


def scan_chunks(c):
    """Chunk count of the cycle scan (the library's choose_chunk is internal; the carry's bytes are reported from
    the chunk length the library reports through pscwin_scan_plan when available, else 256 tokens)."""
    try:
        import paper_2407_02109_b200 as pl
        return pl.scan_chunks(c.B, c.H * c.W, c.D)
    except Exception:
        return -(-(c.H * c.W) // 256)


# ----------------------------------------------------------------------------------------------- roofline
def _ln_fold(T: int):
    """Which LayerNorms the library folds into the next projection for an image of T tokens (abi.cu ln_fold_mode):
    (LN1 -> QKV folded, LN_s / LN2 folded too)."""
    mode = int(os.environ.get("PSCWIN_LN_FOLD", "2"))
    mode = mode if mode in (0, 1) else 2
    on = mode != 0 and T >= int(os.environ.get("PSCWIN_LN_FOLD_MIN_T", "16384"))
    return on, on and mode == 1


def kernel_work(label: str, metas):
    """Algorithmic work of a kernel label over ONE step (DESIGN.md §6 "algorithmic work per unit x units"),
    summed over the layers that launch it: returns (bound, amount, unit_scale, unit) or None."""
    tot = 0.0
    bound = unit = None
    scale = 1.0
    for m in metas:
        T, C, D, N, R = m["T"], m["C"], m["D"], m["N"], m["R"]
        a, cs, Hd = m["attn"], m["cs"], m["Hd"]
        if label == "window_attention":
            bound, scale, unit = "hbm", 1e9, "GB/s"
            tot += a * 8.0 * T * C                      # Q,K,V read + O write, bf16, real tokens
        elif label in ("scan_pass1", "scan_pass2"):
            bound, scale, unit = "alu", 1e9, "Gexp/s"
            tot += cs * 1.0 * T * D * N                 # one ex2 per (token, channel, state)
        elif label == "gemm_qkv_rope":
            bound, scale, unit = "tensor", 1e12, "TFLOP/s"
            tot += a * 2.0 * T * C * 3 * C
        elif label == "gemm_out_proj":
            bound, scale, unit = "tensor", 1e12, "TFLOP/s"
            tot += a * 2.0 * T * C * C
        elif label == "gemm_in_proj":
            bound, scale, unit = "tensor", 1e12, "TFLOP/s"
            tot += cs * 2.0 * T * C * 2 * D
        elif label == "gemm_out_proj_scan":
            bound, scale, unit = "tensor", 1e12, "TFLOP/s"
            tot += cs * 2.0 * T * D * C
        elif label == "gemm_x_proj":     # AI = 2(R+2N)D / (2D + 4(R+2N)) ~ 100 FLOP/B < ridge 255: HBM-bound
            bound, scale, unit = "hbm", 1e9, "GB/s"
            tot += cs * T * (2.0 * D + 4.0 * (R + 2 * N))   # v read (bf16) + (delta, B, C) write (f32)
        elif label == "scan_dt":         # Delta = softplus(delta W_dt^T + b): delta read, Delta write (f32)
            bound, scale, unit = "hbm", 1e9, "GB/s"
            tot += cs * T * (4.0 * R + 4.0 * D)
        elif label == "scan_carry":      # chunk summaries read (a = sum Delta, b = end state), entry states written
            bound, scale, unit = "hbm", 1e9, "GB/s"
            tot += cs * m["B"] * m["chunks"] * (4.0 * D + 2 * 4.0 * D * N)
        elif label == "pad_qkv":         # p W_qkv^T + b: W_qkv read once (bf16), 3C f32 written
            bound, scale, unit = "hbm", 1e9, "GB/s"
            tot += m["pad"] * (2.0 * 3 * C * C + 4.0 * 3 * C)
        elif label == "pad_tables":      # rotated pad keys per padded column / row and the pad value (bf16)
            bound, scale, unit = "hbm", 1e9, "GB/s"
            tot += m["pad"] * 2.0 * (m["Hp"] + m["Wp"] + 2) * C
        elif label == "gemm_fc1_gelu":
            bound, scale, unit = "tensor", 1e12, "TFLOP/s"
            tot += 2.0 * T * C * Hd
        elif label == "gemm_fc2":
            bound, scale, unit = "tensor", 1e12, "TFLOP/s"
            tot += 2.0 * T * Hd * C
        elif label == "layer_norm":
            bound, scale, unit = "hbm", 1e9, "GB/s"
            f_attn, f_all = _ln_fold(T)
            tot += (a * (not f_attn) + (cs + (Hd > 0)) * (not f_all)) * 4.0 * T * C    # bf16 row read + write
        elif label == "row_stats":       # folded LayerNorm: bf16 row read, (mu, rstd) written
            bound, scale, unit = "hbm", 1e9, "GB/s"
            f_attn, f_all = _ln_fold(T)
            tot += (a * f_attn + (cs + (Hd > 0)) * f_all) * T * (2.0 * C + 8.0)
        elif label == "ln_fold":         # weight fold of W_qkv (and W_in / W_fc1 when all are folded): W read, W' written
            bound, scale, unit = "hbm", 1e9, "GB/s"
            f_attn, f_all = _ln_fold(T)
            tot += a * f_attn * (4.0 * 3 * C * C + 8.0 * 3 * C) + f_all * (cs * 4.0 * 2 * D * C + (Hd > 0) * 4.0 * Hd * C)
        elif label == "conv_silu":
            bound, scale, unit = "hbm", 1e9, "GB/s"
            tot += cs * 4.0 * T * D                     # xin read + v write, bf16
        else:
            return None
    return (bound, tot, scale, unit) if bound and tot > 0 else None


def peaks():
    # MEASURED_PEAKS.json (driver-written) first; else this round's measured values as recorded in BASELINE.md §2;
    # else the B200_PROFILING.md fallback
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "BASELINE.md")) as f:
            txt = f.read()
        import re
        m = re.search(r"HBM ([0-9.]+) GB/s\.\n- bf16 dense ([0-9.]+) TF/s \(([0-9.]+) sustained\)", txt)
        if m:
            p.update(hbm_gbs=float(m.group(1)), bf16_tflops=float(m.group(2)),
                     bf16_tflops_sustained=float(m.group(3)), src="recorded")
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update(hbm_gbs=m["hbm_gbs"], bf16_tflops=m["bf16_tflops"],
                 bf16_tflops_sustained=m.get("bf16_tflops_sustained", m["bf16_tflops"]), src="measured",
                 sm_max_mhz=m.get("sm_max_mhz", 1965.0))
    except Exception:
        p["sm_max_mhz"] = 1965.0
    # MUFU ex2: the rate measured by tools/ubench/pipes.cu on a B200 (profiles/alu_peaks.json); else derived from
    # 16 / clk / SM x 148 SMs at the max SM clock
    p["ex2_gps"] = 16 * 148 * p["sm_max_mhz"] * 1e6 / 1e9
    p["ex2_src"] = "derived: 16 ex2/clk/SM x 148 SMs x max SM clock"
    try:
        with open(os.path.join(ROOT, "profiles", "alu_peaks.json")) as f:
            p["ex2_gps"] = float(json.load(f)["ex2_gps"])
            p["ex2_src"] = "measured: MUFU.EX2 rate, tools/ubench/pipes.cu (profiles/alu_peaks.json)"
    except Exception:
        pass
    return p


def traffic_table(workload="1024"):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum, one ncu --set full capture) by kernel
    label, for this workload: profiles/dram_traffic.json holds {workload: {label: bytes}} (a flat table = 1024^2)."""
    path = os.path.join(ROOT, "profiles", "dram_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
    except Exception:
        return {}
    if t and all(isinstance(v, dict) for v in t.values()):
        return t.get(str(workload), {})
    return t if str(workload) == "1024" else {}


# ----------------------------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.out = self.proc.communicate(timeout=5)[0]
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------------------------- ours
def _kind(layer):
    d = getattr(layer, "desc")
    if hasattr(d, "n_scales"):
        cs = {0: "", 1: "CS+", 2: "MSCS"}[d.cycle_scan]
        return cs + ("" if not d.attention else ("S" if d.layer.shift_x else "P"))
    return ("CS+" if d.cycle_scan else "") + ("S" if d.shift_x else "P")


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2407_02109_b200 as pl

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    layers = []
    if args.workload == "ms":
        label, B, specs = ms_workload()
        cfgs = [c for c, _, _, _ in specs]
        for cfg, att, cs, seed in specs:
            w = synth.make_weights(cfg, layer=seed)
            dw = {k: torch.tensor(v, dtype=torch.float32 if k in F32_KEYS else torch.bfloat16, device=dev)
                  for k, v in w.items()}
            layers.append(pl.PSCWinMSLayer(pl.MSDesc.make(cfg, MS_SCALES, att, cs), dw))
        # scale-outermost packing (Q20): [B, H_s, W_s, C] blocks of every scale back to back
        x_host = np.concatenate([synth.make_input(cfgs[0].replace(H=h, W=w), layer=8 * rank + i).reshape(-1, cfgs[0].C)
                                 for i, (h, w) in enumerate(MS_SCALES)])
    else:
        label, B, cfgs = workload(args.workload)
        for i, cfg in enumerate(cfgs):
            w = synth.make_weights(cfg, layer=i)
            dw = {k: torch.tensor(v, dtype=torch.float32 if k in F32_KEYS else torch.bfloat16, device=dev)
                  for k, v in w.items()}
            layers.append(pl.PSCWinLayer(pl.LayerDesc.from_config(cfg), dw))
        x_host = synth.make_input(cfgs[0], layer=rank)
    x0 = torch.tensor(x_host, dtype=torch.bfloat16, device=dev)
    bufs = [torch.empty_like(x0), torch.empty_like(x0)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # the public API's multi-layer step: all kernels of all layers captured once into a CUDA graph
    stack = pl.PSCWinStack(layers, tuple(x0.shape), device=dev, graph=not args.no_graph)
    stack.x_in.copy_(x0)

    def step(x=None):
        return stack.replay()

    def step_eager(x):
        cur = x
        for j, layer in enumerate(layers):
            nxt = bufs[j & 1]
            layer(cur, out=nxt)
            cur = nxt
        return cur

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed before each, CUDA events on the launching stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = stack.launches_per_step * args.steps  # library kernels per step (graph nodes) x steps
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    per_step = [a.elapsed_time(b) for a, b in ev]

    # ---- L2-warm context (untimed for value): the same step back to back without the flush (at 1024^2 the
    # whole working set, ~100 MB, can stay in the 126 MB L2; at 4096^2 it cannot)
    warm = []
    for _ in range(max(3, min(20, args.steps))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        torch.cuda.synchronize()
        warm.append(a.elapsed_time(b))
    l2_warm_ms = float(np.median(warm))

    # ---- per-layer breakdown (untimed for value): each layer timed alone after an L2 flush
    layer_ms = []
    for j, layer in enumerate(layers):
        ts = []
        for _ in range(max(3, min(20, args.steps))):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            layer(x0, out=bufs[0])
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        layer_ms.append(float(np.median(ts)))

    # ---- e2e: public API with pinned host buffers, copies inside the timed region. A job of K steps: every step's
    # input is copied H2D from pinned host memory and its result D2H back; PSCWinStack.run_job overlaps the copies of
    # neighbouring steps with the compute of the current one (two copy streams, double-buffered staging), L2 flushed
    # before each step's compute; timed from the first copy to the last on the device (whole-job throughput)
    x_pin = torch.empty(x0.shape, dtype=torch.bfloat16, pin_memory=True)
    x_pin.copy_(x0.cpu())
    xs_pin = [x_pin] + [x_pin.clone().pin_memory() for _ in range(min(args.steps, 2) - 1)]
    ys_pin = [torch.empty_like(x_pin).pin_memory() for _ in range(min(args.steps, 2))]
    xs_job = [xs_pin[i % len(xs_pin)] for i in range(args.steps)]
    ys_job = [ys_pin[i % len(ys_pin)] for i in range(args.steps)]
    stack.run_job(xs_job[:2], ys_job[:2], before_step=lambda i: flush.zero_())  # warm the copy streams
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    stack.run_job(xs_job, ys_job, before_step=lambda i: flush.zero_())
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    # the unpipelined sequence (copy in, compute, copy out per step), for context
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        e2e_ev[i][0].record(stream)
        out = stack(x_pin)                        # H2D copy into the static input + graph replay
        ys_pin[0].copy_(out, non_blocking=True)   # D2H of the result
        e2e_ev[i][1].record(stream)
    torch.cuda.synchronize()
    e2e_serial_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)

    # ---- per-kernel timing (library CUDA events on the launching stream), separate pass
    pl.profile_enable(True)
    for i in range(args.steps):
        flush.zero_()
        # park the stream ~1 ms so the host enqueues the whole eager step before the GPU reaches it: the per-kernel
        # events then time back-to-back kernels, not host launch latency
        torch.cuda._sleep(2_000_000)
        step_eager(x0)
    torch.cuda.synchronize()
    prof = pl.profile_read()
    pl.profile_enable(False)

    # ---- max over ranks
    if world > 1:
        t = torch.tensor([total_ms, e2e_ms, e2e_serial_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, e2e_ms, e2e_serial_ms = float(t[0]), float(t[1]), float(t[2])
    images = args.steps * B * world
    result = dict(total_ms=total_ms, e2e_ms=e2e_ms, e2e_serial_ms=e2e_serial_ms, images=images, per_step=per_step,
                  layer_ms=layer_ms,
                  l2_warm_ms=l2_warm_ms,
                  prof=prof, launches=launches, clocks=clk.summary(), label=label, B=B, cfgs=cfgs,
                  kinds=[_kind(l) for l in layers],
                  h2d=x0.numel() * 2 * B // B, d2h=x0.numel() * 2)
    return result


def roofline(res, args):
    pk = peaks()
    steps = args.steps
    metas = layer_metas(args)
    rows = []
    total = max(sum(v[0] for v in res["prof"].values()), 1e-12)
    for lab, (ms, cnt) in res["prof"].items():
        per_launch = ms / max(cnt, 1)
        w = kernel_work(lab, metas)
        row = {"kernel": lab, "ms_per_launch": per_launch, "launches": cnt, "share": ms / total}
        if w:
            bound, amount, scale, unit = w
            achieved = amount * steps / (ms * 1e-3) / scale      # work of `steps` steps / time of their launches
            if bound == "hbm":
                peak = pk["hbm_gbs"]
            elif bound == "tensor":
                peak = pk["bf16_tflops"]
            else:
                peak = pk["ex2_gps"]
            row.update(bound=bound, achieved=achieved, peak=peak, unit=unit, frac=achieved / peak)
        rows.append(row)
    rows.sort(key=lambda r: -r["share"])
    dom = next((r for r in rows if "bound" in r), None)
    traffic = traffic_table("ms" if args.workload == "ms" else args.workload)
    out = None
    if dom:
        tr = traffic.get(dom["kernel"])
        src = {"measured": "of measured (MEASURED_PEAKS.json)", "recorded": "of measured (BASELINE.md §2 record)",
               "fallback": "of fallback (B200_PROFILING.md)"}[pk["src"]]
        out = {"kernel": dom["kernel"], "bound": dom["bound"], "achieved": round(dom["achieved"], 2),
               "peak": round(dom["peak"], 2), "unit": dom["unit"], "frac": round(dom["frac"], 4),
               "traffic": tr, "share_of_step": round(dom["share"], 4),
               "peak_src": src if dom["bound"] != "alu" else pk["ex2_src"]}
    return out, rows


def attention_sublayer_roofline(res, args):
    """The north-star attention target (">= 60 % of B200 dense-bf16 tensor peak in attention") graded on the attention
    SUB-LAYER: LN1 + QKV GEMM (+ RoPE) + pad work + window attention + out-proj with residual, timed per layer with
    CUDA events (eager, L2 flushed) on the layers that have no cycle-scan module and no FFN. Algorithmic FLOPs per
    token: QKV 2*C*3C, out-proj 2*C*C, attention 4*w^2*C (QK^T and PV over the w^2 slots of the token's window)."""
    if args.workload == "ms":
        return None
    pk = peaks()
    cfgs, layer_ms = res["cfgs"], res["layer_ms"]
    out = {}
    for name, want_shift in (("P", False), ("S", True)):
        ts = [t for c, t in zip(cfgs, layer_ms)
              if not c.cycle_scan and not c.mlp_hidden and bool(c.shift_x or c.shift_y) == want_shift]
        if not ts:
            continue
        c = next(c for c in cfgs if not c.cycle_scan and bool(c.shift_x or c.shift_y) == want_shift)
        T = c.B * c.H * c.W
        flops = T * (2.0 * c.C * 3 * c.C + 2.0 * c.C * c.C + 4.0 * c.window ** 2 * c.C)
        ms = float(np.median(ts))
        tf = flops / (ms * 1e-3) / 1e12
        out[name] = {"ms": round(ms, 4), "gflop": round(flops / 1e9, 2), "tflops": round(tf, 1),
                     "frac": round(tf / pk["bf16_tflops"], 4)}
    if not out:
        return None
    return {"unit": "TFLOP/s", "peak": pk["bf16_tflops"], "peak_src": "of measured (MEASURED_PEAKS.json, burst)",
            "scope": "LN1 + QKV/RoPE + pad + window attention + out-proj + residual, per layer", **out}


def scan_roofline(rows):
    """Scan passes against the measured MUFU ex2 rate (one ex2 per (token, channel, state) per pass) and the dt /
    x_proj / conv steps against HBM (north-star scan target: ">= 70 % of HBM peak in the scan")."""
    pk = peaks()
    out = {}
    for r in rows:
        if r["kernel"] in ("scan_pass1", "scan_pass2", "scan_dt", "gemm_x_proj", "conv_silu", "scan_carry") \
                and "frac" in r:
            out[r["kernel"]] = {"ms_per_launch": round(r["ms_per_launch"], 4), "achieved": round(r["achieved"], 1),
                                "unit": r["unit"], "frac": round(r["frac"], 4)}
    if not out:
        return None
    out["ex2_peak_gps"] = pk["ex2_gps"]
    out["hbm_peak_gbs"] = pk["hbm_gbs"]
    return out


# ----------------------------------------------------------------------------------------------- oracle (CPU)
def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def time_oracle_layer(cfg, layer_idx):
    import oracle
    x = synth.make_input(cfg, layer=0)
    w = synth.make_weights(cfg, layer=layer_idx)
    t0 = time.perf_counter()
    oracle.pscwin_layer(x, w, cfg)
    return time.perf_counter() - t0


def run_rows(args, rank, world, local_rank):
    """--shard rows: ONE image split by window rows over the ranks (config 4; strong scaling). Each rank runs the
    band phases of every layer (paper_2407_02109_b200.bands) and exchanges halo rows / conv history / scan
    records with its neighbours over NCCL (dist.TorchDistExchange). Eager launches (the exchanges sit between
    phases); time = max over ranks of the device-timed step."""
    import torch
    import paper_2407_02109_b200 as pl
    from paper_2407_02109_b200.bands import BandLayer, band_forward
    from paper_2407_02109_b200.dist import TorchDistExchange, band_rows

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    label, _, cfgs = workload(args.workload)
    cfgs = [c.replace(B=1) for c in cfgs]
    c0 = cfgs[0]
    r0, r1 = band_rows(c0.H, c0.window, world)[rank]
    if world == 1:
        import torch.distributed as tdist
        if not tdist.is_initialized():
            tdist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % _free_port(), rank=0, world_size=1)
    exchange = TorchDistExchange()
    lib_nccl = args.exchange == "nccl-lib"
    comm = None
    if lib_nccl:
        from paper_2407_02109_b200.bands import DistLayer, NcclComm
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")  # one node: bootstrap over loopback (data over NVLink)
        comm = NcclComm(rank, world)
    layers = []
    for i, cfg in enumerate(cfgs):
        w = synth.make_weights(cfg, layer=i)
        dw = {k: torch.tensor(v, dtype=torch.float32 if k in F32_KEYS else torch.bfloat16, device=dev)
              for k, v in w.items()}
        if lib_nccl:
            layers.append(DistLayer(pl.LayerDesc.from_config(cfg), dw, r0, r1, comm))
        else:
            layers.append(BandLayer(pl.LayerDesc.from_config(cfg), dw, r0, r1, rank, world))
    x_full = synth.make_input(cfgs[0], layer=0)
    xb = torch.tensor(x_full[:, r0:r1], dtype=torch.bfloat16, device=dev).contiguous()
    bufs = [torch.empty_like(xb), torch.empty_like(xb)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step_eager(x):
        cur = x
        for j, layer in enumerate(layers):
            nxt = bufs[j & 1]
            if lib_nccl:
                layer(cur, out=nxt)
            else:
                band_forward(layer, cur, exchange, out=nxt)
            cur = nxt
        return cur

    graph = None
    xstatic = torch.empty_like(xb)
    if lib_nccl:  # kernels and NCCL exchanges of the whole step in one CUDA graph
        xstatic.copy_(xb)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step_eager(xstatic)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            gout = step_eager(xstatic)

    def step(x):
        if graph is None:
            return step_eager(x)
        if x is not xstatic:
            xstatic.copy_(x, non_blocking=True)
        graph.replay()
        return gout

    for _ in range(args.warmup):
        step(xb)
    torch.cuda.synchronize()
    n0 = pl.launch_count()
    step_eager(xb)
    torch.cuda.synchronize()
    launches_per_step = pl.launch_count() - n0
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    exchange.dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step(xb)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    # e2e: pinned host band in, band result out, inside the timed region
    x_pin = torch.empty(xb.shape, dtype=torch.bfloat16, pin_memory=True)
    x_pin.copy_(xb.cpu())
    y_pin = torch.empty_like(x_pin).pin_memory()
    xin = torch.empty_like(xb)
    e2e = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    exchange.dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        e2e[i][0].record(stream)
        xin.copy_(x_pin, non_blocking=True)
        y = step(xin)
        y_pin.copy_(y, non_blocking=True)
        e2e[i][1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e)
    if world > 1:
        t = torch.tensor([total_ms, e2e_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, e2e_ms = float(t[0]), float(t[1])
    return dict(total_ms=total_ms, e2e_ms=e2e_ms, images=args.steps, launches=launches_per_step * args.steps,
                clocks=clk.summary(), label=label, cfgs=cfgs, band=(r0, r1), h2d=xb.numel() * 2,
                d2h=xb.numel() * 2)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def tiny_single_thread_ms() -> float:
    """configs[0] (tiny 16x16, dim 64) through the oracle's CS+S layer on ONE thread (SURVEY §8(d) baseline)."""
    from threadpoolctl import threadpool_limits
    cfg = synth.tiny(cycle_scan=1)
    with threadpool_limits(1):
        return round(1e3 * time_oracle_layer(cfg, 0), 1)


def cpu_baseline(args):
    """The fp64 oracle as it stands, timed on this host: one image through one layer of each kind (summed per
    image) — or, for the multi-scale workload, each bounded oracle piece of one sample timed once and scaled.
    Adds the host CPU model and the single-thread time of the tiny configuration's CS+S layer."""
    out = _cpu_baseline(args)
    out["cpu_model"] = cpu_model()
    out["tiny_cs_s_layer_1thread_ms"] = tiny_single_thread_ms()
    return out


def _cpu_baseline(args):
    if args.workload != "1024":
        items = reference_items(reference_entries(args))
        tot = 0.0
        for name, fn, scale in items:
            t0 = time.perf_counter()
            fn()
            tot += (time.perf_counter() - t0) * scale
        what = "sample" if args.workload == "ms" else "image"
        return {"value": round(1e3 * tot, 1), "unit": "ms/image", "cores": oracle_threads(), "kind": "oracle",
                "sample": f"one {what}; {len(items)} bounded oracle pieces (1/16 of the projection rows, one window "
                          f"row per attention kind, 1/16 (1/64 at 4096^2) of the 3L scan tokens) timed once each and "
                          f"scaled to the full stack"}
    label, B, cfgs = workload(args.workload)
    one = [c.replace(B=1) for c in cfgs]
    kinds = {}
    for i, c in enumerate(one):
        key = (c.shift_x != 0, c.cycle_scan)
        kinds.setdefault(key, []).append(i)
    t_kind = {k: time_oracle_layer(one[idx[0]], idx[0]) for k, idx in kinds.items()}
    ms_per_image = 1e3 * sum(t_kind[k] * len(idx) for k, idx in kinds.items())
    sample = (f"one image; one layer of each kind timed once ({', '.join(f'{len(v)}x' for v in kinds.values())}) "
              f"summed over the {len(one)} layers")
    return {"value": round(ms_per_image, 1), "unit": "ms/image", "cores": oracle_threads(), "kind": "oracle",
            "sample": sample}


def reference_entries(args):
    """(cfg, attention repeats, cycle-scan repeats) per distinct piece of one image / sample of the workload."""
    if args.workload == "ms":
        ents = []
        for h, w in MS_SCALES:
            base = synth.vitb(h, B=1, H=h, W=w, mlp_hidden=FFN_HIDDEN)
            ents += [(base.replace(shift_x=0, shift_y=0), 6, 0), (base, 6, 0),
                     (base.replace(shift_x=0, shift_y=0, cycle_scan=1), 0, 4)]      # single-scale modules
        Lt = sum(h * w for h, w in MS_SCALES)
        ents.append((synth.vitb(64, B=1, H=1, W=Lt, shift_x=0, shift_y=0, cycle_scan=1), 0, 4))  # multi-scale
        return ents
    _, _, cfgs = workload(args.workload)
    # one entry per distinct piece (the oracle's cost of a piece depends only on its kind): plain attention,
    # shifted attention, cycle-scan module, each with its repeat count in the stack
    ents = {}
    for c in cfgs:
        one = c.replace(B=1, cycle_scan=0)
        ents.setdefault(("att", one.shift_x), [one, 0, 0])[1] += 1
        if c.cycle_scan:
            ents.setdefault(("cs",), [c.replace(B=1, shift_x=0, shift_y=0), 0, 0])[2] += 1
    return [tuple(v) for v in ents.values()]


def reference_items(entries):
    """The reference arm's bounded samples: every layer split into oracle pieces, each timed on a sample of its
    independent units and scaled back up (projections: 1/16 of the token rows; window attention: one window
    row of the padded grid; cycle-scan SSM: the sequential recurrence over the first 1/16 of the 3L tokens,
    all channels — the oracle's cost per token row / window row / scan token is uniform, so each sample times
    a fixed fraction of the layer's work). entries: (cfg, attention repeats, cycle-scan repeats)."""
    import oracle
    items = []
    for j, (c, na, ncs) in enumerate(entries):
        x = synth.make_input(c, layer=0)
        w = synth.make_weights(c, layer=j)
        T = c.H * c.W
        if na:
            rows = np.arange(0, T, 16)
            xr = x.reshape(T, c.C)[rows]

            def proj(xr=xr, w=w, c=c):
                u = oracle.layer_norm(xr, w["ln1_g"], w["ln1_b"], c.ln_eps)
                qkv = u @ w["w_qkv"].T + w["b_qkv"]
                _ = w["pad"] @ w["w_qkv"].T + w["b_qkv"]
                return qkv[:, :c.C] @ w["w_o"].T + w["b_o"]
            items.append((f"E{j} ln+qkv+out-proj", proj, na * T / len(rows)))
            u = oracle.layer_norm(x, w["ln1_g"], w["ln1_b"], c.ln_eps)
            qkv = u @ w["w_qkv"].T + w["b_qkv"]
            qkv_p = w["pad"] @ w["w_qkv"].T + w["b_qkv"]
            pt, _, pb, _ = oracle.shifted_geometry(c.H, c.W, c.window, c.shift_x, c.shift_y)
            nwy = (c.H + pt + pb) // c.window

            def attn(qkv=qkv, qkv_p=qkv_p, c=c, nwy=nwy):
                return oracle.attention_core_padded(qkv, qkv_p, c.H, c.W, c.heads, c.window, c.shift_x, c.shift_y,
                                                    c.pad_mode, c.rope, window_rows=[nwy // 2])
            items.append((f"E{j} window attention", attn, na * nwy))
            if c.mlp_hidden:
                def ffn(xr=xr, w=w, c=c):
                    return oracle.ffn_sublayer(xr, w, c)
                items.append((f"E{j} FFN", ffn, na * T / len(rows)))
        if ncs:
            L, D = T, c.D
            frac = 16 if L <= 16384 else 64      # the SSM sample: 1/16 (1/64 at 4096^2) of the 3L tokens
            rows3 = np.arange(0, 3 * L, 16)

            def cs_proj(x=x, w=w, c=c, rows3=rows3, L=L):
                u0 = oracle.layer_norm(x, w["lns_g"], w["lns_b"], c.ln_eps).reshape(L, c.C)
                X3 = np.concatenate([u0, u0, u0])[rows3]
                xz = X3 @ w["w_in"].T
                return xz[:, :c.D] @ w["w_out"].T
            items.append((f"E{j} cycle-scan LN+in/out-proj", cs_proj, ncs * 3 * L / len(rows3)))
            u0 = oracle.layer_norm(x, w["lns_g"], w["lns_b"], c.ln_eps).reshape(L, c.C)
            n3 = 3 * L // frac
            xz = np.concatenate([u0, u0, u0])[:n3] @ w["w_in"].T

            def cs_ssm(xz=xz, w=w, c=c, D=D):  # the recurrence over the first 1/frac of the 3L tokens
                return oracle.cycle_ssm_3L(xz[:, :D], xz[:, D:], w, c.bbar_mode)
            items.append((f"E{j} cycle-scan SSM", cs_ssm, ncs * 3 * L / n3))
    return items


def run_reference(args):
    """--impl reference: the fp64 oracle timed as the reference arm, same metric/config. Each step runs one
    bounded sample (reference_items, round-robin) so any --steps K finishes in minutes; value = sum over the
    pieces of (mean sample time x its scale) = oracle ms per image."""
    label = ms_workload()[0] if args.workload == "ms" else workload(args.workload)[0]
    items = reference_items(reference_entries(args))
    for i in range(max(args.warmup, 1)):
        items[i % len(items)][1]()
    times = {}
    t0 = time.perf_counter()
    for i in range(max(args.steps, len(items))):
        name, fn, _ = items[i % len(items)]
        t1 = time.perf_counter()
        fn()
        times.setdefault(name, []).append(time.perf_counter() - t1)
    wall = time.perf_counter() - t0
    n_run = max(args.steps, len(items))
    ms_img = 1e3 * sum(np.mean(times[name]) * scale for name, _, scale in items)
    cores = oracle_threads()
    sample = (f"{n_run} steps round-robin over {len(items)} oracle pieces of one image (projections on 1/16 of "
              f"the token rows, attention on one window row per attention kind, the SSM on 1/16 (1/64 at 4096^2) of "
              f"the 3L tokens), each scaled to its repeats in the full stack")
    line = {"metric": METRIC, "value": round(ms_img, 2), "unit": "ms/image", "n_gpus": 0, "steps": n_run,
            "warmup": args.warmup, "ms_per_step": round(1e3 * wall / max(n_run, 1), 2),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": label, "images_per_rank": 1, "pieces": len(items)},
            "cpu_baseline": {"value": round(ms_img, 2), "unit": "ms/image", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(ms_img, 2), "unit": "ms/image", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------- ablation
# Table 3 as a B200 rendition: the 12-block ViT-B encoder body (attention +
# FFN 768x4 per block) with each attention / cycle-scan combination the paper ablates, one image, bf16.
# Patch embedding and the neck are not part of the timed body. The paper's latencies (unstated GPU) are context.
PAPER_TABLE3 = {  # variant -> (1024^2 ms, 2048^2 ms)
    "Global": (104, 1338), "Global+PlainWin": (61, 528), "PlainWin+VanSwin": (37, 122),
    "PlainWin+PadSwin": (44, 136), "PlainWin+VanSwin+SSCScan": (52, 178),
    "PlainWin+PadSwin+SSCScan (HRSAM)": (58, 192), "PlainWin+PadSwin+SSCScan+MSCScan (HRSAM++)": (98, 277)}


def ablation_specs(side: int, variant: str):
    """[(kind, cfg, attention, cs_mode)] for one encoder variant on a side x side token grid."""
    out = []
    for i in range(12):
        shifted, cs = synth.stack_layer_kind(i)
        base = synth.vitb(side, mlp_hidden=3072)
        if variant == "Global":
            cfg, csm = base.replace(window=side, shift_x=0, shift_y=0), 0
        elif variant == "Global+PlainWin":  # SAM-style: global attention in blocks 2, 5, 8, 11
            cfg = base.replace(window=side, shift_x=0, shift_y=0) if cs else base.replace(shift_x=0, shift_y=0)
            csm = 0
        else:
            pad = synth.PAD_MASKED if "VanSwin" in variant else synth.PAD_LEARNABLE
            cfg = base.replace(shift_x=8 if shifted else 0, shift_y=8 if shifted else 0, pad_mode=pad)
            csm = 1 if (cs and "SSCScan" in variant) else 0
        out.append(("ms" if "MSCScan" in variant else "layer", cfg, 1, csm))
        if cs and "MSCScan" in variant:
            out.append(("ms", base.replace(shift_x=0, shift_y=0), 0, 2))
    return out


def run_ablation(args):
    import torch
    import paper_2407_02109_b200 as pl
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    rows = []
    for side in (64, 128):
        for variant, paper in PAPER_TABLE3.items():
            specs = ablation_specs(side, variant)
            scales = [(side, side), (32, 32)]   # HRSAM++: the 512^2 overview image -> 32 x 32 tokens
            layers = []
            for j, (kind, cfg, att, csm) in enumerate(specs):
                w = synth.make_weights(cfg, layer=j)
                dw = {k: torch.tensor(v, dtype=torch.float32 if k in F32_KEYS else torch.bfloat16, device=dev)
                      for k, v in w.items()}
                if kind == "ms":
                    layers.append(pl.PSCWinMSLayer(pl.MSDesc.make(cfg, scales, att, csm), dw))
                else:
                    layers.append(pl.PSCWinLayer(pl.LayerDesc.from_config(cfg.replace(cycle_scan=csm)), dw))
            T = side * side + (32 * 32 if "MSCScan" in variant else 0)
            shape = (T, 768) if "MSCScan" in variant else (1, side, side, 768)
            stack = pl.PSCWinStack(layers, shape, device=dev, graph=True)
            stack.x_in.copy_(torch.randn(shape, device=dev).to(torch.bfloat16))
            for _ in range(3):
                stack.replay()
            ts = []
            for _ in range(max(3, min(args.steps, 20))):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                stack.replay()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = float(np.median(ts))
            res = {"metric": "encoder body latency ms/image (Table 3 rendition)", "variant": variant,
                   "input": f"{16 * side}^2", "value": round(ms, 4), "unit": "ms/image",
                   "paper_ms_context": paper[0 if side == 64 else 1], "dtype": "bf16", "data": "synthetic",
                   "config": {"blocks": 12, "ffn": 3072, "launches_per_step": stack.launches_per_step}}
            print(json.dumps(res), flush=True)
            rows.append(res)
            del stack, layers
            torch.cuda.empty_cache()
    print("| variant | input | B200 ms | paper ms (GPU unstated) |\n|---|---|---|---|", file=sys.stderr)
    for r in rows:
        print(f"| {r['variant']} | {r['input']} | {r['value']:.3f} | {r['paper_ms_context']} |", file=sys.stderr)


# ----------------------------------------------------------------------------------------------- encoder
def run_encoder(args):
    """--encoder: the whole HRSAM encoder on one image: patch embedding -> the 12-block stack with FFN
    (global alternation, cycle scan before blocks 2, 5, 8, 11) -> fusion of the four stage outputs (neck) ->
    [H/16, W/16, 256] embeddings. One CUDA graph; the image [1, 3, 16H, 16W] is resident (value)
    or copied from pinned host memory with the embedding copied back (e2e)."""
    import torch
    import paper_2407_02109_b200 as pl
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    side = {"1024": 64, "2048": 128, "4096": 256}[args.workload]
    todev = lambda w: {k: torch.tensor(v, dtype=torch.float32 if k in F32_KEYS else torch.bfloat16, device=dev)  # noqa
                       for k, v in w.items()}
    layers, stage_ends = [], [2, 5, 8, 11]
    scales = [(side, side)] + ([(OVERVIEW, OVERVIEW)] if args.overview else [])
    if args.overview:
        # HRSAM++ (P:L174-189): the 512^2 overview image (32 x 32 tokens) packed after the main grid; blocks
        # with a single-scale cycle scan, each stage closed by a multi-scale cycle-scan module (as --workload ms)
        stage_ends = []
        for i in range(12):
            shifted, cs = synth.stack_layer_kind(i)
            cfg = synth.vitb(side, shift_x=8 if shifted else 0, shift_y=8 if shifted else 0, mlp_hidden=3072)
            layers.append(pl.PSCWinMSLayer(pl.MSDesc.make(cfg, scales, 1, 1 if cs else 0),
                                           todev(synth.make_weights(cfg, layer=i))))
            if cs:
                ms = synth.vitb(side, shift_x=0, shift_y=0)
                layers.append(pl.PSCWinMSLayer(pl.MSDesc.make(ms, scales, 0, 2),
                                               todev(synth.make_weights(ms, layer=100 + i))))
                stage_ends.append(len(layers) - 1)
    else:
        for i in range(12):
            shifted, cs = synth.stack_layer_kind(i)
            cfg = synth.vitb(side, shift_x=8 if shifted else 0, shift_y=8 if shifted else 0, cycle_scan=int(cs),
                             mlp_hidden=3072)
            layers.append(pl.PSCWinLayer(pl.LayerDesc.from_config(cfg), todev(synth.make_weights(cfg, layer=i))))
    ew = synth.make_ends_weights()
    ends = {k: torch.tensor(v, dtype=torch.float32 if v.ndim == 1 else torch.bfloat16, device=dev)
            for k, v in ew.items()}
    ends["w_neck_conv"] = ends["w_neck_conv"].permute(0, 2, 3, 1).contiguous()
    enc = pl.HRSAMEncoder(layers, ends, 1, side, side, stage_ends=stage_ends, graph=True, scales=scales)
    imgs = [torch.tensor(synth.make_image(1, h, w, seed=50 + i), dtype=torch.bfloat16, device=dev)
            for i, (h, w) in enumerate(scales)]
    img = imgs[0]
    for dst, src in zip(enc.imgs, imgs):
        dst.copy_(src)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        enc.graph.replay()
    torch.cuda.synchronize()
    ts = []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            enc.graph.replay()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ts) / args.steps
    img_pins = [im.cpu().pin_memory() for im in imgs]
    out_pin = torch.empty(enc.out.shape, dtype=torch.bfloat16).pin_memory()
    te = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        y = enc(img_pins)
        out_pin.copy_(y, non_blocking=True)
        b.record()
        te.append((a, b))
    torch.cuda.synchronize()
    e2e = sum(a.elapsed_time(b) for a, b in te) / args.steps
    name = "HRSAM++ encoder" if args.overview else "HRSAM encoder"
    line = {"metric": f"{name} latency ms/image (patch embedding + 12 blocks with FFN + neck)",
            "value": round(ms, 4), "unit": "ms/image", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic image and random-init weights",
            "config": {"workload": f"{16 * side}^2 image" + (f" + {16 * OVERVIEW}^2 overview (HRSAM++, multi-scale "
                                                             f"cycle scan closing each stage)" if args.overview else "")
                       + f" -> {side}x{side}x256 embeddings", "blocks": 12,
                       "ffn": 3072, "stage_ends": stage_ends, "launch": "CUDA graph",
                       "l2": "flushed before every timed step (256 MiB write)"},
            "e2e": {"value": round(e2e, 4), "unit": "ms/image", "h2d_bytes_per_step": int(sum(im.numel() * 2 for im in imgs)),
                    "d2h_bytes_per_step": int(enc.out.numel() * 2)},
            "gpu_launches": int(enc.launches_per_step * args.steps), "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------- micro
def run_partition_micro(args):
    """--micro partition: the standalone a5 / a7 data-movement entry points (pscwin_window_partition,
    pscwin_shifted_pad_partition, pscwin_window_merge with and without the residual) on a 4096^2 token grid
    (256 x 256, w = 16, s = 8) for the QKV width (Cx = 3C = 2304) and the model width (Cx = 768), L2 flushed
    before every launch, CUDA events on the launching stream. Algorithmic bytes: partition = grid read + every
    window slot written (pads included); merge = the real window rows read + the grid written (+ residual read).
    One JSON line per case (GB/s and fraction of the measured HBM copy bandwidth)."""
    import torch
    import paper_2407_02109_b200 as pl
    torch.cuda.set_device(0)
    pk = peaks()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    H = W = 256
    w, s_ = 16, 8

    def timed(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(max(5, min(args.steps, 50))):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    for Cx in (2304, 768):
        x = torch.randn(1, H, W, Cx, device="cuda").to(torch.bfloat16)
        pad = torch.randn(Cx, device="cuda").to(torch.bfloat16)
        res = torch.randn_like(x)
        grid = H * W * Cx * 2
        n_s = pl.window_count(H, W, w, s_, s_)
        win_p = pl.window_partition(x, w)
        win_s = pl.shifted_pad_partition(x, pad, w, s_, s_)
        cases = [("window_partition", lambda: pl.window_partition(x, w), 2 * grid),
                 ("shifted_pad_partition", lambda: pl.shifted_pad_partition(x, pad, w, s_, s_),
                  grid + n_s * w * w * Cx * 2),
                 ("window_merge", lambda: pl.window_merge(win_p, 1, H, W, w), 2 * grid),
                 ("window_merge_shifted_residual", lambda: pl.window_merge(win_s, 1, H, W, w, s_, s_, residual=res),
                  3 * grid)]
        for name, fn, nbytes in cases:
            ms = timed(fn)
            gbs = nbytes / (ms * 1e-3) / 1e9
            print(json.dumps({"micro": name, "grid": f"{H}x{W}", "Cx": Cx, "window": w, "shift": s_ if "shift" in name else 0,
                              "ms": round(ms, 4), "bytes": int(nbytes), "GB/s": round(gbs, 1),
                              "frac_hbm": round(gbs / pk["hbm_gbs"], 4), "peak_gbs": pk["hbm_gbs"],
                              "l2": "flushed before every launch"}), flush=True)


# ----------------------------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="4096", choices=["1024", "2048", "4096", "ms"],
                    help="4096: the north-star 12-layer stack on one 4096^2 image (configs[3], default); 1024: "
                         "HRSAM stage 1 (configs[1]); 2048: the 12-layer stack, batch 8 (configs[2]); ms: HRSAM++ "
                         "multi-scale (configs[4])")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--breakdown", action="store_true", help="also print the per-kernel table to stderr")
    ap.add_argument("--no-graph", action="store_true", help="launch layer by layer instead of a CUDA graph")
    ap.add_argument("--shard", default="images", choices=["images", "rows"],
                    help="images: each rank its own image(s) (weak scaling, default); rows: one image split by "
                         "window rows over the ranks with halo / scan-carry exchange (config 4, strong scaling)")
    ap.add_argument("--exchange", default="nccl-lib", choices=["nccl-lib", "torch"],
                    help="--shard rows: exchanges inside libpscwin over NCCL (pscwin_dist_forward, graph-captured) or "
                         "between the band phases via torch.distributed")
    ap.add_argument("--ablation", action="store_true",
                    help="Table 3 rendition: the 12-block encoder body per attention / cycle-scan variant at 1024^2 and "
                         "2048^2 (one JSON line per variant; SURVEY NEXT-4)")
    ap.add_argument("--overview", action="store_true",
                    help="with --encoder: HRSAM++ (the 512^2 overview image packed with the main grid)")
    ap.add_argument("--encoder", action="store_true",
                    help="the whole HRSAM encoder on one image: patch embedding + 12 blocks with FFN + neck (NEXT-3)")
    ap.add_argument("--micro", choices=["partition"], help="micro-benchmark of one standalone entry point family")
    ap.add_argument("--ffn", action="store_true",
                    help="add the FFN sub-layer (hidden 768 x 4, P:L625; SURVEY NEXT-2) after every attention sub-layer")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    global FFN_HIDDEN
    FFN_HIDDEN = 3072 if args.ffn else 0

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` without a launcher: re-run under torch.distributed.run with one rank per GPU (the
        # driver's own launch is the same command, already under torchrun)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
        raise SystemExit(subprocess.call(cmd + sys.argv[1:]))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; running {world} rank(s)", file=sys.stderr)

    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return
    if args.ablation:
        if rank == 0:
            run_ablation(args)
        return
    if args.encoder:
        if rank == 0:
            run_encoder(args)
        return
    if args.micro:
        if rank == 0:
            run_partition_micro(args)
        return

    if world > 1:
        import torch
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")  # one node (the contract): bootstrap over loopback
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.shard == "rows":
        if args.workload == "ms":
            raise SystemExit("--shard rows splits one image (config 4); the multi-scale workload shards by sample")
        res = run_rows(args, rank, world, local_rank)
        if rank == 0:
            c0 = res["cfgs"][0]
            line = {
                "metric": METRIC, "value": round(res["total_ms"] / res["images"], 4), "unit": "ms/image",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(res["total_ms"] / args.steps, 4), "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded splitmix64; random-init ViT-B PSCWin weights)",
                "config": {"workload": res["label"].replace("one image per GPU", f"one image split by window rows "
                                                             f"over {world} GPU(s)"),
                           "grid": f"{c0.H}x{c0.W}", "layers": len(res["cfgs"]),
                           "parallelism": f"window-row bands x{world} (halo + scan-carry exchange)",
                           "rank0_band_rows": list(res["band"]),
                           "l2": "flushed before every timed step (256 MiB write)",
                           "exchange": args.exchange,
                           "launch": "CUDA graph (kernels + NCCL)" if args.exchange == "nccl-lib" else "eager"},
                "e2e": {"value": round(res["e2e_ms"] / res["images"], 4), "unit": "ms/image",
                        "h2d_bytes_per_step": int(res["h2d"]), "d2h_bytes_per_step": int(res["d2h"])},
                "gpu_launches": int(res["launches"]), "clocks": res["clocks"], "roofline": None}
            print(json.dumps(line), flush=True)
        if world > 1:
            import torch
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return
    res = run_ours(args, rank, world, local_rank)
    if rank == 0:
        rl, rows = roofline(res, args)
        ms_img = res["total_ms"] / res["images"]
        e2e_img = res["e2e_ms"] / res["images"]
        c0 = res["cfgs"][0]
        line = {
            "metric": METRIC, "value": round(ms_img, 4), "unit": "ms/image", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(res["total_ms"] / args.steps, 4),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded splitmix64; random-init ViT-B PSCWin weights)",
            "config": {"workload": res["label"],
                       "grid": ("+".join(f"{h}x{w}" for h, w in MS_SCALES) if args.workload == "ms"
                                else f"{c0.H}x{c0.W}"),
                       "images_per_rank": res["B"], "layers": res["kinds"],
                       "C": c0.C, "heads": c0.heads, "window": c0.window, "shift": 8, "ssm_state": c0.N,
                       "ssm_expand": c0.ssm_expand, "pad_mode": "learnable", "parallelism": f"images x{world}",
                       "l2": "flushed before every timed step (256 MiB write)",
                       "l2_warm_ms_per_image": round(res["l2_warm_ms"] / res["B"], 4),
                       "launch": "eager" if args.no_graph else "CUDA graph of the whole step",
                       "per_layer_ms": [round(t, 4) for t in res["layer_ms"]]},
            "e2e": {"value": round(e2e_img, 4), "unit": "ms/image", "h2d_bytes_per_step": int(res["h2d"]),
                    "d2h_bytes_per_step": int(res["d2h"]),
                    "how": "K-step job, each step's input H2D from pinned host memory and result D2H inside the timed "
                           "region; copies of neighbouring steps overlapped with compute (PSCWinStack.run_job)",
                    "unpipelined_value": round(res["e2e_serial_ms"] / res["images"], 4)},
            "gpu_launches": int(res["launches"]),
            "clocks": res["clocks"],
            "roofline": rl,
            "attention_sublayer": attention_sublayer_roofline(res, args),
            "scan": scan_roofline(rows),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args)
        if args.breakdown:
            for r in rows:
                print(json.dumps({k: (round(v, 5) if isinstance(v, float) else v) for k, v in r.items()}),
                      file=sys.stderr)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
