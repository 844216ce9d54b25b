"""Run one attention layer with PSCWIN_ATTN_TIMELINE and print per-CTA phase timings (debug).

    python tools/attn_timeline.py [side=64]      # ViT-B, side x side token grid, plain and shifted layers
Events per CTA (globaltimer ns): loader = item load issued; mma = S issued / PV issued; wg0/wg1 = S ready,
max done, P written, O ready, O stored (per q-tile slot)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
path = "/tmp/attn_tl.bin"
if os.path.exists(path): os.remove(path)
os.environ["PSCWIN_ATTN_TIMELINE"] = path
import torch, synth
import paper_2407_02109_b200 as pl
from gpu_util import dev
side = int(sys.argv[1]) if len(sys.argv) > 1 else 64
for shift in (0, 8):
    cfg = synth.vitb(side, shift_x=shift, shift_y=shift)
    qkv = dev(synth.make_qkv(cfg)); qp = dev(synth.make_pad_qkv(cfg), "f32")
    d = pl.LayerDesc.from_config(cfg)
    for _ in range(3):
        pl.window_attention(d, qkv, qp)
    torch.cuda.synchronize()
raw = np.fromfile(path, dtype=np.uint64).reshape(-1, 148, 128).astype(np.int64)
for run in (2, 5):
    t = raw[run]
    t0 = t[t > 0].min()
    print(f"--- run {run} (shift {'8' if run >= 3 else '0'}), kernel span {(t[t>0].max()-t0)/1e3:.1f} us")
    for cta in (0, 1, 100, 147):
        row = t[cta]
        def ev(base):
            v = row[base:base + 32]; v = v[v > 0]; return ((v - t0) / 1e3).round(2).tolist()
        print(f"cta {cta}: load {ev(0)[:12]}\n   mma {ev(32)[:12]}\n   wg0 {ev(64)[:12]}\n   wg1 {ev(96)[:12]}")
    # steady-state per-item spacing of slot 0's "S ready" events (every 4th wg0 event), median over CTAs
    gaps = []
    for cta in range(148):
        v = np.sort(t[cta][64:96]); v = v[v > 0]
        if len(v) >= 12:
            s = v[::5]
            gaps.append(np.median(np.diff(s)) / 1e3)
    if gaps:
        print(f"median per-item period (slot 0): {np.median(gaps):.2f} us over {len(gaps)} CTAs")
    # median phase durations of slot 0: S ready -> max done -> P written -> O ready -> O stored -> next S ready
    ph = [[] for _ in range(5)]
    for cta in range(148):
        v = np.sort(t[cta][64:96]); v = v[v > 0]
        for i in range(0, len(v) - 5, 5):
            for k in range(5):
                ph[k].append((v[i + k + 1] - v[i + k]) / 1e3)
    names = ["max pass", "exp pass", "PV wait", "O readout+store", "to next S"]
    print("slot-0 phase medians (us): " + ", ".join(f"{n} {np.median(x):.2f}" for n, x in zip(names, ph) if x))
