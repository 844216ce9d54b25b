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
row2 = os.environ.get("PSCWIN_ATTN_ROW2") == "1"
names = ["S->max", "max->turn", "exp", "P->O", "O->end", "end->nextS"]
for run in (2, 5):
    t = raw[run]
    t0 = t[t > 0].min()
    print(f"--- run {run} (shift {'8' if run >= 3 else '0'}), kernel span {(t[t>0].max()-t0)/1e3:.1f} us")
    if row2:
        continue
    # ROW1: slot a's events of its k-th item at 64 + 32a + (k % 5) * 6 + e, e = S ready, max done, exp turn,
    # P written, O ready, end
    for a in (0, 1):
        ph = [[] for _ in range(6)]
        per = []
        for cta in range(148):
            ev = t[cta][64 + 32 * a: 64 + 32 * a + 30].reshape(5, 6)
            ok = [i for i in range(5) if np.all(ev[i] > 0)]
            items = sorted(ok, key=lambda i: ev[i][0])
            for j, i in enumerate(items):
                for e in range(5):
                    ph[e].append((ev[i][e + 1] - ev[i][e]) / 1e3)
                if j + 1 < len(items):
                    nxt = ev[items[j + 1]][0]
                    ph[5].append((nxt - ev[i][5]) / 1e3)
                    per.append((nxt - ev[i][0]) / 1e3)
        clk = t[:, 64 + 32 * a + 30].astype(np.float64)
        ns = t[:, 64 + 32 * a + 31].astype(np.float64)
        ok = (clk > 0) & (ns > 0)
        if ok.any():
            print(f"slot {a}: last exp pass {np.median(clk[ok]):.0f} SM clocks in {np.median(ns[ok]):.0f} ns "
                  f"-> {np.median(clk[ok] / ns[ok]) * 1e3:.0f} MHz effective")
        print(f"slot {a}: period {np.median(per):.2f} us; phase medians: " +
              ", ".join(f"{n} {np.median(x):.2f}" for n, x in zip(names, ph) if x))
