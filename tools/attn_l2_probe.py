"""Window attention with L2-cold vs L2-warm QKV (is the kernel bound by where its operands come from?):
    python tools/attn_l2_probe.py   (ViT-B, plain and shifted, 128^2 and 256^2 token grids)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2407_02109_b200 as pl  # noqa: E402
from paper_2407_02109_b200.api import Workspace, workspace_bytes  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, cold):
    if cold:
        flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1000


for side in (128, 256):
    for shift in (0, 8):
        cfg = synth.vitb(side, shift_x=shift, shift_y=shift)
        d = pl.LayerDesc.from_config(cfg)
        qkv = (torch.randn(side * side, 3 * 768, device="cuda") * 0.5).to(torch.bfloat16)
        qp = torch.randn(3 * 768, device="cuda")
        out = torch.empty(side * side, 768, device="cuda", dtype=torch.bfloat16)
        ws = Workspace(workspace_bytes(d), qkv.device)
        fn = lambda: pl.window_attention(d, qkv, qp, ws=ws, out=out)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        cold = min(timed(fn, True) for _ in range(5))
        warm = min(timed(fn, False) for _ in range(5))
        mb = qkv.numel() * 2 / 1e6
        print(f"grid {side}^2 shift {shift}: qkv {mb:.0f} MB  cold {cold:.1f} us  warm {warm:.1f} us", flush=True)
