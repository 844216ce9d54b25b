"""Graph-timed LayerNorm (pscwin_layer_norm) at the step's shapes, L2 flushed between replays by a 256 MiB write:
python tools/rowops_probe.py   (PSCWIN_LN_RPW = 1 / 2 / 4 selects rows per warp)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_02109_b200 as pl  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1000)
    return best


for rows, C in [(65536, 768), (4096, 768), (32768, 768)]:
    x = torch.randn(rows, C, device="cuda").to(torch.bfloat16)
    g = torch.randn(C, device="cuda")
    b = torch.randn(C, device="cuda")
    y = pl.layer_norm(x, g, b)
    ref = torch.nn.functional.layer_norm(x.float(), (C,), g, b, 1e-6)
    err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
    us = timed(lambda: pl.layer_norm(x, g, b))
    gbs = 2 * rows * C * 2 / us / 1e3
    print(f"LN rows={rows} C={C} rpw={os.environ.get('PSCWIN_LN_RPW', 'default')}: {us:7.2f} us {gbs:7.1f} GB/s "
          f"rel err {err:.2e}", flush=True)
