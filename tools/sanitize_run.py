"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over every hot kernel family:
tiny and ViT-B-width layers (plain / learnable-shifted / masked-shifted / cycle scan + FFN), so the attention
kernel runs with one and two q-tile slots, the GEMM with single-CTA and paired tiles, both residual placements
and every epilogue kind. Usage: compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2407_02109_b200 as pl  # noqa: E402
from gpu_util import dev, dev_weights  # noqa: E402

cfgs = [
    ("tiny P", synth.tiny(shift_x=0, shift_y=0)),
    ("tiny S learnable", synth.tiny()),
    ("tiny S masked", synth.tiny(pad_mode=1)),
    ("tiny CS+P", synth.tiny(shift_x=0, shift_y=0, cycle_scan=1)),
    ("vitb 32^2 S learnable + CS + FFN", synth.vitb(32, cycle_scan=1, mlp_hidden=3072)),
    ("vitb 48^2 P (residual GEMM 2 row tiles)", synth.vitb(48, shift_x=0, shift_y=0)),
]
if os.environ.get("PSAN_TINY"):  # initcheck is slow: tiny configurations only
    cfgs = cfgs[:4]
for name, cfg in cfgs:
    x = dev(synth.make_input(cfg, scale=0.05))
    layer = pl.PSCWinLayer(pl.LayerDesc.from_config(cfg), dev_weights(synth.make_weights(cfg), cfg))
    y = layer(x)
    torch.cuda.synchronize()
    print(f"{name}: ok, |y| max {float(y.float().abs().max()):.3f}", flush=True)
