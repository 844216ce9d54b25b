"""Run the bench workload's step a few times (for ncu captures): python tools/run_stage.py [steps] [workload]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2407_02109_b200 as pl  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = sys.argv[2] if len(sys.argv) > 2 else "1024"
label, B, cfgs = bench.workload(wl)
layers = []
for i, cfg in enumerate(cfgs):
    w = synth.make_weights(cfg, layer=i)
    dw = {k: torch.tensor(v, dtype=torch.float32 if k in bench.F32_KEYS else torch.bfloat16, device="cuda")
          for k, v in w.items()}
    layers.append(pl.PSCWinLayer(pl.LayerDesc.from_config(cfg), dw))
x = torch.tensor(synth.make_input(cfgs[0]), dtype=torch.bfloat16, device="cuda")
bufs = [torch.empty_like(x), torch.empty_like(x)]
for _ in range(steps):
    cur = x
    for j, layer in enumerate(layers):
        layer(cur, out=bufs[j & 1])
        cur = bufs[j & 1]
torch.cuda.synchronize()
print("ok", label)
