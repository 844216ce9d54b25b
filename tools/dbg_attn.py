import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import torch, synth
import paper_2407_02109_b200 as pl
from gpu_util import dev
for side, mk in ((0, lambda: synth.tiny(H=32, W=16)), (1, lambda: synth.vitb(64, shift_x=8, shift_y=8))):
    cfg = mk()
    qkv = dev(synth.make_qkv(cfg)); qp = dev(synth.make_pad_qkv(cfg), "f32")
    d = pl.LayerDesc.from_config(cfg)
    try:
        o = pl.window_attention(d, qkv, qp); torch.cuda.synchronize(); print("ok", side, float(o.float().abs().sum()))
    except Exception as e:
        print("FAIL", side, e); break
