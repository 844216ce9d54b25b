"""Debug helper: run each attention parity case in its own process (a fault in one cannot poison the others)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CASE = r'''
import sys; sys.path.insert(0, "{root}"); sys.path.insert(0, "{root}/tests")
import numpy as np, torch, synth, oracle
import paper_2407_02109_b200 as pl
from test_gpu_parity import ATTN_CASES, _attn_inputs
from gpu_util import dev, host, rel_err
cfg = ATTN_CASES[{i}]
qkv, qkv_p, gq = _attn_inputs(cfg)
O = pl.window_attention(pl.LayerDesc.from_config(cfg), dev(gq), dev(qkv_p, "f32"))
torch.cuda.synchronize()
ref = oracle.attention_core_padded(qkv, qkv_p, cfg.H, cfg.W, cfg.heads, cfg.window, cfg.shift_x, cfg.shift_y, cfg.pad_mode, cfg.rope)
print("case {i}", cfg.H, cfg.W, cfg.C, cfg.heads, cfg.window, cfg.shift_x, cfg.pad_mode, cfg.rope, "err", rel_err(host(O), ref))
'''

if __name__ == "__main__":
    from test_gpu_parity import ATTN_CASES
    pre = sys.argv[1:]  # e.g. compute-sanitizer
    for i in range(len(ATTN_CASES)):
        r = subprocess.run(pre + [sys.executable, "-c", CASE.format(root=ROOT, i=i)], capture_output=True, text=True,
                           timeout=300, env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"))
        out = (r.stdout + r.stderr).strip().splitlines()
        print(f"[{i}] rc={r.returncode}", *out[-4:], sep="\n   ", flush=True)
