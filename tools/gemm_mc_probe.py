"""B multicast across CTA pairs (PSCWIN_GEMM_MC): outputs and graph-timed speed of the 4096^2 projection shapes.

    PSCWIN_GEMM_MC=1 python tools/gemm_mc_probe.py save /tmp/mc1.pt     # reference run (pairs, no multicast)
    python tools/gemm_mc_probe.py cmp /tmp/mc1.pt                      # multicast run: bit-identity + timings
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_02109_b200 as pl  # noqa: E402


def graph_time(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1000 / reps)
    return best

SHAPES = [  # name, M, K, N, bias, residual
    ("qkv", 65536, 768, 2304, True, False),
    ("out_proj", 65536, 768, 768, True, True),
    ("in_proj", 65536, 768, 3072, False, False),
    ("out_proj_scan", 65536, 1536, 768, False, True),
    ("fc1", 65536, 768, 3072, True, False),
    ("ragged_superTile", 65536 + 128, 768, 768, True, True),
    ("ragged_rows", 1000 + 512, 768, 320, True, True),
    ("n_tail", 4096, 768, 2304 - 32, True, False),
]


def run(mode, path):
    g = torch.Generator(device="cuda").manual_seed(7)
    outs = {}
    for name, M, K, N, bias, resid in SHAPES:
        A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
        b = torch.randn(N, device="cuda", generator=g) if bias else None
        r = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16) if resid else None
        y = pl.linear(A, W, bias=b, residual=r)
        torch.cuda.synchronize()
        ref = (A.float() @ W.float().t() + (b if bias else 0) + (r.float() if resid else 0))
        err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
        us = graph_time(lambda: pl.linear(A, W, bias=b, residual=r))
        tf = 2 * M * N * K / us / 1e6
        line = f"{name:18s} M={M:6d} K={K:5d} N={N:5d} {us:8.2f} us {tf:7.1f} TF/s  rel err vs fp32 {err:.2e}"
        if mode == "cmp":
            prev = torch.load(path)[name].cuda()
            same = torch.equal(prev, y)
            line += f"  bit-identical to MC=1: {same}"
            if not same:
                line += f" (max diff {(prev.float() - y.float()).abs().max().item():.3e})"
        outs[name] = y.cpu()
        print(line, flush=True)
    if mode == "save":
        torch.save(outs, path)


if __name__ == "__main__":
    run(sys.argv[1], sys.argv[2])
