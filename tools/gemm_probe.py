"""Time the library GEMM (pscwin_linear) with CUDA graphs (no host launch gaps): python tools/gemm_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2407_02109_b200 as pl  # noqa: E402

REPS = 20


def graph_time(fn):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(REPS):
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
        best = min(best, a.elapsed_time(b) * 1000 / REPS)
    return best


shapes = [("qkv", 4096, 768, 2304, False), ("out", 4096, 768, 768, False), ("in_proj", 4096, 768, 3072, False),
          ("out_scan", 4096, 1536, 768, False), ("x_proj", 4099, 1536, 112, True),
          ("xp_N16", 4096, 1536, 16, True), ("xp_N64", 4096, 1536, 64, True), ("xp_N256", 4096, 1536, 256, True),
          ("xp_K384", 4096, 384, 112, True), ("xp_K768", 4096, 768, 112, True), ("xp_K3072", 4096, 3072, 112, True),
          ("m1tile_K1536", 128, 1536, 128, False), ("m1tile_K6144", 128, 6144, 128, False),
          ("m148_K1536", 128 * 148, 1536, 128, False),
          ("big", 8192, 4096, 4096, False)]
only = sys.argv[1:]  # optional subset of shape names
shapes += [("out+bias+res", 4096, 768, 768, "br"), ("qkv+bias", 4096, 768, 2304, "b"), ("in_proj+bias", 4096, 768, 3072, "b")]
for name, M, K, N, f32 in shapes:
    if only and name not in only:
        continue
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    if isinstance(f32, str):
        bias = torch.randn(N, device="cuda")
        res = torch.randn(M, N, device="cuda").to(torch.bfloat16) if "r" in f32 else None
        us = graph_time(lambda: pl.linear(A, W, bias=bias, residual=res))
    else:
        us = graph_time(lambda: pl.linear(A, W, out_f32=f32))
    tf = 2 * M * N * K / us / 1e6
    kb = (K + 63) // 64
    print(f"{name:14s} M={M:6d} K={K:5d} N={N:5d} {us:8.2f} us  {tf:7.1f} TF/s  {us / kb:6.3f} us/kblock(if 1 tile/CTA)",
          flush=True)

# 4096^2 shapes (M = 65536 tokens) against cuBLAS (torch.matmul, no epilogue) as the library-GEMM yardstick
if not only or "cublas" in only:
    for name, M, K, N in [("qkv4096", 65536, 768, 2304), ("out4096", 65536, 768, 768), ("in4096", 65536, 768, 3072),
                          ("outscan4096", 65536, 1536, 768), ("fc1_4096", 65536, 768, 3072),
                          ("fc2_4096", 65536, 3072, 768)]:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        ours = graph_time(lambda: pl.linear(A, W))
        cub = graph_time(lambda: torch.matmul(A, W.t()))
        f = 2 * M * N * K / 1e6
        print(f"{name:12s} M={M} K={K} N={N}  ours {ours:8.2f} us {f / ours:7.1f} TF/s   cuBLAS {cub:8.2f} us "
              f"{f / cub:7.1f} TF/s", flush=True)
