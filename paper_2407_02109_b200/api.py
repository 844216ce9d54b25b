"""Torch-facing wrappers over the C ABI (same names as include/pscwin.h, minus the `pscwin_` prefix).

PyTorch supplies device memory and the current CUDA stream; every computation runs in libpscwin.so.
Tensors must be CUDA, contiguous, 16-byte aligned; dtype bf16 (activations, GEMM weights) or f32 (LN params,
biases, scan parameters) as documented per call in include/pscwin.h.
"""
from __future__ import annotations

import ctypes
from typing import Dict, Optional

import torch

from ._lib import (BF16, CS_MULTI_SCALE, CS_NONE, CS_SINGLE_SCALE, F32, LayerDesc, LayerWeights,  # noqa: F401
                   MSDesc, ScanDesc, check, index_map, lib, ms_index_map, window_count)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libpscwin needs CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("libpscwin needs contiguous tensors")
    return t.data_ptr()


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported dtype {t.dtype}")


# ------------------------------------------------------------------------------- a5 / a7 data movement

def window_partition(x: torch.Tensor, window: int) -> torch.Tensor:
    B, H, W, Cx = x.shape
    n = window_count(H, W, window)
    out = torch.empty(B * n, window * window, Cx, dtype=x.dtype, device=x.device)
    check(lib().pscwin_window_partition(_ptr(x), B, H, W, Cx, window, _dt(x), _ptr(out), _stream()),
          "window_partition")
    return out


def shifted_pad_partition(x: torch.Tensor, pad_row: Optional[torch.Tensor], window: int, sx: int,
                          sy: int) -> torch.Tensor:
    B, H, W, Cx = x.shape
    n = window_count(H, W, window, sx, sy)
    out = torch.empty(B * n, window * window, Cx, dtype=x.dtype, device=x.device)
    check(lib().pscwin_shifted_pad_partition(_ptr(x), _ptr(pad_row), B, H, W, Cx, window, sx, sy, _dt(x),
                                             _ptr(out), _stream()), "shifted_pad_partition")
    return out


def window_merge(win: torch.Tensor, B: int, H: int, W: int, window: int, sx: int = 0, sy: int = 0,
                 residual: Optional[torch.Tensor] = None) -> torch.Tensor:
    Cx = win.shape[-1]
    out = torch.empty(B, H, W, Cx, dtype=win.dtype, device=win.device)
    check(lib().pscwin_window_merge(_ptr(win), B, H, W, Cx, window, sx, sy, _ptr(residual), _dt(win), _ptr(out),
                                    _stream()), "window_merge")
    return out


# ------------------------------------------------------------------------------- step entry points

def layer_norm(x: torch.Tensor, g: torch.Tensor, b: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    C = x.shape[-1]
    out = torch.empty_like(x)
    check(lib().pscwin_layer_norm(_ptr(x), x.numel() // C, C, _ptr(g), _ptr(b), eps, _dt(x), _ptr(out), _stream()),
          "layer_norm")
    return out


def linear(A: torch.Tensor, Wt: torch.Tensor, bias: Optional[torch.Tensor] = None,
           residual: Optional[torch.Tensor] = None, out_f32: bool = False) -> torch.Tensor:
    K = A.shape[-1]
    M = A.numel() // K
    N = Wt.shape[0]
    out = torch.empty(*A.shape[:-1], N, dtype=torch.float32 if out_f32 else torch.bfloat16, device=A.device)
    check(lib().pscwin_linear(_ptr(A), M, K, _ptr(Wt), N, _ptr(bias), _ptr(residual), int(out_f32), _ptr(out),
                              _stream()), "linear")
    return out


class Workspace:
    """Caller-owned scratch buffer (the ABI never allocates)."""

    def __init__(self, nbytes: int, device="cuda"):
        self.nbytes = max(int(nbytes), 256)
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()


def workspace_bytes(desc: LayerDesc) -> int:
    return int(lib().pscwin_workspace_bytes(ctypes.byref(desc)))


def qkv_project(desc: LayerDesc, weights: Dict[str, torch.Tensor], x: torch.Tensor, ws: Optional[Workspace] = None):
    C = desc.C
    ws = ws or Workspace(workspace_bytes(desc), x.device)
    qkv = torch.empty(*x.shape[:-1], 3 * C, dtype=torch.bfloat16, device=x.device)
    qkv_pad = torch.empty(3 * C, dtype=torch.float32, device=x.device)
    wts = LayerWeights.from_tensors(weights)
    check(lib().pscwin_qkv_project(ctypes.byref(desc), ctypes.byref(wts), _ptr(x), _ptr(qkv), _ptr(qkv_pad), ws.ptr,
                                   ws.nbytes, _stream()), "qkv_project")
    return qkv, qkv_pad


def window_attention(desc: LayerDesc, qkv: torch.Tensor, qkv_pad: Optional[torch.Tensor],
                     ws: Optional[Workspace] = None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    ws = ws or Workspace(workspace_bytes(desc), qkv.device)
    if out is None:
        out = torch.empty(desc.B, desc.H, desc.W, desc.C, dtype=torch.bfloat16, device=qkv.device)
    check(lib().pscwin_window_attention(ctypes.byref(desc), _ptr(qkv), _ptr(qkv_pad), _ptr(out), ws.ptr, ws.nbytes,
                                        _stream()), "window_attention")
    return out


def scan_workspace_bytes(sd: ScanDesc) -> int:
    return int(lib().pscwin_scan_workspace_bytes(ctypes.byref(sd)))


def cycle_scan(sd: ScanDesc, xin: torch.Tensor, z: Optional[torch.Tensor], w: Dict[str, torch.Tensor],
               ws: Optional[Workspace] = None) -> torch.Tensor:
    ws = ws or Workspace(scan_workspace_bytes(sd), xin.device)
    out = torch.empty_like(xin)
    check(lib().pscwin_cycle_scan(ctypes.byref(sd), _ptr(xin), _ptr(z), _ptr(w["conv_w"]), _ptr(w["conv_b"]),
                                  _ptr(w["w_x"]), _ptr(w["w_dt"]), _ptr(w["b_dt"]), _ptr(w["a_log"]),
                                  _ptr(w["d_skip"]), _ptr(out), ws.ptr, ws.nbytes, _stream()), "cycle_scan")
    return out


def forward(desc: LayerDesc, weights: Dict[str, torch.Tensor], x: torch.Tensor, out: Optional[torch.Tensor] = None,
            ws: Optional[Workspace] = None, wts: Optional[LayerWeights] = None) -> torch.Tensor:
    ws = ws or Workspace(workspace_bytes(desc), x.device)
    if out is None:
        out = torch.empty_like(x)
    wts = wts or LayerWeights.from_tensors(weights)
    check(lib().pscwin_forward(ctypes.byref(desc), ctypes.byref(wts), _ptr(x), _ptr(out), ws.ptr, ws.nbytes,
                               _stream()), "forward")
    return out


class PSCWinLayer:
    """One PSCWin layer with device-resident weights and a persistent workspace."""

    def __init__(self, desc: LayerDesc, weights: Dict[str, torch.Tensor]):
        self.desc = desc
        self.weights = weights
        self.wts = LayerWeights.from_tensors(weights)
        dev = next(iter(weights.values())).device
        self.ws = Workspace(workspace_bytes(desc), dev)

    def __call__(self, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        return forward(self.desc, self.weights, x, out=out, ws=self.ws, wts=self.wts)


def ms_workspace_bytes(desc: MSDesc) -> int:
    return int(lib().pscwin_ms_workspace_bytes(ctypes.byref(desc)))


def ms_forward(desc: MSDesc, weights: Dict[str, torch.Tensor], x: torch.Tensor, out: Optional[torch.Tensor] = None,
               ws: Optional[Workspace] = None, wts: Optional[LayerWeights] = None) -> torch.Tensor:
    """pscwin_ms_forward: x, out [B * sum_s H_s W_s, C] bf16, scale-outermost packing (include/pscwin.h)."""
    ws = ws or Workspace(ms_workspace_bytes(desc), x.device)
    if out is None:
        out = torch.empty_like(x)
    wts = wts or LayerWeights.from_tensors(weights)
    check(lib().pscwin_ms_forward(ctypes.byref(desc), ctypes.byref(wts), _ptr(x), _ptr(out), ws.ptr, ws.nbytes,
                                  _stream()), "ms_forward")
    return out


class PSCWinMSLayer:
    """One HRSAM++ layer (multi-scale attention and / or a single- or multi-scale cycle-scan module) over a packed
    multi-scale sequence, with device-resident weights and a persistent workspace."""

    def __init__(self, desc: MSDesc, weights: Dict[str, torch.Tensor]):
        self.desc = desc
        self.weights = weights
        self.wts = LayerWeights.from_tensors(weights)
        dev = next(iter(weights.values())).device
        self.ws = Workspace(ms_workspace_bytes(desc), dev)

    def __call__(self, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        return ms_forward(self.desc, self.weights, x, out=out, ws=self.ws, wts=self.wts)


class PSCWinStack:
    """A sequence of PSCWin layers with static device buffers, optionally captured once into a CUDA graph and
    replayed (all kernels of all layers become one graph launch; shapes are fixed per resolution).

        stack = PSCWinStack(layers, x_shape)
        y = stack(x)            # copies x into the static input, replays, returns the static output
    """

    def __init__(self, layers, x_shape, device="cuda", graph: bool = True):
        self.layers = list(layers)
        self.x_in = torch.empty(x_shape, dtype=torch.bfloat16, device=device)
        self.bufs = [torch.empty_like(self.x_in), torch.empty_like(self.x_in)]
        self.graph = None
        self.out = self.bufs[(len(self.layers) - 1) & 1] if self.layers else self.x_in
        self.launches_per_step = 0
        # eager warm-up (sets kernel attributes; counts launches)
        from ._lib import launch_count
        n0 = launch_count()
        self._run()
        torch.cuda.synchronize()
        self.launches_per_step = launch_count() - n0
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._run()
            torch.cuda.synchronize()
            self.graph = g

    def _run(self):
        cur = self.x_in
        for j, layer in enumerate(self.layers):
            layer(cur, out=self.bufs[j & 1])
            cur = self.bufs[j & 1]
        return cur

    def replay(self) -> torch.Tensor:
        if self.graph is not None:
            self.graph.replay()
        else:
            self._run()
        return self.out

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        self.x_in.copy_(x, non_blocking=True)
        return self.replay()
