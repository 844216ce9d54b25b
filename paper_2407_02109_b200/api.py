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
                   MSDesc, NeckDesc, ScanDesc, check, index_map, lib, ms_index_map, window_count)


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


def scan_chunks(B: int, L: int, D: int, N: int = 32, R: int = 48, conv_k: int = 4) -> int:
    """Number of chunks the bf16 cycle scan splits each image's L tokens into (pscwin_scan_chunk_length)."""
    sd = ScanDesc()
    sd.B, sd.H, sd.W, sd.D, sd.N, sd.R, sd.conv_k = B, 1, L, D, N, R, conv_k
    lc = int(lib().pscwin_scan_chunk_length(ctypes.byref(sd)))
    return -(-L // lc) if lc > 0 else 0


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

    def run_job(self, xs_host, ys_host, before_step=None) -> None:
        """A job of len(xs_host) inputs from pinned host memory through the stack into pinned host outputs, with the
        host<->device copies overlapped with compute: the H2D copy of input i+1 (one copy stream) and the D2H copy of
        output i-1 (another) run while the graph of input i runs on the current stream; device staging buffers are
        double-buffered and ordered with events. Enqueues everything; the current stream ends after the last D2H.
        before_step(i), if given, is called on the current stream before step i's compute (e.g. an L2 flush)."""
        n = len(xs_host)
        if n == 0:
            return
        cur = torch.cuda.current_stream()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        if not hasattr(self, "_stage_in"):
            self._stage_in = [torch.empty_like(self.x_in) for _ in range(2)]
            self._stage_out = [torch.empty_like(self.out) for _ in range(2)]
        ev = lambda: torch.cuda.Event()  # noqa: E731
        in_ready, in_free = [ev() for _ in range(n)], [ev() for _ in range(n)]
        out_ready, out_free = [ev() for _ in range(n)], [ev() for _ in range(n)]
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        for i in range(n):
            with torch.cuda.stream(s_in):  # H2D of input i into staging slot i % 2 once step i-2 has consumed it
                if i >= 2:
                    s_in.wait_event(in_free[i - 2])
                self._stage_in[i & 1].copy_(xs_host[i], non_blocking=True)
                in_ready[i].record(s_in)
            cur.wait_event(in_ready[i])
            if before_step is not None:
                before_step(i)
            self.x_in.copy_(self._stage_in[i & 1], non_blocking=True)
            in_free[i].record(cur)
            self.replay()
            if i >= 2:
                cur.wait_event(out_free[i - 2])  # staging slot i % 2 read out by the D2H of output i-2
            self._stage_out[i & 1].copy_(self.out, non_blocking=True)
            out_ready[i].record(cur)
            with torch.cuda.stream(s_out):
                s_out.wait_event(out_ready[i])
                ys_host[i].copy_(self._stage_out[i & 1], non_blocking=True)
                out_free[i].record(s_out)
        cur.wait_stream(s_out)


# ------------------------------------------------------------------------------------------- encoder ends

def patch_embed(img: torch.Tensor, w_patch: torch.Tensor, b_patch: torch.Tensor,
                ws: Optional[Workspace] = None) -> torch.Tensor:
    """pscwin_patch_embed: img [B, 3, 16H, 16W] bf16 -> tokens [B, H, W, C] bf16 (w_patch [C, 768] bf16)."""
    B, _, Hi, Wi = img.shape
    H, W, C = Hi // 16, Wi // 16, w_patch.shape[0]
    ws = ws or Workspace(int(lib().pscwin_patch_embed_workspace_bytes(B, H, W)), img.device)
    out = torch.empty(B, H, W, C, dtype=torch.bfloat16, device=img.device)
    check(lib().pscwin_patch_embed(_ptr(img), B, H, W, C, _ptr(w_patch), _ptr(b_patch), _ptr(out), ws.ptr, ws.nbytes,
                                   _stream()), "patch_embed")
    return out


def resize_bilinear(x: torch.Tensor, H: int, W: int, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """pscwin_resize_bilinear: x [B, h, w, C] bf16 -> [B, H, W, C] (accumulates into `out` when given)."""
    B, h, w, C = x.shape
    acc = out is not None
    if out is None:
        out = torch.empty(B, H, W, C, dtype=x.dtype, device=x.device)
    check(lib().pscwin_resize_bilinear(_ptr(x), B, h, w, C, H, W, int(acc), _ptr(out), _stream()), "resize_bilinear")
    return out


def neck_workspace_bytes(desc: NeckDesc) -> int:
    return int(lib().pscwin_neck_workspace_bytes(ctypes.byref(desc)))


def neck(desc: NeckDesc, stage_outs, w: Dict[str, torch.Tensor], ws: Optional[Workspace] = None,
         out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """pscwin_neck: stage outputs (device tensors) -> fused image embedding [B, H0, W0, C_out] bf16.
    w: w_stage{i} [C_out, C], neck_ln1_g/b, w_neck_conv [C_out, 3, 3, C_out] (channels-last), neck_ln2_g/b."""
    dev = stage_outs[0].device
    ws = ws or Workspace(neck_workspace_bytes(desc), dev)
    if out is None:
        out = torch.empty(desc.B, desc.H[0], desc.W[0], desc.C_out, dtype=torch.bfloat16, device=dev)
    n = desc.n_stages
    xs = (ctypes.c_void_p * n)(*[_ptr(t) for t in stage_outs])
    wsv = (ctypes.c_void_p * n)(*[_ptr(w[f"w_stage{i}"]) for i in range(n)])
    check(lib().pscwin_neck(ctypes.byref(desc), xs, wsv, _ptr(w["neck_ln1_g"]), _ptr(w["neck_ln1_b"]),
                            _ptr(w["w_neck_conv"]), _ptr(w["neck_ln2_g"]), _ptr(w["neck_ln2_b"]), _ptr(out), ws.ptr,
                            ws.nbytes, _stream()), "neck")
    return out


class HRSAMEncoder:
    """The whole HRSAM encoder: patch embedding -> the layers (stage outputs after every layer listed in
    `stage_ends`) -> output fusion (neck). All buffers static; optionally captured once into a CUDA graph.

        enc = HRSAMEncoder(layers, ends_weights, B, H, W, stage_ends=(2, 5, 8, 11))
        emb = enc(img)     # img [B, 3, 16H, 16W] bf16 -> [B, H, W, 256]

    HRSAM++ (reading Q20 / Q22): pass `scales=[(H, W), (H1, W1), ...]` (scale 0 = the main grid, e.g. the
    512^2 overview image as (32, 32)) and PSCWinMSLayer layers; every scale's image is patch-embedded straight into
    its slice of the packed [B * sum H_s W_s, C] sequence, the layers run on the packed sequence, and the neck fuses
    each scale's stage sum, resizing the other scales onto the main grid before the conv block.

        enc = HRSAMEncoder(ms_layers, ends, B, 64, 64, scales=[(64, 64), (32, 32)])
        emb = enc([img_1024, img_512])   # -> [B, 64, 64, 256]
    """

    def __init__(self, layers, ends: Dict[str, torch.Tensor], B: int, H: int, W: int, stage_ends=(2, 5, 8, 11),
                 C: int = 768, C_out: int = 256, graph: bool = True, scales=None):
        dev = ends["w_patch"].device
        self.layers, self.ends, self.stage_ends = list(layers), ends, tuple(stage_ends)
        self.scales = [(H, W)] if scales is None else [tuple(s) for s in scales]
        if self.scales[0] != (H, W):
            raise ValueError("scale 0 is the main grid (H, W)")
        T = B * sum(h * w for h, w in self.scales)
        self.imgs = [torch.empty(B, 3, 16 * h, 16 * w, dtype=torch.bfloat16, device=dev) for h, w in self.scales]
        self.img = self.imgs[0]
        self.x0 = torch.empty(T, C, dtype=torch.bfloat16, device=dev)
        self.bufs = [torch.empty_like(self.x0), torch.empty_like(self.x0)]
        self.stage = [torch.empty_like(self.x0) for _ in self.stage_ends]
        self.desc = NeckDesc.make(B, C, C_out, self.scales, n_stages=len(self.stage_ends))
        self.ws_pe = Workspace(max(int(lib().pscwin_patch_embed_workspace_bytes(B, h, w)) for h, w in self.scales), dev)
        self.ws_neck = Workspace(neck_workspace_bytes(self.desc), dev)
        self.out = torch.empty(B, H, W, C_out, dtype=torch.bfloat16, device=dev)
        self.w_patch = ends["w_patch"].reshape(C, -1).contiguous()
        # packed rows of scale s: [B * off_s, B * off_{s+1}) as a [B, H_s, W_s, C] grid
        off = [0]
        for h, w in self.scales:
            off.append(off[-1] + h * w)
        self.x0_views = [self.x0[B * off[i]:B * off[i + 1]].view(B, h, w, C) for i, (h, w) in enumerate(self.scales)]
        from ._lib import launch_count
        n0 = launch_count()
        self._run()
        torch.cuda.synchronize()
        self.launches_per_step = launch_count() - n0
        self.graph = None
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._run()
            torch.cuda.synchronize()
            self.graph = g

    def _run(self):
        for img, xv in zip(self.imgs, self.x0_views):
            check(lib().pscwin_patch_embed(_ptr(img), xv.shape[0], xv.shape[1], xv.shape[2], xv.shape[3],
                                           _ptr(self.w_patch), _ptr(self.ends["b_patch"]), _ptr(xv), self.ws_pe.ptr,
                                           self.ws_pe.nbytes, _stream()), "patch_embed")
        cur, k = self.x0, 0
        for j, layer in enumerate(self.layers):
            if j in self.stage_ends:
                nxt = self.stage[self.stage_ends.index(j)]
            else:
                nxt = self.bufs[k & 1] if self.bufs[k & 1] is not cur else self.bufs[(k + 1) & 1]
                k += 1
            layer(cur, out=nxt)
            cur = nxt
        neck(self.desc, self.stage, self.ends, ws=self.ws_neck, out=self.out)
        return self.out

    def __call__(self, img) -> torch.Tensor:
        imgs = img if isinstance(img, (list, tuple)) else [img]
        if len(imgs) != len(self.imgs):
            raise ValueError(f"{len(self.imgs)} images expected (one per scale)")
        for dst, src in zip(self.imgs, imgs):
            dst.copy_(src, non_blocking=True)
        if self.graph is not None:
            self.graph.replay()
        else:
            self._run()
        return self.out
