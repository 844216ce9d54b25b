"""ctypes binding of libpscwin.so (include/pscwin.h). Argument marshalling only: every step of the path runs
in the CUDA library. PyTorch provides device memory and the current stream.

The library is REQUIRED: there is no CPU or eager fallback. `lib()` raises if libpscwin.so is missing or
cannot be loaded, and every call raises PscwinError on a non-zero status.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpscwin.so")

OK, ERR_SHAPE, ERR_CONTRACT, ERR_ALIGN, ERR_WORKSPACE, ERR_CUDA, ERR_UNSUPPORTED, ERR_NCCL, ERR_TIMEOUT = range(9)
BF16, F32 = 0, 1
PAD_LEARNABLE, PAD_MASKED = 0, 1
CS_NONE, CS_SINGLE_SCALE, CS_MULTI_SCALE = 0, 1, 2
MAX_SCALES = 4

# every symbol include/pscwin.h declares (checked by tests/test_abi_cpu.py)
EXPORTS = [
    "pscwin_version", "pscwin_status_string", "pscwin_last_async_error", "pscwin_window_count",
    "pscwin_index_map", "pscwin_window_partition", "pscwin_shifted_pad_partition", "pscwin_window_merge",
    "pscwin_layer_norm", "pscwin_linear", "pscwin_qkv_project", "pscwin_window_attention", "pscwin_cycle_scan",
    "pscwin_scan_workspace_bytes", "pscwin_scan_chunk_length", "pscwin_workspace_bytes", "pscwin_forward",
    "pscwin_launch_count", "pscwin_profile_enable", "pscwin_profile_read",
    "pscwin_band_workspace_bytes", "pscwin_band_io_offsets", "pscwin_band_scan_begin", "pscwin_band_scan_mid",
    "pscwin_band_scan_end", "pscwin_band_attn_begin", "pscwin_band_attn_end", "pscwin_band_window_split",
    "pscwin_band_attn_windows", "pscwin_band_out_proj",
    "pscwin_ms_window_count", "pscwin_ms_index_map", "pscwin_ms_workspace_bytes", "pscwin_ms_forward",
    "pscwin_patch_embed_workspace_bytes", "pscwin_patch_embed", "pscwin_resize_bilinear", "pscwin_neck_workspace_bytes",
    "pscwin_neck", "pscwin_nccl_get_unique_id", "pscwin_nccl_comm_init", "pscwin_nccl_comm_destroy",
    "pscwin_nccl_comm_check", "pscwin_nccl_comm_abort", "pscwin_nccl_wait",
    "pscwin_dist_workspace_bytes", "pscwin_dist_forward",
]


class PscwinError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _LIB.pscwin_status_string(status).decode() if _LIB is not None else str(status)
        super().__init__(f"{where}: {msg} (status {status})")


class LayerDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "B", "H", "W", "C", "heads", "window", "shift_x", "shift_y", "pad_mode", "rope", "cycle_scan",
        "ssm_state", "ssm_expand", "ssm_dt_rank", "ssm_conv", "scan_order", "bbar_mode", "dtype")] + \
        [("ln_eps", ctypes.c_float), ("mlp_hidden", ctypes.c_int32)]

    @classmethod
    def from_config(cls, cfg) -> "LayerDesc":
        d = cls()
        for name, _ in cls._fields_:
            if name == "dtype":
                d.dtype = BF16 if getattr(cfg, "dtype", "bf16") == "bf16" else F32
            elif name == "ssm_dt_rank":
                d.ssm_dt_rank = getattr(cfg, "R", 0)
            elif name == "mlp_hidden":
                d.mlp_hidden = getattr(cfg, "mlp_hidden", 0)
            else:
                setattr(d, name, getattr(cfg, name))
        return d


class LayerWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "ln1_g", "ln1_b", "w_qkv", "b_qkv", "pad", "w_o", "b_o",
        "lns_g", "lns_b", "w_in", "conv_w", "conv_b", "w_x", "w_dt", "b_dt", "w_out", "a_log", "d_skip",
        "ln2_g", "ln2_b", "w_fc1", "b_fc1", "w_fc2", "b_fc2")]

    @classmethod
    def from_tensors(cls, t: Dict[str, "torch.Tensor"]) -> "LayerWeights":
        w = cls()
        for name, _ in cls._fields_:
            if name in t and t[name] is not None:
                setattr(w, name, t[name].data_ptr())
        return w


class MSDesc(ctypes.Structure):
    """pscwin_ms_desc: one HRSAM++ layer over a packed multi-scale sequence (scale-outermost packing, Q20)."""
    _fields_ = [("layer", LayerDesc), ("n_scales", ctypes.c_int32), ("H", ctypes.c_int32 * MAX_SCALES),
                ("W", ctypes.c_int32 * MAX_SCALES), ("attention", ctypes.c_int32), ("cycle_scan", ctypes.c_int32)]

    @classmethod
    def make(cls, cfg, scales, attention: int = 1, cycle_scan: int = CS_NONE) -> "MSDesc":
        if not 1 <= len(scales) <= MAX_SCALES:
            raise ValueError(f"1..{MAX_SCALES} scales")
        m = cls()
        m.layer = LayerDesc.from_config(cfg.replace(H=scales[0][0], W=scales[0][1], cycle_scan=0))
        m.n_scales = len(scales)
        for i, (h, w) in enumerate(scales):
            m.H[i], m.W[i] = h, w
        m.attention = int(attention)
        m.cycle_scan = int(cycle_scan)
        return m

    @property
    def tokens_per_sample(self) -> int:
        return sum(self.H[i] * self.W[i] for i in range(self.n_scales))


class NeckDesc(ctypes.Structure):
    """pscwin_neck_desc: output fusion of the stages (1x1 projections summed, HRSAM++ scales resized, conv block)."""
    _fields_ = [("B", ctypes.c_int32), ("C", ctypes.c_int32), ("C_out", ctypes.c_int32), ("n_stages", ctypes.c_int32),
                ("n_scales", ctypes.c_int32), ("H", ctypes.c_int32 * MAX_SCALES), ("W", ctypes.c_int32 * MAX_SCALES),
                ("ln_eps", ctypes.c_float)]

    @classmethod
    def make(cls, B, C, C_out, scales, n_stages=4, eps=1e-6) -> "NeckDesc":
        d = cls()
        d.B, d.C, d.C_out, d.n_stages, d.n_scales, d.ln_eps = B, C, C_out, n_stages, len(scales), eps
        for i, (h, w) in enumerate(scales):
            d.H[i], d.W[i] = h, w
        return d


class ScanDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("B", "H", "W", "D", "N", "R", "conv_k", "scan_order", "bbar_mode",
                                              "dtype", "window")]


class BandDesc(ctypes.Structure):
    """pscwin_band: this rank's token rows [row_begin, row_end) of one image split over `world` ranks."""
    _fields_ = [(n, ctypes.c_int32) for n in ("row_begin", "row_end", "rank", "world")]


class BandIO(ctypes.Structure):
    """pscwin_band_io: workspace byte offsets / sizes of the buffers the ranks exchange."""
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "hist_send", "hist_recv", "hist_bytes", "rec_send", "rec_recv", "rec_bytes",
        "send_prev", "send_prev_bytes", "send_next", "send_next_bytes",
        "recv_prev", "recv_prev_bytes", "recv_next", "recv_next_bytes")]


_LIB: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
    sig = {
        "pscwin_version": ([], ctypes.c_char_p),
        "pscwin_status_string": ([ctypes.c_int], ctypes.c_char_p),
        "pscwin_last_async_error": ([], ctypes.c_int),
        "pscwin_window_count": ([i32, i32, i32, i32, i32, ctypes.POINTER(i32)], ctypes.c_int),
        "pscwin_index_map": ([i32, i32, i32, i32, i32, vp], ctypes.c_int),
        "pscwin_window_partition": ([vp, i32, i32, i32, i32, i32, i32, vp, vp], ctypes.c_int),
        "pscwin_shifted_pad_partition": ([vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, vp, vp], ctypes.c_int),
        "pscwin_window_merge": ([vp, i32, i32, i32, i32, i32, i32, i32, vp, i32, vp, vp], ctypes.c_int),
        "pscwin_layer_norm": ([vp, i64, i32, vp, vp, f32, i32, vp, vp], ctypes.c_int),
        "pscwin_linear": ([vp, i64, i32, vp, i32, vp, vp, i32, vp, vp], ctypes.c_int),
        "pscwin_qkv_project": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(LayerWeights), vp, vp, vp, vp, sz, vp],
                               ctypes.c_int),
        "pscwin_window_attention": ([ctypes.POINTER(LayerDesc), vp, vp, vp, vp, sz, vp], ctypes.c_int),
        "pscwin_cycle_scan": ([ctypes.POINTER(ScanDesc), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp],
                              ctypes.c_int),
        "pscwin_scan_workspace_bytes": ([ctypes.POINTER(ScanDesc)], sz),
        "pscwin_scan_chunk_length": ([ctypes.POINTER(ScanDesc)], ctypes.c_int32),
        "pscwin_workspace_bytes": ([ctypes.POINTER(LayerDesc)], sz),
        "pscwin_forward": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(LayerWeights), vp, vp, vp, sz, vp],
                           ctypes.c_int),
        "pscwin_band_workspace_bytes": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc)], sz),
        "pscwin_band_io_offsets": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc), ctypes.POINTER(BandIO)],
                                   ctypes.c_int),
        "pscwin_band_scan_begin": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc), ctypes.POINTER(LayerWeights),
                                    vp, vp, sz, vp], ctypes.c_int),
        "pscwin_band_scan_mid": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc), ctypes.POINTER(LayerWeights),
                                  vp, sz, vp], ctypes.c_int),
        "pscwin_band_scan_end": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc), ctypes.POINTER(LayerWeights),
                                  vp, vp, sz, vp], ctypes.c_int),
        "pscwin_band_attn_begin": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc), ctypes.POINTER(LayerWeights),
                                    vp, vp, sz, vp], ctypes.c_int),
        "pscwin_band_attn_end": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc), ctypes.POINTER(LayerWeights),
                                  vp, vp, vp, sz, vp], ctypes.c_int),
        "pscwin_band_window_split": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc), ctypes.POINTER(i32),
                                      ctypes.POINTER(i32), ctypes.POINTER(i32)], ctypes.c_int),
        "pscwin_band_attn_windows": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc),
                                      ctypes.POINTER(LayerWeights), vp, sz, i32, i32, vp], ctypes.c_int),
        "pscwin_band_out_proj": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(BandDesc), ctypes.POINTER(LayerWeights),
                                  vp, vp, vp, sz, vp], ctypes.c_int),
        "pscwin_ms_window_count": ([ctypes.POINTER(MSDesc), ctypes.POINTER(i32)], ctypes.c_int),
        "pscwin_ms_index_map": ([ctypes.POINTER(MSDesc), vp], ctypes.c_int),
        "pscwin_ms_workspace_bytes": ([ctypes.POINTER(MSDesc)], sz),
        "pscwin_ms_forward": ([ctypes.POINTER(MSDesc), ctypes.POINTER(LayerWeights), vp, vp, vp, sz, vp],
                              ctypes.c_int),
        "pscwin_patch_embed_workspace_bytes": ([i32, i32, i32], sz),
        "pscwin_patch_embed": ([vp, i32, i32, i32, i32, vp, vp, vp, vp, sz, vp], ctypes.c_int),
        "pscwin_resize_bilinear": ([vp, i32, i32, i32, i32, i32, i32, i32, vp, vp], ctypes.c_int),
        "pscwin_neck_workspace_bytes": ([ctypes.POINTER(NeckDesc)], sz),
        "pscwin_neck": ([ctypes.POINTER(NeckDesc), ctypes.POINTER(vp), ctypes.POINTER(vp), vp, vp, vp, vp, vp, vp, vp,
                         sz, vp], ctypes.c_int),
        "pscwin_nccl_get_unique_id": ([vp], ctypes.c_int),
        "pscwin_nccl_comm_init": ([vp, i32, i32, ctypes.POINTER(vp)], ctypes.c_int),
        "pscwin_nccl_comm_destroy": ([vp], ctypes.c_int),
        "pscwin_nccl_comm_check": ([vp], ctypes.c_int),
        "pscwin_nccl_comm_abort": ([vp], ctypes.c_int),
        "pscwin_nccl_wait": ([vp, vp, ctypes.c_int64], ctypes.c_int),
        "pscwin_dist_workspace_bytes": ([ctypes.POINTER(LayerDesc), i32, i32, i32, i32], sz),
        "pscwin_dist_forward": ([ctypes.POINTER(LayerDesc), ctypes.POINTER(LayerWeights), vp, vp, i32, i32, vp, vp, sz,
                                 vp, vp], ctypes.c_int),
        "pscwin_launch_count": ([], ctypes.c_int64),
        "pscwin_profile_enable": ([ctypes.c_int], None),
        "pscwin_profile_read": ([ctypes.c_char_p, sz, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32), i32],
                                ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = L
    return L


def check(status: int, where: str) -> None:
    if status != OK:
        raise PscwinError(status, where)


# ------------------------------------------------------------------------------------------------ host helpers

def window_count(H: int, W: int, window: int, sx: int = 0, sy: int = 0) -> int:
    n = ctypes.c_int32()
    check(lib().pscwin_window_count(H, W, window, sx, sy, ctypes.byref(n)), "window_count")
    return n.value


def launch_count() -> int:
    return int(lib().pscwin_launch_count())


def profile_enable(on: bool = True) -> None:
    lib().pscwin_profile_enable(int(on))


def profile_read(max_entries: int = 64) -> Dict[str, tuple]:
    """{kernel label: (total_ms, launches)} for the launches recorded since profile_enable()."""
    names = ctypes.create_string_buffer(8192)
    ms = (ctypes.c_double * max_entries)()
    cnt = (ctypes.c_int32 * max_entries)()
    n = lib().pscwin_profile_read(names, 8192, ms, cnt, max_entries)
    labels = names.value.decode().split("\n")[:n]
    return {labels[i]: (ms[i], cnt[i]) for i in range(n)}


def index_map(H: int, W: int, window: int, sx: int = 0, sy: int = 0) -> np.ndarray:
    n = window_count(H, W, window, sx, sy)
    out = np.empty(n * window * window, dtype=np.uint32)
    check(lib().pscwin_index_map(H, W, window, sx, sy, out.ctypes.data), "index_map")
    return out


def ms_index_map(desc: "MSDesc") -> np.ndarray:
    """Multi-scale indexing operator (App. C over a packed multi-scale sequence), host-side."""
    n = ctypes.c_int32()
    check(lib().pscwin_ms_window_count(ctypes.byref(desc), ctypes.byref(n)), "ms_window_count")
    w = desc.layer.window
    out = np.empty(n.value * w * w, dtype=np.uint32)
    check(lib().pscwin_ms_index_map(ctypes.byref(desc), out.ctypes.data), "ms_index_map")
    return out
