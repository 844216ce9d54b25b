"""Window-row sharding of one image over several GPUs, driving the band phases of
libpscwin.so (include/pscwin.h "row bands"). Every step runs in the library; between phases the ranks exchange
the conv history (ring), the scan records (all-gather) and the QKV halo rows (neighbours) — over NCCL with
`dist.TorchDistExchange`, or by device copies between virtual ranks on one GPU with `LoopbackBands` (tests)."""
from __future__ import annotations

import ctypes
from typing import Dict, List

import torch

from ._lib import ERR_NCCL, ERR_TIMEOUT, BandDesc, BandIO, LayerDesc, LayerWeights, check, lib
from .api import _ptr, _stream
from .dist import band_rows


class BandLayer:
    """One PSCWin layer on this rank's band of token rows (global layer desc + band)."""

    def __init__(self, desc: LayerDesc, weights: Dict[str, torch.Tensor], row_begin: int, row_end: int, rank: int,
                 world: int):
        self.desc, self.weights = desc, weights
        self.wts = LayerWeights.from_tensors(weights)
        self.band = BandDesc(row_begin, row_end, rank, world)
        dev = next(iter(weights.values())).device
        n = int(lib().pscwin_band_workspace_bytes(ctypes.byref(desc), ctypes.byref(self.band)))
        if n == 0:
            raise ValueError("invalid band for this layer (rows must be whole window rows, B = 1, bf16, "
                             "row-major scan)")
        self.ws = torch.empty(max(n, 256), dtype=torch.uint8, device=dev)
        self.io = BandIO()
        check(lib().pscwin_band_io_offsets(ctypes.byref(desc), ctypes.byref(self.band), ctypes.byref(self.io)),
              "band_io_offsets")

    def view(self, off_name: str, size_name: str, count: int = 1) -> torch.Tensor:
        off, size = getattr(self.io, off_name), getattr(self.io, size_name) * count
        return self.ws[off:off + size]

    def _call(self, name, *args):
        fn = getattr(lib(), "pscwin_band_" + name)
        check(fn(ctypes.byref(self.desc), ctypes.byref(self.band), ctypes.byref(self.wts), *args, self.ws.data_ptr(),
                 self.ws.numel(), _stream()), "band_" + name)

    def scan_begin(self, x):
        self._call("scan_begin", _ptr(x))

    def scan_mid(self):
        fn = lib().pscwin_band_scan_mid
        check(fn(ctypes.byref(self.desc), ctypes.byref(self.band), ctypes.byref(self.wts), self.ws.data_ptr(),
                 self.ws.numel(), _stream()), "band_scan_mid")

    def scan_end(self, x):
        self._call("scan_end", _ptr(x))

    def attn_begin(self, x):
        self._call("attn_begin", _ptr(x))

    def attn_end(self, x, out):
        self._call("attn_end", _ptr(x), _ptr(out))

    # attn_end split around the halo exchange (what pscwin_dist_forward overlaps on two streams)
    def window_split(self):
        t, b, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        check(lib().pscwin_band_window_split(ctypes.byref(self.desc), ctypes.byref(self.band), ctypes.byref(t),
                                             ctypes.byref(b), ctypes.byref(n)), "band_window_split")
        return t.value, b.value, n.value

    def attn_windows(self, wy0, wy1):
        check(lib().pscwin_band_attn_windows(ctypes.byref(self.desc), ctypes.byref(self.band), ctypes.byref(self.wts),
                                             self.ws.data_ptr(), self.ws.numel(), wy0, wy1, _stream()),
              "band_attn_windows")

    def out_proj(self, x, out):
        self._call("out_proj", _ptr(x), _ptr(out))

    # exchange buffers
    def hist(self):
        return self.view("hist_send", "hist_bytes"), self.view("hist_recv", "hist_bytes")

    def records(self):
        return self.view("rec_send", "rec_bytes"), self.view("rec_recv", "rec_bytes", self.band.world)

    def halo(self):
        return (self.view("send_prev", "send_prev_bytes"), self.view("send_next", "send_next_bytes"),
                self.view("recv_prev", "recv_prev_bytes"), self.view("recv_next", "recv_next_bytes"))


def band_forward(layer: BandLayer, x_band: torch.Tensor, exchange, out: torch.Tensor = None) -> torch.Tensor:
    """This rank's part of one layer; `exchange` is a dist.TorchDistExchange (all ranks call together)."""
    out = torch.empty_like(x_band) if out is None else out
    if layer.desc.cycle_scan:
        layer.scan_begin(x_band)
        exchange.ring(*layer.hist())
        layer.scan_mid()
        exchange.allgather(*layer.records())
        layer.scan_end(x_band)
    layer.attn_begin(x_band)
    exchange.halo(*layer.halo())
    layer.attn_end(x_band, out)
    return out


class LoopbackBands:
    """All `world` bands of one image on one GPU, phases run in lockstep and the exchanges done as device copies
    (the same byte movements NCCL performs across GPUs). Used to check the band path against pscwin_forward."""

    def __init__(self, desc: LayerDesc, weights: Dict[str, torch.Tensor], world: int, overlap: bool = False):
        self.overlap = overlap  # interior windows before the halo copies, band-edge windows after (dist schedule)
        self.rows = band_rows(desc.H, desc.window, world)
        self.layers: List[BandLayer] = [BandLayer(desc, weights, r0, r1, g, world)
                                        for g, (r0, r1) in enumerate(self.rows)]

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        L, G = self.layers, len(self.layers)
        xs = [x[:, r0:r1].contiguous() for r0, r1 in self.rows]
        outs = [torch.empty_like(xb) for xb in xs]
        if L[0].desc.cycle_scan:
            for g in range(G):
                L[g].scan_begin(xs[g])
            for g in range(G):  # ring: rank g receives rank g-1's tail (rank 0: the last rank's)
                L[g].hist()[1].copy_(L[(g - 1) % G].hist()[0])
            for g in range(G):
                L[g].scan_mid()
            recs = torch.cat([L[g].records()[0] for g in range(G)])
            for g in range(G):
                L[g].records()[1].copy_(recs)
            for g in range(G):
                L[g].scan_end(xs[g])
        for g in range(G):
            L[g].attn_begin(xs[g])
        split = [L[g].window_split() for g in range(G)] if self.overlap else None
        if self.overlap:
            for g in range(G):
                top, bot, _ = split[g]
                L[g].attn_windows(top, bot)
        for g in range(G):
            sp, sn, rp, rn = L[g].halo()
            if rp.numel():
                rp.copy_(L[g - 1].halo()[1])
            if rn.numel():
                rn.copy_(L[g + 1].halo()[0])
        for g in range(G):
            if self.overlap:
                top, bot, nwy = split[g]
                L[g].attn_windows(0, top)
                L[g].attn_windows(bot, nwy)
                L[g].out_proj(xs[g], outs[g])
            else:
                L[g].attn_end(xs[g], outs[g])
        return torch.cat(outs, dim=1)


class NcclComm:
    """A communicator owned by libpscwin (pscwin_nccl_comm_init) for pscwin_dist_forward: rank 0 creates the NCCL
    unique id and torch.distributed broadcasts it (any backend); world = 1 needs no process group."""

    def __init__(self, rank: int = 0, world: int = 1):
        import numpy as np
        idb = np.zeros(128, dtype=np.uint8)
        if rank == 0:
            check(lib().pscwin_nccl_get_unique_id(idb.ctypes.data), "nccl_get_unique_id")
        if world > 1:
            import torch.distributed as tdist
            obj = [idb.tobytes()]
            tdist.broadcast_object_list(obj, src=0)
            idb = np.frombuffer(obj[0], dtype=np.uint8).copy()
        self.ptr = ctypes.c_void_p()
        check(lib().pscwin_nccl_comm_init(idb.ctypes.data, world, rank, ctypes.byref(self.ptr)), "nccl_comm_init")
        self.rank, self.world = rank, world

    def close(self):
        """ncclCommDestroy; call only after every CUDA graph that captured operations on this communicator has
        been destroyed (NCCL waits for them)."""
        if self.ptr:
            lib().pscwin_nccl_comm_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()

    def check(self) -> None:
        """Raise PscwinError(ERR_NCCL) if NCCL reports an asynchronous error on this communicator."""
        check(lib().pscwin_nccl_comm_check(self.ptr), "nccl_comm_check")

    def abort(self) -> None:
        """ncclCommAbort: cancel every outstanding operation; the communicator cannot be used again."""
        if self.ptr:
            lib().pscwin_nccl_comm_abort(self.ptr)
            self.ptr = ctypes.c_void_p()

    def wait(self, stream=None, timeout_s: float = 0.0) -> None:
        """Wait for `stream` (default: torch's current stream) to drain while watching the communicator: on an
        asynchronous NCCL error or after timeout_s (> 0) seconds the communicator is aborted and PscwinError
        (ERR_NCCL / ERR_TIMEOUT) raised -- a stalled or failed peer surfaces as an error instead of a hang."""
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = lib().pscwin_nccl_wait(self.ptr, s.cuda_stream, int(timeout_s * 1000))
        if rc in (ERR_NCCL, ERR_TIMEOUT):
            self.ptr = ctypes.c_void_p()  # aborted inside the library
        check(rc, "nccl_wait")


class DistLayer:
    """One PSCWin layer on this rank's band, exchanges inside the library over NCCL (pscwin_dist_forward). With
    overlap=True the QKV halo exchange runs on a second (comm) stream while the interior windows compute."""

    def __init__(self, desc: LayerDesc, weights: Dict[str, torch.Tensor], row_begin: int, row_end: int,
                 comm: NcclComm, overlap: bool = True, comm_stream: "torch.cuda.Stream" = None):
        self.desc, self.weights, self.comm = desc, weights, comm
        self.wts = LayerWeights.from_tensors(weights)
        self.r0, self.r1 = row_begin, row_end
        n = int(lib().pscwin_dist_workspace_bytes(ctypes.byref(desc), row_begin, row_end, comm.rank, comm.world))
        if n == 0:
            raise ValueError("invalid band for this layer")
        dev = next(iter(weights.values())).device
        self.ws = torch.empty(n, dtype=torch.uint8, device=dev)
        self.comm_stream = (comm_stream or torch.cuda.Stream(device=dev)) if overlap else None

    def __call__(self, x_band: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
        out = torch.empty_like(x_band) if out is None else out
        check(lib().pscwin_dist_forward(ctypes.byref(self.desc), ctypes.byref(self.wts), _ptr(x_band), _ptr(out),
                                        self.r0, self.r1, self.comm.ptr, self.ws.data_ptr(), self.ws.numel(),
                                        _stream(), self.comm_stream.cuda_stream if self.comm_stream else None),
              "dist_forward")
        return out
