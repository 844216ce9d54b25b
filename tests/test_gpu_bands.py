"""Window-row sharding on one GPU: every band of the image runs its own phases and the
bands exchange the conv history, the scan records and the QKV halo rows by device copies (the bytes NCCL moves
between GPUs). The stitched output must equal pscwin_forward on the whole image — bit-identical for attention
layers, within fp32 summation-order noise for cycle-scan layers (different chunking) — and the oracle."""
import pytest

import oracle
import synth
from gpu_util import BF16_TOL, X_SCALE, dev, dev_weights, host, layer_gate, n_residual, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2407_02109_b200 as p
    return p


CASES = [
    (synth.tiny(H=32, W=16, shift_x=0, shift_y=0), 2),                    # P
    (synth.tiny(H=32, W=16), 2),                                           # S, learnable
    (synth.tiny(H=32, W=16), 4),
    (synth.tiny(H=40, W=24, shift_x=3, shift_y=5), 3),                     # asymmetric shift: 5 / 3 halo rows
    (synth.tiny(H=36, W=16, pad_mode=synth.PAD_MASKED), 3),                # ragged tail joins the last band
    (synth.tiny(H=34, W=16), 3),                                           # 2-row ragged tail, shift 4
    (synth.tiny(H=36, W=16, shift_x=4, shift_y=5, cycle_scan=1), 3),       # 5-row halo to the previous rank
    (synth.tiny(H=32, W=16, cycle_scan=1, shift_x=0, shift_y=0), 2),       # CS + P
    (synth.tiny(H=32, W=16, cycle_scan=1), 4),                             # CS + S
    (synth.tiny(H=32, W=16, cycle_scan=1, bbar_mode=synth.BBAR_EULER), 3),
    (synth.vitb(64, cycle_scan=1), 4),                                     # ViT-B 1024^2 as 4 bands
    (synth.tiny(H=32, W=16, cycle_scan=1, mlp_hidden=256), 2),             # CS + S + FFN
    (synth.tiny(H=32, W=16, cycle_scan=1, scan_order=synth.SCAN_WINDOW_MAJOR), 4),   # window-major segments
    (synth.tiny(H=48, W=24, cycle_scan=1, shift_x=0, shift_y=0, scan_order=synth.SCAN_WINDOW_MAJOR), 3),
]


@pytest.mark.parametrize("cfg,world", CASES, ids=lambda c: str(c) if isinstance(c, int) else
                         f"{c.H}x{c.W}C{c.C}s{c.shift_x},{c.shift_y}m{c.pad_mode}cs{c.cycle_scan}b{c.bbar_mode}f{c.mlp_hidden}"
                         f"o{c.scan_order}")
def test_bands_equal_whole_image(pl, cfg, world):
    import torch
    from paper_2407_02109_b200.bands import LoopbackBands
    x, w = synth.make_input(cfg, scale=X_SCALE), synth.make_weights(cfg)
    dw = dev_weights(w, cfg)
    desc = pl.LayerDesc.from_config(cfg)
    xd = dev(x)
    whole = pl.PSCWinLayer(desc, dw)(xd)
    banded = LoopbackBands(desc, dw, world)(xd)
    torch.cuda.synchronize()
    if cfg.cycle_scan:  # different chunk boundaries: fp32 summation order, then bf16 rounding (2 ulp at max scale)
        assert rel_err(host(banded), host(whole)) < 8e-3
    else:
        assert torch.equal(banded, whole)
    ref = oracle.pscwin_layer(x, w, cfg)
    assert rel_err(host(banded), ref) < BF16_TOL
    assert layer_gate(host(banded), x, ref, n_residual(cfg)) < 1.0


@pytest.mark.parametrize("cfg,world", [(synth.tiny(H=32, W=16), 4), (synth.tiny(H=40, W=24, shift_x=3, shift_y=5), 3),
                                       (synth.tiny(H=34, W=16, cycle_scan=1), 3), (synth.vitb(64, B=1), 4)],
                         ids=["S4", "asym3", "ragged_cs3", "vitb4"])
def test_bands_overlap_schedule_equals_whole_image(pl, cfg, world):
    # the pscwin_dist_forward overlap schedule: interior window rows before the halo arrives, band-edge window rows
    # after, then out-proj — stitched bit-identical to the one-launch band schedule (and the whole image for
    # attention layers); the interior rows must not read any halo row: the halo buffers hold garbage until copied
    import torch
    from paper_2407_02109_b200.bands import LoopbackBands
    x, w = synth.make_input(cfg, scale=X_SCALE), synth.make_weights(cfg)
    dw = dev_weights(w, cfg)
    desc = pl.LayerDesc.from_config(cfg)
    xd = dev(x)
    plain = LoopbackBands(desc, dw, world)(xd)
    ov = LoopbackBands(desc, dw, world, overlap=True)
    for layer in ov.layers:
        layer.ws.fill_(0x7F)   # NaN-ish bf16 garbage everywhere, including the halo rows, before the first call
    got = ov(xd)
    torch.cuda.synchronize()
    assert torch.equal(got, plain)
    tops = [layer.window_split() for layer in ov.layers]
    assert all(0 <= t <= b <= n for t, b, n in tops)
    assert tops[0][0] == 0 and tops[-1][1] == tops[-1][2]          # image edges have no halo
    if not cfg.cycle_scan:
        assert torch.equal(got, pl.PSCWinLayer(desc, dw)(xd))


def test_band_contract(pl):
    from paper_2407_02109_b200.bands import BandLayer
    cfg = synth.tiny(H=32, W=16)
    desc = pl.LayerDesc.from_config(cfg)
    dw = dev_weights(synth.make_weights(cfg), cfg)
    with pytest.raises(ValueError):
        BandLayer(desc, dw, 4, 20, 1, 2)  # not whole window rows


_NCCL_CASE = r"""
import os, sys
os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")   # single-node bootstrap over loopback
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import torch, numpy as np, synth, oracle
import paper_2407_02109_b200 as pl
from paper_2407_02109_b200.bands import DistLayer, NcclComm
from gpu_util import BF16_TOL, X_SCALE, dev, dev_weights, host, layer_gate, n_residual, rel_err
cfg = [synth.tiny(H=32, W=16), synth.tiny(H=32, W=16, cycle_scan=1, mlp_hidden=128), synth.vitb(64, cycle_scan=1)][{i}]
x, w = synth.make_input(cfg, scale=X_SCALE), synth.make_weights(cfg)
dw = dev_weights(w, cfg)
desc = pl.LayerDesc.from_config(cfg)
xd = dev(x)
whole = pl.PSCWinLayer(desc, dw)(xd)
comm = NcclComm(0, 1)
layer = DistLayer(desc, dw, 0, cfg.H, comm)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
xin = xd[0].contiguous()
with torch.cuda.stream(s):
    got = layer(xin)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
if cfg.cycle_scan:
    assert rel_err(host(got), host(whole[0])) < 8e-3
else:
    assert torch.equal(got, whole[0])
ref = oracle.pscwin_layer(x, w, cfg)
assert rel_err(host(got)[None], ref) < BF16_TOL
assert layer_gate(host(got)[None], x, ref, n_residual(cfg)) < 1.0
out = torch.empty_like(got)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    layer(xin, out=out)
out.zero_()
g.replay()
torch.cuda.synchronize()
assert torch.equal(out, got)
print("ok", flush=True)
# (the communicator is not destroyed here: ncclCommDestroy waits while a CUDA graph holding its operations is
# alive; the process exit releases both)
os._exit(0)
"""


@pytest.mark.parametrize("i", [0, 1, 2])
def test_dist_forward_nccl_world1(pl, i):
    # pscwin_dist_forward with a library-owned NCCL communicator of one rank: the in-library ring / all-gather
    # exchanges run for real; the whole image as one band equals pscwin_forward, and the call captures into a
    # CUDA graph (NCCL operations on the layer's stream). Run in a subprocess with a timeout: an NCCL bootstrap
    # problem must fail the test, not hang the suite.
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _NCCL_CASE.format(root=root, tests=os.path.join(root, "tests"), i=i)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


_NCCL_WATCHDOG = r'''
import sys
sys.path.insert(0, {root!r})
import torch
import paper_2407_02109_b200 as pl
from paper_2407_02109_b200.bands import NcclComm
from paper_2407_02109_b200._lib import ERR_TIMEOUT, PscwinError
c = NcclComm(0, 1)
c.check()                                   # no asynchronous error on a fresh communicator
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    torch.cuda._sleep(3_000_000_000)        # a stream that does not drain (~1.5 s of spinning): a stalled peer
try:
    c.wait(s, timeout_s=0.05)
    raise SystemExit("no timeout")
except PscwinError as e:
    assert e.status == ERR_TIMEOUT, e
assert not c.ptr                            # the watchdog aborted the communicator
torch.cuda.synchronize()
c2 = NcclComm(0, 1)                         # a new communicator works after the abort
c2.check()
c2.wait(timeout_s=10.0)
c2.abort()
print("ok")
'''


def test_nccl_watchdog_times_out_and_aborts(pl):
    # failure detection of the multi-GPU path: pscwin_nccl_wait turns a stream that never drains into
    # PSCWIN_ERR_TIMEOUT and aborts the communicator instead of hanging; a fresh communicator works afterwards
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _NCCL_WATCHDOG.format(root=root)], capture_output=True, text=True,
                       timeout=240)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
