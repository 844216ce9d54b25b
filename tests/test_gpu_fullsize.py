"""GPU parity at the sizes bench.py times (BASELINE.json configs[2]-[4]), in the launch configuration it uses
(whole-layer pscwin_forward / pscwin_ms_forward, ViT-B widths), against the fp64 oracle evaluated on samples it can
afford: padded-grid window rows of the attention sub-layer (exact for those windows: each window depends only on
its own cells) and SSM channels of the cycle-scan module (exact when W_out is zero outside them:
gpu_util.masked_w_out; the GPU still computes every channel). LN, every projection, RoPE at all coordinates, the
conv and x_proj run over the full token set on both sides.

The gate is the increment gate of the layer tests (gpu_util.layer_gate) on a small residual stream, restricted to
the sampled tokens.
"""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import BF16_TOL, X_SCALE, dev, dev_weights, host, masked_w_out, n_residual, rel_err, sampled_gate

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CH = [0, 1, 700, 1535]     # sampled SSM channels (first, second, interior, last of D = 1536)


@pytest.fixture(scope="module")
def pl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2407_02109_b200 as p
    return p


def _run_layer(pl, cfg, w, x):
    import torch
    got = host(pl.PSCWinLayer(pl.LayerDesc.from_config(cfg), dev_weights(w, cfg))(dev(x)))
    torch.cuda.synchronize()
    return got


def test_qkv_rope_4096(pl):
    # a4 over all 65536 tokens: the GPU RoPE epilogue at every grid coordinate 0..255 against oracle.rope_2d
    cfg = synth.vitb(256, shift_x=0, shift_y=0)
    x, w = synth.make_input(cfg), synth.make_weights(cfg)
    qkv, _ = pl.qkv_project(pl.LayerDesc.from_config(cfg), dev_weights(w, cfg), dev(x))
    u = oracle.layer_norm(x, w["ln1_g"], w["ln1_b"], cfg.ln_eps)
    ref = (u @ w["w_qkv"].T + w["b_qkv"]).reshape(1, 256, 256, 3, cfg.heads, cfg.d_head)
    yy, xx = np.meshgrid(np.arange(256), np.arange(256), indexing="ij")
    for i in (0, 1):
        ref[:, :, :, i] = oracle.rope_2d(ref[:, :, :, i], xx[None, :, :, None], yy[None, :, :, None])
    got = host(qkv).reshape(ref.shape)
    assert rel_err(got, ref) < BF16_TOL
    # per-coordinate check on the last rows / columns (largest rotation angles): q and k of every head
    assert rel_err(got[:, 240:, 240:, :2], ref[:, 240:, 240:, :2]) < BF16_TOL


@pytest.mark.parametrize("shift,mode", [(0, synth.PAD_LEARNABLE), (8, synth.PAD_LEARNABLE), (8, synth.PAD_MASKED)],
                         ids=["P", "S-learnable", "S-masked"])
def test_layer_4096_sampled(pl, shift, mode):
    # configs[3]: one 4096^2 image (256 x 256 tokens), attention layer as bench.py runs it
    cfg = synth.vitb(256, shift_x=shift, shift_y=shift, pad_mode=mode)
    x, w = synth.make_input(cfg, scale=X_SCALE), synth.make_weights(cfg)
    got = _run_layer(pl, cfg, w, x)
    rows = [0, 7, 16] if shift else [0, 8, 15]   # first (pad) / interior / last (pad) window rows
    ref = oracle.pscwin_layer(x, w, cfg, window_rows=rows)
    assert sampled_gate(got, x, ref, n_residual(cfg)) < 1.0


def test_cs_layer_4096_sampled(pl):
    # CS + S at 4096^2: the scan over the cycled 3 x 65536-token sequence, sampled SSM channels, sampled windows
    cfg = synth.vitb(256, cycle_scan=1)
    x, w = synth.make_input(cfg, scale=X_SCALE), masked_w_out(synth.make_weights(cfg), CH)
    got = _run_layer(pl, cfg, w, x)
    ref = oracle.pscwin_layer(x, w, cfg, window_rows=[0, 16], channels=CH)
    assert sampled_gate(got, x, ref, n_residual(cfg)) < 1.0


def test_cs_layer_2048_b8_sampled(pl):
    # configs[2]: 2048^2 inputs (128 x 128 tokens), batch 8 per GPU; CS + S layer, every image sampled
    cfg = synth.vitb(128, B=8, cycle_scan=1)
    x, w = synth.make_input(cfg, scale=X_SCALE), masked_w_out(synth.make_weights(cfg), CH)
    got = _run_layer(pl, cfg, w, x)
    ref = oracle.pscwin_layer(x, w, cfg, window_rows=[0, 4, 8], channels=CH)
    assert sampled_gate(got, x, ref, n_residual(cfg)) < 1.0


@pytest.mark.parametrize("cs", [oracle.CS_SINGLE_SCALE, oracle.CS_MULTI_SCALE], ids=["SS", "MS"])
def test_ms_config5_sampled(pl, cs):
    # configs[4]: HRSAM++ multi-scale, 64^2 + 128^2 + 256^2 token grids packed per sample, B = 2 per GPU (batch 16
    # over 8 GPUs); shifted learnable attention after a single- or multi-scale cycle-scan module
    import torch
    scales = [(64, 64), (128, 128), (256, 256)]
    B = 2
    cfg = synth.vitb(64, B=B)
    xp = np.concatenate([synth.make_input(cfg.replace(H=h, W=ww), layer=i, scale=X_SCALE).reshape(-1, cfg.C)
                         for i, (h, ww) in enumerate(scales)])
    w = masked_w_out(synth.make_weights(cfg), CH)
    layer = pl.PSCWinMSLayer(pl.MSDesc.make(cfg, scales, 1, cs), dev_weights(w, cfg))
    got = host(layer(dev(xp)))
    torch.cuda.synchronize()
    ref = oracle.ms_layer(xp, w, cfg, scales, 1, cs, window_rows=[[0], [4], [0, 16]], channels=CH)
    assert sampled_gate(got, xp, ref, n_residual(cfg, 1, cs)) < 1.0


@pytest.mark.parametrize("cs", [0, 1], ids=["S", "CS+S"])
def test_bands_4096_eight(pl, cs):
    # configs[3] row split: the 4096^2 image as 8 window-row bands (32 token rows each) with halo / conv-history /
    # scan-record exchanges (loopback copies of the NCCL bytes) == the whole-image layer; band-edge windows vs oracle
    import torch
    from paper_2407_02109_b200.bands import LoopbackBands
    cfg = synth.vitb(256, cycle_scan=cs)
    x, w = synth.make_input(cfg, scale=X_SCALE), masked_w_out(synth.make_weights(cfg), CH)
    dw = dev_weights(w, cfg)
    desc = pl.LayerDesc.from_config(cfg)
    xd = dev(x)
    whole = pl.PSCWinLayer(desc, dw)(xd)
    banded = LoopbackBands(desc, dw, 8)(xd)
    torch.cuda.synchronize()
    if cs:
        assert rel_err(host(banded), host(whole)) < 8e-3
    else:
        assert torch.equal(banded, whole)
    # padded-grid window rows 2 and 4 straddle the band edges at token rows 32 and 64 (pad_top = 8)
    ref = oracle.pscwin_layer(x, w, cfg, window_rows=[2, 4], channels=CH if cs else None)
    assert sampled_gate(host(banded), x, ref, n_residual(cfg)) < 1.0
