"""GPU parity of the HRSAM++ multi-scale layer through the C ABI
(pscwin_ms_forward) against the fp64 oracle (oracle.ms_layer) on the same seeded inputs.

Cases: plain / padded-shift (learnable and masked) attention over packed scales, single-scale and multi-scale
cycle-scan modules (B = 1: no gather; B = 2 and window-major order: the multi-scale gather / scatter), the
cycle-scan-only module, ragged scale grids under shifted windows, and a ViT-B-width case. Index maps bit-exact.
"""
import numpy as np
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


def _packed(cfg, scales, B, scale=X_SCALE):
    grids = [synth.make_input(cfg.replace(B=B, H=h, W=w), layer=i, scale=scale) for i, (h, w) in enumerate(scales)]
    return oracle.ms_pack(grids)


def _run(pl, cfg, scales, B, attention, cs):
    import torch
    xp = _packed(cfg, scales, B)
    w = synth.make_weights(cfg.replace(H=scales[0][0], W=scales[0][1]))
    desc = pl.MSDesc.make(cfg.replace(B=B), scales, attention, cs)
    layer = pl.PSCWinMSLayer(desc, dev_weights(w, cfg))
    got = host(layer(dev(xp)))
    torch.cuda.synchronize()
    ref = oracle.ms_layer(xp, w, cfg.replace(B=B), scales, attention, cs)
    return xp, got, ref


def test_ms_index_map_bit_exact(pl):
    for scales, w, sx, sy in [([(4, 4), (2, 2)], 2, 0, 0), ([(16, 16), (8, 8), (24, 8)], 8, 4, 4),
                              ([(12, 20), (7, 9)], 4, 1, 3)]:
        desc = pl.MSDesc.make(synth.tiny(window=w, shift_x=sx, shift_y=sy), scales)
        assert np.array_equal(pl.ms_index_map(desc), oracle.ms_index_map(scales, w, sx, sy))


CS = {"none": 0, "ss": 1, "ms": 2}
CASES = [
    # (cfg, scales, B, attention, cs)
    (synth.tiny(shift_x=0, shift_y=0), [(16, 16), (8, 8)], 1, 1, "none"),
    (synth.tiny(), [(16, 16), (8, 8)], 1, 1, "none"),
    (synth.tiny(pad_mode=synth.PAD_MASKED), [(16, 16), (8, 8), (24, 16)], 2, 1, "none"),
    (synth.tiny(shift_x=3, shift_y=5), [(12, 20), (7, 9)], 1, 1, "none"),          # ragged grids, asym shift
    (synth.tiny(shift_x=0, shift_y=0), [(16, 16), (8, 8)], 1, 1, "ss"),
    (synth.tiny(shift_x=0, shift_y=0), [(16, 16), (8, 8)], 1, 1, "ms"),            # B = 1: packed = sequence
    (synth.tiny(shift_x=0, shift_y=0), [(16, 16), (8, 8), (8, 16)], 2, 1, "ms"),   # gather / scatter
    (synth.tiny(), [(16, 16), (8, 8)], 2, 0, "ms"),                                # cycle-scan module only
    (synth.tiny(shift_x=0, shift_y=0, scan_order=synth.SCAN_WINDOW_MAJOR), [(16, 16), (8, 8)], 1, 1, "ms"),
    (synth.tiny(shift_x=0, shift_y=0, scan_order=synth.SCAN_COL_MAJOR), [(16, 16), (8, 8)], 2, 0, "ss"),
    (synth.tiny(mlp_hidden=256), [(16, 16), (8, 8)], 2, 1, "ss"),                  # + FFN sub-layer
]


@pytest.mark.parametrize("cfg,scales,B,attention,cs", CASES,
                         ids=lambda v: str(v) if not hasattr(v, "H") else f"s{v.shift_x}m{v.pad_mode}o{v.scan_order}f{v.mlp_hidden}")
def test_ms_layer(pl, cfg, scales, B, attention, cs):
    xp, got, ref = _run(pl, cfg, scales, B, attention, CS[cs])
    assert rel_err(got, ref) < BF16_TOL
    # gate on the increment x_out - x (gpu_util.layer_gate; small residual stream X_SCALE)
    assert layer_gate(got, xp, ref, n_residual(cfg, attention, CS[cs])) < 1.0


def test_ms_single_scale_equals_layer_forward(pl):
    # one scale: the multi-scale layer is the single-scale layer (same kernels, same rounding points)
    import torch
    cfg = synth.tiny(cycle_scan=1)
    x = synth.make_input(cfg)
    w = dev_weights(synth.make_weights(cfg), cfg)
    a = pl.PSCWinLayer(pl.LayerDesc.from_config(cfg), w)(dev(x))
    b = pl.PSCWinMSLayer(pl.MSDesc.make(cfg, [(cfg.H, cfg.W)], 1, 1), w)(dev(x.reshape(-1, cfg.C)))
    c = pl.PSCWinMSLayer(pl.MSDesc.make(cfg, [(cfg.H, cfg.W)], 1, 2), w)(dev(x.reshape(-1, cfg.C)))
    torch.cuda.synchronize()
    assert torch.equal(a.reshape(-1, cfg.C), b) and torch.equal(b, c)


def test_ms_vitb_width(pl):
    cfg = synth.vitb(32)
    xp, got, ref = _run(pl, cfg, [(32, 32), (16, 16)], 2, 1, CS["ms"])
    assert rel_err(got, ref) < BF16_TOL


def test_ms_contract(pl):
    import torch
    cfg = synth.tiny(shift_x=0, shift_y=0)
    w = dev_weights(synth.make_weights(cfg), cfg)
    for scales in ([(16, 16), (12, 8)], [(16, 16), (0, 8)]):   # plain windows need divisible grids; empty grid
        desc = pl.MSDesc.make(cfg, scales, 1, 0)
        with pytest.raises(pl.PscwinError):
            pl.PSCWinMSLayer(desc, w)(torch.zeros(16 * 16 + 96, cfg.C, dtype=torch.bfloat16, device="cuda"))
