"""GPU parity of the encoder ends (reading Q22) through the C ABI against the fp64 oracle:
patch embedding, bilinear resize (plain and accumulating), the output-fusion neck (one scale; HRSAM++ two scales),
and a whole tiny HRSAMEncoder (patch embedding -> 6 PSCWin layers with FFN -> neck) against the oracle's
composition of the same steps."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import BF16_TOL, dev, dev_weights, host, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2407_02109_b200 as p
    return p


def _ends_dev(w, C):
    import torch
    d = {k: dev(v, "f32" if v.ndim == 1 else "bf16") for k, v in w.items()}
    d["w_patch"] = dev(w["w_patch"].reshape(C, -1))
    d["w_neck_conv"] = dev(np.ascontiguousarray(w["w_neck_conv"].transpose(0, 2, 3, 1)))  # [o, dy, dx, i]
    torch.cuda.synchronize()
    return d


@pytest.mark.parametrize("B,H,W,C", [(1, 4, 6, 64), (2, 8, 8, 128), (1, 64, 64, 768)])
def test_patch_embed(pl, B, H, W, C):
    img = synth.make_image(B, H, W)
    w = synth.make_ends_weights(C=C, C_out=64)
    d = _ends_dev(w, C)
    got = host(pl.patch_embed(dev(img), d["w_patch"], d["b_patch"]))
    ref = oracle.patch_embed(img, w["w_patch"], w["b_patch"])
    assert rel_err(got, ref) < BF16_TOL


@pytest.mark.parametrize("h,w,H,W,C", [(5, 7, 10, 14, 16), (32, 32, 64, 64, 256), (8, 8, 8, 8, 64),
                                        (32, 32, 256, 256, 64)])
def test_resize_bilinear(pl, h, w, H, W, C):
    import torch
    rng = np.random.default_rng(h * w)
    x = synth.round_bf16(rng.standard_normal((2, h, w, C)))
    base = synth.round_bf16(rng.standard_normal((2, H, W, C)))
    got = host(pl.resize_bilinear(dev(x), H, W))
    acc = dev(base)
    pl.resize_bilinear(dev(x), H, W, out=acc)
    torch.cuda.synchronize()
    ref = oracle.resize_bilinear(x, H, W)
    assert rel_err(got, ref) < 1e-2
    assert rel_err(host(acc), ref + base) < 1e-2
    if (h, w) == (H, W):
        assert np.array_equal(got, x)  # identity size: exact copy


@pytest.mark.parametrize("scales", [[(8, 6)], [(16, 16), (8, 8)], [(64, 64), (32, 32)]])
def test_neck(pl, scales):
    C, Co, B = 128, 64, 2
    w = synth.make_ends_weights(C=C, C_out=Co)
    d = _ends_dev(w, C)
    rng = np.random.default_rng(len(scales))
    outs = [synth.round_bf16(rng.standard_normal((B * sum(h * ww for h, ww in scales), C))) for _ in range(4)]
    desc = pl.NeckDesc.make(B, C, Co, scales)
    got = host(pl.neck(desc, [dev(o) for o in outs], d))
    # oracle: per scale stage sum, other scales resized onto scale 0 and added, then the conv block
    off = oracle.ms_offsets(scales)
    f = None
    for j, (h, ww) in enumerate(scales):
        fj = sum(o[B * off[j]:B * off[j + 1]].reshape(B, h, ww, C) @ w[f"w_stage{i}"].T for i, o in enumerate(outs))
        f = fj if f is None else f + oracle.resize_bilinear(fj, scales[0][0], scales[0][1])
    f = oracle.layer_norm(f, w["neck_ln1_g"], w["neck_ln1_b"], 1e-6)
    f = oracle.conv3x3(f, w["w_neck_conv"])
    ref = oracle.layer_norm(f, w["neck_ln2_g"], w["neck_ln2_b"], 1e-6)
    if len(scales) == 1:  # the oracle's neck itself
        ref1 = oracle.encoder_neck([o.reshape(B, *scales[0], C) for o in outs], w)
        assert np.max(np.abs(ref - ref1)) < 1e-9
    assert rel_err(got, ref) < BF16_TOL


def test_hrsam_encoder_tiny(pl):
    # patch embedding -> 6 layers (P, S, CS+P, S, P, CS+S; FFN) with stage ends after layers 2 and 5 -> neck
    import torch
    C, H, W = 64, 16, 16
    cfg = synth.tiny(H=H, W=W, mlp_hidden=128)
    kinds = [synth.stack_layer_kind(i) for i in range(6)]
    cfgs = [cfg.replace(shift_x=4 if s else 0, shift_y=4 if s else 0, cycle_scan=int(cs)) for s, cs in kinds]
    ws = [synth.make_weights(c, layer=i) for i, c in enumerate(cfgs)]
    ends = synth.make_ends_weights(C=C, C_out=64, n_stages=2)
    layers = [pl.PSCWinLayer(pl.LayerDesc.from_config(c), dev_weights(w, c)) for c, w in zip(cfgs, ws)]
    enc = pl.HRSAMEncoder(layers, _ends_dev(ends, C), 1, H, W, stage_ends=(2, 5), C=C, C_out=64, graph=True)
    img = synth.make_image(1, H, W)
    got = host(enc(dev(img)))
    torch.cuda.synchronize()
    x = oracle.patch_embed(img, ends["w_patch"], ends["b_patch"])
    stages = []
    for j, (c, w) in enumerate(zip(cfgs, ws)):
        x = oracle.pscwin_layer(synth.round_bf16(x), w, c)   # the GPU stores x in bf16 between layers
        if j in (2, 5):
            stages.append(x)
    ref = oracle.encoder_neck(stages, ends)
    assert got.shape == (1, H, W, 64)
    assert rel_err(got, ref) < BF16_TOL


def test_hrsampp_encoder_tiny(pl):
    # HRSAM++ (P:L174-189): main 16x16 grid + 8x8 overview (the 512^2-overview role at tiny scale), each image
    # patch-embedded into its slice of the packed sequence -> 6 multi-scale blocks (P, S, CS+P, S, P, CS+S; the
    # cycle-scan blocks single-scale, each stage closed by a multi-scale cycle-scan module) -> neck over both scales
    # (the overview's stage sum resized onto the main grid, reading Q22), against the oracle's composition.
    import torch
    C, B = 64, 1
    scales = [(16, 16), (8, 8)]
    base = synth.tiny(H=16, W=16, mlp_hidden=128)
    specs = []  # (cfg, attention, cs mode, weight seed)
    for i in range(6):
        shifted, cs = synth.stack_layer_kind(i)
        specs.append((base.replace(shift_x=4 if shifted else 0, shift_y=4 if shifted else 0), 1, 1 if cs else 0, i))
        if cs:
            specs.append((base.replace(shift_x=0, shift_y=0, mlp_hidden=0), 0, 2, 100 + i))
    stage_ends = tuple(j for j, sp in enumerate(specs) if sp[1] == 0)   # after each stage's multi-scale module
    ws = [synth.make_weights(c, layer=seed) for c, _, _, seed in specs]
    ends = synth.make_ends_weights(C=C, C_out=64, n_stages=len(stage_ends))
    layers = [pl.PSCWinMSLayer(pl.MSDesc.make(c, scales, att, cs), dev_weights(w, c))
              for (c, att, cs, _), w in zip(specs, ws)]
    enc = pl.HRSAMEncoder(layers, _ends_dev(ends, C), B, *scales[0], stage_ends=stage_ends, C=C, C_out=64,
                          scales=scales)
    imgs = [synth.make_image(B, h, w, seed=50 + i) for i, (h, w) in enumerate(scales)]
    got = host(enc([dev(im) for im in imgs]))
    torch.cuda.synchronize()
    xp = oracle.ms_pack([oracle.patch_embed(im, ends["w_patch"], ends["b_patch"]) for im in imgs])
    stages = []
    for j, ((c, att, cs, _), w) in enumerate(zip(specs, ws)):
        xp = oracle.ms_layer(synth.round_bf16(xp), w, c, scales, att, cs)   # the GPU stores x in bf16
        if j in stage_ends:
            stages.append(synth.round_bf16(xp))
    off = oracle.ms_offsets(scales)
    f = None
    for s, (h, w) in enumerate(scales):
        fs = sum(o[B * off[s]:B * off[s + 1]].reshape(B, h, w, C) @ ends[f"w_stage{i}"].T for i, o in enumerate(stages))
        f = fs if f is None else f + oracle.resize_bilinear(fs, *scales[0])
    f = oracle.layer_norm(f, ends["neck_ln1_g"], ends["neck_ln1_b"], 1e-6)
    f = oracle.conv3x3(f, ends["w_neck_conv"])
    ref = oracle.layer_norm(f, ends["neck_ln2_g"], ends["neck_ln2_b"], 1e-6)
    assert got.shape == (B, *scales[0], 64)
    assert rel_err(got, ref) < BF16_TOL
    # the overview image matters: dropping its contribution moves the embedding by more than the tolerance
    enc_only = [np.zeros_like(imgs[1])]
    got0 = host(enc([dev(imgs[0]), dev(enc_only[0])]))
    assert rel_err(got0, ref) > 3 * BF16_TOL
