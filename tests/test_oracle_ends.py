"""Pins for the encoder-end oracle functions (reading Q22), CPU only: each against the torch
fp64 library routine it restates (conv2d, interpolate, layer_norm) plus the paper's shape law (a 1024^2
image gives 64 x 64 tokens; the stages' output dimension is 256)."""
import numpy as np
import torch
import torch.nn.functional as F

import oracle
import synth


def test_patch_embed_vs_conv2d_and_shape():
    rng = np.random.default_rng(0)
    img = rng.standard_normal((2, 3, 64, 48))
    w, b = rng.standard_normal((32, 3, 16, 16)), rng.standard_normal(32)
    got = oracle.patch_embed(img, w, b)
    ref = F.conv2d(torch.from_numpy(img), torch.from_numpy(w), torch.from_numpy(b), stride=16).numpy()
    assert got.shape == (2, 4, 3, 32)
    assert np.max(np.abs(got - ref.transpose(0, 2, 3, 1))) < 1e-11
    # P:L625 shape law: 1024^2 -> 64 x 64 tokens (ViT-B width)
    assert oracle.patch_embed(np.zeros((1, 3, 1024, 1024)), np.zeros((768, 3, 16, 16)), np.zeros(768)).shape == \
        (1, 64, 64, 768)


def test_conv3x3_vs_conv2d():
    rng = np.random.default_rng(1)
    x, w = rng.standard_normal((2, 7, 5, 6)), rng.standard_normal((4, 6, 3, 3))
    ref = F.conv2d(torch.from_numpy(x.transpose(0, 3, 1, 2)), torch.from_numpy(w), padding=1).numpy()
    assert np.max(np.abs(oracle.conv3x3(x, w) - ref.transpose(0, 2, 3, 1))) < 1e-12


def test_resize_bilinear_vs_interpolate():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((1, 5, 7, 3))
    for H, W in [(10, 14), (16, 16), (5, 7), (3, 20)]:
        ref = F.interpolate(torch.from_numpy(x.transpose(0, 3, 1, 2)), size=(H, W), mode="bilinear",
                            align_corners=False).numpy().transpose(0, 2, 3, 1)
        assert np.max(np.abs(oracle.resize_bilinear(x, H, W) - ref)) < 1e-12
    assert np.array_equal(oracle.resize_bilinear(x, 5, 7), x)  # identity size


def test_neck_vs_torch_and_shape():
    rng = np.random.default_rng(3)
    wt = synth.make_ends_weights(C=64, C_out=32)
    outs = [rng.standard_normal((1, 6, 5, 64)) for _ in range(4)]
    got = oracle.encoder_neck(outs, wt)
    t = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float64))
    f = sum(t(o) @ t(wt[f"w_stage{i}"]).T for i, o in enumerate(outs))
    f = F.layer_norm(f, (32,), t(wt["neck_ln1_g"]), t(wt["neck_ln1_b"]), 1e-6)
    f = F.conv2d(f.permute(0, 3, 1, 2), t(wt["w_neck_conv"]), padding=1).permute(0, 2, 3, 1)
    ref = F.layer_norm(f, (32,), t(wt["neck_ln2_g"]), t(wt["neck_ln2_b"]), 1e-6).numpy()
    assert got.shape == (1, 6, 5, 32)
    assert np.max(np.abs(got - ref)) < 1e-11
