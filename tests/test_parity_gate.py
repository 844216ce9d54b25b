"""CPU tests of the parity machinery itself (no GPU):

* the oracle's RoPE against hand-computed worked values (tests/golden/rope_2d_d8.txt, reading
  Q6), so a mis-transcribed frequency schedule or pairing fails (the invariant pins of test_oracle_pins.py hold for
  every schedule and pairing);
* negative controls of the layer-level gate (gpu_util.layer_gate): an identity layer, a layer whose attention,
  cycle-scan module or FFN is zeroed, must FAIL the gate the GPU layer tests apply (VERDICT r1 "What's weak" 3).
"""
import numpy as np
import pytest

import oracle
import synth
from conftest import read_golden
from gpu_util import X_SCALE, layer_gate, masked_w_out, n_residual


def test_rope_golden_values():
    rows = read_golden("rope_2d_d8.txt")
    t = np.arange(1.0, 9.0)
    assert len(rows) == 3
    for r in rows:
        X, Y, want = r[0], r[1], np.array(r[2:], dtype=np.float64)
        got = oracle.rope_2d(t, np.float64(X), np.float64(Y))
        assert np.max(np.abs(got - want)) < 1e-14, (X, Y, got, want)


def test_rope_golden_rejects_plausible_mistranscriptions():
    # the golden values distinguish the reading from its near neighbours: theta_j = 10000^(-2j/d), half-split
    # (non-interleaved) pairs, and swapped axes
    rows = read_golden("rope_2d_d8.txt")
    t = np.arange(1.0, 9.0)

    def variant(tt, X, Y, theta_exp, interleaved=True, swap=False):
        d = tt.shape[-1]
        q = d // 4
        theta = 10000.0 ** (-theta_exp * np.arange(q) / d)
        out = tt.copy()
        if swap:
            X, Y = Y, X
        for half, pos in ((0, X), (1, Y)):
            ang = pos * theta
            base = half * (d // 2)
            i0 = base + (2 * np.arange(q) if interleaved else np.arange(q))
            i1 = i0 + (1 if interleaved else q)
            a, b = tt[i0], tt[i1]
            out[i0] = a * np.cos(ang) - b * np.sin(ang)
            out[i1] = a * np.sin(ang) + b * np.cos(ang)
        return out

    for r in rows:
        X, Y, want = r[0], r[1], np.array(r[2:])
        assert np.max(np.abs(variant(t, X, Y, 4.0) - want)) < 1e-14            # the reading itself
        assert np.max(np.abs(variant(t, X, Y, 2.0) - want)) > 1e-3              # 10000^(-2j/d)
        assert np.max(np.abs(variant(t, X, Y, 4.0, interleaved=False) - want)) > 1e-3
        assert np.max(np.abs(variant(t, X, Y, 4.0, swap=True) - want)) > 1e-3


GATE_CASES = [synth.tiny(), synth.tiny(shift_x=0, shift_y=0, cycle_scan=1),
              synth.tiny(cycle_scan=1, mlp_hidden=320, H=12, W=20), synth.tiny(pad_mode=synth.PAD_MASKED)]


@pytest.mark.parametrize("cfg", GATE_CASES, ids=lambda c: f"s{c.shift_x}m{c.pad_mode}cs{c.cycle_scan}f{c.mlp_hidden}")
def test_layer_gate_negative_controls(cfg):
    x, w = synth.make_input(cfg, scale=X_SCALE), synth.make_weights(cfg)
    ref = oracle.pscwin_layer(x, w, cfg)
    n_res = n_residual(cfg)
    # the exact answer passes; bf16 storage rounding of the exact answer passes
    assert layer_gate(ref, x, ref, n_res) == 0.0
    assert layer_gate(synth.round_bf16(ref), x, ref, n_res) < 0.5
    # an identity layer fails by a wide margin
    assert layer_gate(x, x, ref, n_res) > 5.0
    # dropping any one sub-layer fails
    ablations = {"attention": dict(w_o=np.zeros_like(w["w_o"]))}
    if cfg.cycle_scan:
        ablations["cycle-scan"] = dict(w_out=np.zeros_like(w["w_out"]))
    if cfg.mlp_hidden:
        ablations["ffn"] = dict(w_fc2=np.zeros_like(w["w_fc2"]))
    for name, repl in ablations.items():
        bad = oracle.pscwin_layer(x, dict(w, **repl), cfg)
        assert layer_gate(bad, x, ref, n_res) > 3.0, name
    # a 5 % error in the increment fails; a 0.5 % error passes
    inc = ref - x
    assert layer_gate(x + 1.05 * inc, x, ref, n_res) > 1.0
    assert layer_gate(x + 1.005 * inc, x, ref, n_res) < 1.0


def test_varied_scan_parameters_are_channel_dependent():
    # the default synth SSM parameters vary per channel, so a kernel reading A_log / D_skip at the wrong channel
    # index produces a different scan (VERDICT r1 "What's weak" 4)
    cfg = synth.tiny()
    w = synth.make_weights(cfg)
    assert np.ptp(w["d_skip"]) > 0.5
    assert np.min(np.ptp(w["a_log"], axis=0)) > 0.5
    L, D = 40, cfg.D
    xin = synth.round_bf16(0.6 * synth.normal(synth.stream_seed(3, 1), L * D).reshape(1, L, D))
    ref = oracle.cycle_scan(xin, None, w, 5, 8)
    perm = np.roll(np.arange(D), 1)
    wp = dict(w, a_log=w["a_log"][perm], d_skip=w["d_skip"][perm])
    bad = oracle.cycle_scan(xin, None, wp, 5, 8)
    assert np.max(np.abs(bad - ref)) > 0.05 * np.max(np.abs(ref))


@pytest.mark.parametrize("cfg", [synth.tiny(cycle_scan=1), synth.tiny(cycle_scan=1, shift_x=0, shift_y=0,
                                                                       mlp_hidden=128)])
def test_oracle_sampling_is_exact(cfg):
    # the full-size GPU parity cases compare against the oracle evaluated on window rows / SSM channels only;
    # on a tiny layer the sampled evaluation must equal the full one where it is defined
    ch = [0, 5, 77, 127]
    x, w = synth.make_input(cfg, scale=X_SCALE), masked_w_out(synth.make_weights(cfg), ch)
    full = oracle.pscwin_layer(x, w, cfg)
    rows = [1]
    samp = oracle.pscwin_layer(x, w, cfg, window_rows=rows, channels=ch)
    sel = ~np.isnan(samp)
    assert sel.sum() > 0 and (~sel).sum() > 0
    assert np.max(np.abs(samp[sel] - full[sel])) < 1e-13
    with pytest.raises(ValueError):
        oracle.pscwin_layer(x, synth.make_weights(cfg), cfg, channels=ch)   # unmasked W_out: not exact, refused
    scales = [(16, 16), (8, 8)]
    xp = np.concatenate([synth.make_input(cfg.replace(H=h, W=ww), layer=i, scale=X_SCALE).reshape(-1, cfg.C)
                         for i, (h, ww) in enumerate(scales)])
    for mode in (oracle.CS_SINGLE_SCALE, oracle.CS_MULTI_SCALE):
        f = oracle.ms_layer(xp, w, cfg, scales, 1, mode)
        sp = oracle.ms_layer(xp, w, cfg, scales, 1, mode, window_rows=[[1], [0]], channels=ch)
        sel = ~np.isnan(sp)
        assert sel.sum() > 0 and np.max(np.abs(sp[sel] - f[sel])) < 1e-13
