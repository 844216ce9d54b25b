"""Pins for the multi-scale (HRSAM++) part of the oracle, CPU only (`-m "not gpu"`).

Pinned against: SPEC's worked example of the multi-scale index map (tests/golden), the App. C route
(pad appended at the end of the packed sequence, gather, ONE block-diagonal SDPA over all scales), the
single-scale special case, the independent cycle-scan closed form applied to the concatenated sequence
(test_oracle_pins._closed_form_cycle), and the defining difference of the two cycle-scan modes (single-scale
outputs of one scale never depend on another scale's tokens; multi-scale outputs do).
"""
import numpy as np
import torch
import torch.nn.functional as F

import oracle
import synth
from conftest import read_golden
from test_oracle_pins import _closed_form_cycle

PAD = oracle.PAD


def _packed(cfg, scales, B, seed=0):
    grids = [synth.make_input(cfg.replace(B=B, H=h, W=w), layer=seed + i) for i, (h, w) in enumerate(scales)]
    return oracle.ms_pack(grids), grids


def test_ms_pack_bounds_and_roundtrip():
    # grids 4x4 and 2x2 -> length 20, bounds [0, 16, 20]; unpack(pack(g)) = g bit-exactly
    assert list(oracle.ms_offsets([(4, 4), (2, 2)])) == [0, 16, 20]
    rng = np.random.default_rng(0)
    grids = [rng.standard_normal((3, 4, 4, 5)), rng.standard_normal((3, 2, 2, 5)), rng.standard_normal((3, 6, 2, 5))]
    xp = oracle.ms_pack(grids)
    assert xp.shape == (3 * (16 + 4 + 12), 5)
    for a, b in zip(oracle.ms_unpack(xp, 3, [(4, 4), (2, 2), (6, 2)]), grids):
        assert np.array_equal(a, b)


def test_ms_index_map_worked_example():
    gold = np.array(read_golden("ms_index_map_4x4_2x2_w2.txt"), dtype=np.uint32)
    m = oracle.ms_index_map([(4, 4), (2, 2)], 2).reshape(-1, 4)
    assert np.array_equal(m, gold)


def test_ms_index_map_blocks_stay_in_one_scale():
    scales = [(12, 20), (6, 10), (3, 5)]
    off = oracle.ms_offsets(scales)
    for sx, sy in [(0, 0), (1, 3), (2, 2)]:
        w = 4
        if (sx, sy) == (0, 0):
            scales_t = [(12, 20), (8, 4)]
        else:
            scales_t = scales
        offt = oracle.ms_offsets(scales_t)
        m = oracle.ms_index_map(scales_t, w, sx, sy).reshape(-1, w * w)
        seen = np.zeros(int(offt[-1]), dtype=int)
        for blk in m:
            real = blk[blk != PAD].astype(np.int64)
            assert len(real) > 0
            sc = np.searchsorted(offt, real, side="right") - 1
            assert np.all(sc == sc[0])      # no block spans a scale boundary
            seen[real] += 1
        assert np.all(seen == 1)            # every token in exactly one slot
    del off


def test_ms_attention_single_scale_is_attention_sublayer():
    cfg = synth.tiny(dtype="f32")
    x = synth.make_input(cfg)
    wt = synth.make_weights(cfg)
    got = oracle.ms_attention_sublayer(x.reshape(-1, cfg.C), wt, cfg, [(cfg.H, cfg.W)])
    assert np.array_equal(got, oracle.attention_sublayer(x, wt, cfg).reshape(-1, cfg.C))


def _index_operator_ms(xp, wt, cfg, scales):
    """App. C over the PACKED multi-scale sequence of one sample: append p's projection at
    the sequence end, gather every scale's windows with the multi-scale index map (pad slots -> the appended
    row), RoPE at each cell's scale-local geometric coordinate, ONE block-diagonal SDPA over all scales."""
    C, heads, w = cfg.C, cfg.heads, cfg.window
    d = C // heads
    Lt = xp.shape[0]
    u = oracle.layer_norm(xp, wt["ln1_g"], wt["ln1_b"], cfg.ln_eps)
    seq = np.concatenate([u @ wt["w_qkv"].T + wt["b_qkv"], (wt["pad"] @ wt["w_qkv"].T + wt["b_qkv"])[None]])
    idx, coords = [], []
    base = 0
    for (H, W) in scales:  # independent enumeration: pad left/top = (w - s) mod w, complete windows
        pl, pt = (w - cfg.shift_x) % w, (w - cfg.shift_y) % w
        Wp, Hp = -(-(pl + W) // w) * w, -(-(pt + H) // w) * w
        for wy in range(Hp // w):
            for wx in range(Wp // w):
                for iy in range(w):
                    for ix in range(w):
                        Y, X = wy * w + iy - pt, wx * w + ix - pl
                        idx.append(base + Y * W + X if (0 <= Y < H and 0 <= X < W) else Lt)
                        coords.append((X, Y))
        base += H * W
    idx, coords = np.array(idx), np.array(coords)
    g = seq[idx].reshape(-1, 3, heads, d)
    q = oracle.rope_2d(g[:, 0], coords[:, 0, None], coords[:, 1, None])
    k = oracle.rope_2d(g[:, 1], coords[:, 0, None], coords[:, 1, None])
    v = g[:, 2]
    blk = np.arange(len(idx)) // (w * w)
    mask = torch.from_numpy(blk[:, None] == blk[None, :])
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(1, 0, 2)))
    o = F.scaled_dot_product_attention(tt(q), tt(k), tt(v), attn_mask=mask).numpy().transpose(1, 0, 2)
    O = np.zeros((Lt, heads, d))
    real = idx < Lt
    O[idx[real]] = o[real]
    return xp + O.reshape(Lt, C) @ wt["w_o"].T + wt["b_o"]


def test_ms_attention_equals_block_diagonal_index_operator():
    for sx, sy, scales in [(0, 0, [(16, 16), (8, 8)]), (4, 4, [(16, 16), (8, 8), (12, 4)]), (1, 3, [(10, 6), (5, 3)])]:
        cfg = synth.tiny(shift_x=sx, shift_y=sy, dtype="f32")
        wt = synth.make_weights(cfg)
        xp, _ = _packed(cfg, scales, 1)
        got = oracle.ms_attention_sublayer(xp, wt, cfg, scales)
        ref = _index_operator_ms(xp, wt, cfg, scales)
        assert np.max(np.abs(got - ref)) < 1e-12


def _scan_cfg():
    return synth.tiny(C=16, heads=2, ssm_state=4, ssm_dt_rank=2, ssm_expand=2, dtype="f32")


def test_ms_cycle_scan_single_scale_modes_agree():
    # with one scale, "split by scale" and "across all scales" are the same sequence
    cfg = _scan_cfg().replace(H=4, W=6)
    wt = synth.make_weights(cfg)
    xp, grids = _packed(cfg, [(4, 6)], 2)
    a = oracle.ms_cycle_scan_module(xp, wt, cfg, [(4, 6)], oracle.CS_SINGLE_SCALE)
    b = oracle.ms_cycle_scan_module(xp, wt, cfg, [(4, 6)], oracle.CS_MULTI_SCALE)
    assert np.max(np.abs(a - b)) < 1e-13
    assert np.array_equal(a, oracle.cycle_scan_module(grids[0], wt, cfg.replace(B=2, H=4, W=6)).reshape(-1, cfg.C))


def test_ms_cycle_scan_multi_scale_equals_closed_form_over_concatenation():
    # MULTI-SCALE = the cycled SSM over the concatenated sequence; compared with the independent closed form
    # (per-copy conv prefix + one summed-state pass) on the concatenation
    cfg = _scan_cfg()
    scales = [(4, 4), (2, 3), (3, 1)]
    wt = synth.make_weights(cfg.replace(H=4, W=4))
    xp, grids = _packed(cfg, scales, 2)
    got = oracle.ms_cycle_scan_module(xp, wt, cfg, scales, oracle.CS_MULTI_SCALE)
    off = oracle.ms_offsets(scales)
    D = cfg.D
    for b in range(2):
        seq = np.concatenate([g[b].reshape(-1, cfg.C) for g in grids])
        u0 = oracle.layer_norm(seq, wt["lns_g"], wt["lns_b"], cfg.ln_eps)
        xz = u0 @ wt["w_in"].T
        y = _closed_form_cycle(xz[:, :D], xz[:, D:], wt) @ wt["w_out"].T
        ref = seq + y
        mine = np.concatenate([got[2 * off[i]:2 * off[i + 1]].reshape(2, -1, cfg.C)[b] for i in range(len(scales))])
        assert np.max(np.abs(mine - ref)) < 1e-12


def test_ms_cycle_scan_mode_defines_cross_scale_influence():
    # the single-scale module scans each scale separately (scale 0's output cannot depend on scale 1's
    # tokens); the multi-scale module fuses the scales (it must)
    cfg = _scan_cfg()
    scales = [(4, 4), (2, 2)]
    wt = synth.make_weights(cfg.replace(H=4, W=4))
    xp, _ = _packed(cfg, scales, 1)
    xq = xp.copy()
    xq[16:] += np.random.default_rng(1).standard_normal(xq[16:].shape)  # (a constant shift would vanish in LN)
    for mode, same in [(oracle.CS_SINGLE_SCALE, True), (oracle.CS_MULTI_SCALE, False)]:
        a = oracle.ms_cycle_scan_module(xp, wt, cfg, scales, mode)[:16]
        b = oracle.ms_cycle_scan_module(xq, wt, cfg, scales, mode)[:16]
        assert np.array_equal(a, b) == same
