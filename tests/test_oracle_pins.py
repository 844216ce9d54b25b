"""Pins for the fp64 oracle against things other than itself (CPU only, `-m "not gpu"`).

Each test names what pins it: a worked example printed in the paper/SPEC (tests/golden), a closed form,
an invariant, a special case that reduces to a library routine (torch fp64 SDPA / layer_norm / linear,
numpy convolve), or brute force on tiny inputs. See DESIGN.md "Parity pins" (P1-P10).
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth
from conftest import read_golden

PAD = oracle.PAD


# ------------------------------------------------------------------------------------------
# synth generator sanity (determinism, storage rounding)
# ------------------------------------------------------------------------------------------

def test_synth_deterministic_and_bf16_exact():
    a = synth.normal(synth.stream_seed(3, 4), 1000)
    b = synth.normal(synth.stream_seed(3, 4), 1000)
    c = synth.normal(synth.stream_seed(3, 5), 1000)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert abs(a.mean()) < 0.15 and abs(a.std() - 1) < 0.1
    r = synth.round_bf16(a)
    assert np.array_equal(synth.round_bf16(r), r)                 # idempotent => representable
    assert np.array_equal(synth.bf16_bits_to_f64(synth.to_bf16_bits(r)), r)
    assert np.max(np.abs(r - a) / np.abs(a)) <= 2.0 ** -8


# ------------------------------------------------------------------------------------------
# P5: index maps — worked examples (golden), structural invariants, merge∘partition = id
# ------------------------------------------------------------------------------------------

def test_index_map_plain_worked_example():
    gold = np.array(read_golden("index_map_plain_4x4_w2.txt"), dtype=np.uint64).reshape(-1)
    m = oracle.index_map(4, 4, 2, 0, 0)
    assert np.array_equal(m.astype(np.uint64), gold)
    assert m.reshape(4, 4)[1, 1] == 3  # token (0,3) -> window 1, slot 1


def test_index_map_shift_worked_example():
    gold = np.array(read_golden("index_map_shift_4x4_w2_s1.txt"), dtype=np.uint64).reshape(-1)
    m = oracle.index_map(4, 4, 2, 1, 1)
    assert oracle.shifted_geometry(4, 4, 2, 1, 1) == (1, 1, 1, 1)
    assert oracle.window_count(4, 4, 2, 1, 1) == 9
    assert np.array_equal(m.astype(np.uint64), gold)


@pytest.mark.parametrize("H,W,w,s,nplain,nshift", [
    (64, 64, 16, 8, 16, 25), (128, 128, 16, 8, 64, 81), (256, 256, 16, 8, 256, 289), (16, 16, 8, 4, 4, 9)])
def test_window_counts_configs(H, W, w, s, nplain, nshift):
    # padded grids 80/144/272 (25/81/289 windows), tiny 24 (9 windows)
    assert oracle.window_count(H, W, w) == nplain
    assert oracle.window_count(H, W, w, s, s) == nshift


@pytest.mark.parametrize("H,W,w,sx,sy", [(16, 16, 8, 4, 4), (12, 20, 4, 1, 3), (7, 9, 4, 2, 1), (8, 8, 4, 0, 0)])
def test_index_map_is_partition(H, W, w, sx, sy):
    m = oracle.index_map(H, W, w, sx, sy)
    real = m[m != PAD].astype(np.int64)
    assert np.array_equal(np.sort(real), np.arange(H * W))          # every token exactly once
    pt, pl, pb, pr = oracle.shifted_geometry(H, W, w, sx, sy)
    assert (m == PAD).sum() == (pt + H + pb) * (pl + W + pr) - H * W
    assert max(pt, pl, pb, pr) < w
    # brute-force window membership: token (y,x) sits in padded window ((y+pt)//w, (x+pl)//w)
    nwx = (pl + W + pr) // w
    for slot, src in enumerate(m):
        if src == PAD:
            continue
        y, x = divmod(int(src), W)
        win, s = divmod(slot, w * w)
        assert win == ((y + pt) // w) * nwx + (x + pl) // w
        assert s == ((y + pt) % w) * w + (x + pl) % w


def test_partition_merge_roundtrip_bit_exact():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 12, 20, 5))
    pad = rng.standard_normal(5)
    for (w, sx, sy) in [(4, 0, 0), (4, 1, 3), (4, 2, 2)]:
        p = oracle.shifted_pad_partition(x, pad, w, sx, sy)
        m = oracle.index_map(12, 20, w, sx, sy)
        assert np.array_equal(p.reshape(2, -1, 5)[:, m == PAD], np.broadcast_to(pad, (2, int((m == PAD).sum()), 5)))
        back = oracle.window_merge(p, 2, 12, 20, w, sx, sy)
        assert np.array_equal(back, x)
        res = rng.standard_normal(x.shape)
        assert np.array_equal(oracle.window_merge(p, 2, 12, 20, w, sx, sy, res), x + res)
    with pytest.raises(ValueError):
        oracle.shifted_pad_partition(x, None, 4, 1, 1)
    with pytest.raises(ValueError):
        oracle.index_map(10, 12, 4, 0, 0)


# ------------------------------------------------------------------------------------------
# P6: App. A softmax / flash recurrences vs the plain definition and torch SDPA
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("x", [[0.0, 0.0], list(range(1, 9)), [1e4, -1e4, 3.0], [1000.0] * 3])
def test_online_softmax_forms(x):
    x = np.array(x, dtype=np.float64)
    ref = np.exp(x - x.max()) / np.exp(x - x.max()).sum()
    for f in (oracle.stable_softmax, oracle.online_softmax_3pass, oracle.online_softmax_2pass):
        y = f(x)
        assert np.all(np.isfinite(y)) and abs(y.sum() - 1) < 1e-12
        assert np.max(np.abs(y - ref)) < 1e-14
    assert np.max(np.abs(oracle.stable_softmax(x + 777.0) - oracle.stable_softmax(x))) < 1e-12


@pytest.mark.parametrize("L", [1, 7, 64, 257])
@pytest.mark.parametrize("b", [1, 7, 64])
def test_flash_tiled_equals_naive_and_sdpa(L, b):
    rng = np.random.default_rng(L * 100 + b)
    q, k, v = (rng.uniform(-1, 1, (2, L, 16)) for _ in range(3))
    scale = 1 / math.sqrt(16)
    naive = oracle.attention_naive(q, k, v, scale)
    flash = oracle.flash_attention_tiled(q, k, v, scale, b)
    sdpa = F.scaled_dot_product_attention(*(torch.from_numpy(t) for t in (q, k, v))).numpy()
    assert np.max(np.abs(flash - naive)) < 1e-12
    assert np.max(np.abs(naive - sdpa)) < 1e-12
    if L == 1:
        assert np.array_equal(naive, v)  # single key -> V row exactly


# ------------------------------------------------------------------------------------------
# P9: RoPE invariants
# ------------------------------------------------------------------------------------------

def test_rope_invariants():
    rng = np.random.default_rng(1)
    d = 64
    t = rng.standard_normal((10, d))
    assert np.array_equal(oracle.rope_2d(t, np.zeros(10), np.zeros(10)), t)       # zero rotation
    X, Y = rng.integers(-40, 300, 10), rng.integers(-40, 300, 10)
    r = oracle.rope_2d(t, X, Y)
    pairs = lambda a: (a[:, 0::2] ** 2 + a[:, 1::2] ** 2)
    assert np.max(np.abs(pairs(r) - pairs(t))) < 1e-12                             # plane norms kept
    q, k = rng.standard_normal(d), rng.standard_normal(d)
    for _ in range(5):
        (x1, y1, x2, y2, tx, ty) = rng.integers(-50, 300, 6)
        a = oracle.rope_2d(q, x1, y1) @ oracle.rope_2d(k, x2, y2)
        b = oracle.rope_2d(q, x1 + tx, y1 + ty) @ oracle.rope_2d(k, x2 + tx, y2 + ty)
        assert abs(a - b) < 1e-10                                                   # relative positions only
    # first half depends on X only, second half on Y only
    r2 = oracle.rope_2d(t, X, Y + 7)
    assert np.array_equal(r2[:, : d // 2], r[:, : d // 2]) and not np.allclose(r2[:, d // 2:], r[:, d // 2:])


# ------------------------------------------------------------------------------------------
# LayerNorm vs torch
# ------------------------------------------------------------------------------------------

def test_layer_norm_vs_torch():
    rng = np.random.default_rng(2)
    x, g, b = rng.standard_normal((5, 33)), rng.standard_normal(33), rng.standard_normal(33)
    ref = F.layer_norm(torch.from_numpy(x), (33,), torch.from_numpy(g), torch.from_numpy(b), 1e-6).numpy()
    assert np.max(np.abs(oracle.layer_norm(x, g, b, 1e-6) - ref)) < 1e-12


# ------------------------------------------------------------------------------------------
# P1 / P2: attention sub-layer special cases
# ------------------------------------------------------------------------------------------

def _torch_sublayer_global(x, wt, cfg, rope):
    """Independent route: torch fp64 layer_norm / linear / SDPA over the WHOLE grid (global attention)."""
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    B, H, W, C = x.shape
    heads, d = cfg.heads, C // cfg.heads
    u = F.layer_norm(T(x), (C,), T(wt["ln1_g"]), T(wt["ln1_b"]), cfg.ln_eps)
    qkv = F.linear(u, T(wt["w_qkv"]), T(wt["b_qkv"])).reshape(B, H * W, 3, heads, d)
    q, k, v = (qkv[:, :, i].permute(0, 2, 1, 3) for i in range(3))  # [B, heads, L, d]
    if rope:
        yy, xx = np.divmod(np.arange(H * W), W)
        q = T(oracle.rope_2d(q.numpy(), xx, yy))
        k = T(oracle.rope_2d(k.numpy(), xx, yy))
    o = F.scaled_dot_product_attention(q, k, v).permute(0, 2, 1, 3).reshape(B, H, W, C)
    return (T(x) + F.linear(o, T(wt["w_o"]), T(wt["b_o"]))).numpy()


@pytest.mark.parametrize("rope", [0, 1])
def test_P1_window_equals_grid_is_global_attention(rope):
    cfg = synth.tiny(window=16, shift_x=0, shift_y=0, rope=rope, dtype="f32")
    x, wt = synth.make_input(cfg), synth.make_weights(cfg)
    got = oracle.attention_sublayer(x, wt, cfg)
    ref = _torch_sublayer_global(x, wt, cfg, rope)
    assert np.max(np.abs(got - ref)) < 1e-12


def test_P1_window_equals_grid_multiwindow_grid():
    # 2x2 windows of 8 on a 16x16 grid = 4 independent global attentions on 8x8 sub-grids (rope off)
    cfg = synth.tiny(shift_x=0, shift_y=0, rope=0, dtype="f32")
    x, wt = synth.make_input(cfg), synth.make_weights(cfg)
    got = oracle.attention_sublayer(x, wt, cfg)
    for wy in range(2):
        for wx in range(2):
            sub = x[:, wy * 8:(wy + 1) * 8, wx * 8:(wx + 1) * 8]
            ref = _torch_sublayer_global(sub, wt, cfg.replace(H=8, W=8), 0)
            assert np.max(np.abs(got[:, wy * 8:(wy + 1) * 8, wx * 8:(wx + 1) * 8] - ref)) < 1e-12


def test_P2_shift_zero_is_plain():
    cfg = synth.tiny(shift_x=0, shift_y=0)
    x, wt = synth.make_input(cfg), synth.make_weights(cfg)
    a = oracle.attention_sublayer(x, wt, cfg)
    for mode in (synth.PAD_LEARNABLE, synth.PAD_MASKED):
        b = oracle.attention_sublayer(x, {**wt, "pad": wt["pad"] * 3 + 1}, cfg.replace(pad_mode=mode))
        assert np.array_equal(a, b)
    assert np.array_equal(oracle.index_map(16, 16, 8, 0, 0), oracle.index_map(16, 16, 8, 0, 0))


# ------------------------------------------------------------------------------------------
# P3: MASKED mode — pads never influence real tokens; equals truncated-window brute force
# ------------------------------------------------------------------------------------------

def test_P3_masked_independent_of_pad_and_brute_force():
    cfg = synth.tiny(pad_mode=synth.PAD_MASKED, H=12, W=20, window=8, shift_x=3, shift_y=5)
    x, wt = synth.make_input(cfg), synth.make_weights(cfg)
    a = oracle.attention_sublayer(x, wt, cfg)
    b = oracle.attention_sublayer(x, {**wt, "pad": -5 * wt["pad"] + 2}, cfg)
    assert np.array_equal(a, b)
    # brute force: each real token attends to the real tokens of its own (differently sized) window
    B, H, W, C = x.shape
    heads, d, w = cfg.heads, C // cfg.heads, cfg.window
    pt, pl, _, _ = oracle.shifted_geometry(H, W, w, cfg.shift_x, cfg.shift_y)
    u = oracle.layer_norm(x, wt["ln1_g"], wt["ln1_b"], cfg.ln_eps)
    qkv = (u @ wt["w_qkv"].T + wt["b_qkv"]).reshape(B, H, W, 3, heads, d)
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    q = oracle.rope_2d(qkv[..., 0, :, :], xx[None, :, :, None], yy[None, :, :, None])
    k = oracle.rope_2d(qkv[..., 1, :, :], xx[None, :, :, None], yy[None, :, :, None])
    v = qkv[..., 2, :, :]
    win_id = ((yy + pt) // w) * 100 + (xx + pl) // w
    O = np.zeros((B, H, W, heads, d))
    for wid in np.unique(win_id):
        sel = win_id == wid
        qs, ks, vs = (torch.from_numpy(np.ascontiguousarray(t[:, sel].transpose(0, 2, 1, 3))) for t in (q, k, v))
        O[:, sel] = F.scaled_dot_product_attention(qs, ks, vs).numpy().transpose(0, 2, 1, 3)
    ref = x + O.reshape(B, H, W, C) @ wt["w_o"].T + wt["b_o"]
    assert np.max(np.abs(a - ref)) < 1e-12


# ------------------------------------------------------------------------------------------
# P4: LEARNABLE mode (the paper's Pad Swin)
# ------------------------------------------------------------------------------------------

def test_P4_windows_without_pads_ignore_p():
    cfg = synth.tiny(H=24, W=24, window=8, shift_x=4, shift_y=4)
    x, wt = synth.make_input(cfg), synth.make_weights(cfg)
    a = oracle.attention_sublayer(x, wt, cfg)
    b = oracle.attention_sublayer(x, {**wt, "pad": wt["pad"] + 1.0}, cfg)
    # padded grid 32x32 (pt=pl=4): windows 1..2 in each axis hold only real tokens: rows/cols 4..19
    inner = (slice(None), slice(4, 20), slice(4, 20))
    assert np.array_equal(a[inner], b[inner])
    assert not np.allclose(a[:, :4], b[:, :4])  # border windows do see p


def test_P4_all_tokens_equal_p_closed_form():
    # If every real token projects exactly like p (LN(x_t) = p) and RoPE is off, every key/value in every
    # padded window is identical, so softmax is uniform and O = v_p for every token:
    # x_out = x + (p W_v^T + b_v) W_o^T + b_o. (Fails if pad slots carried zeros or were skipped.)
    cfg = synth.tiny(rope=0, dtype="f32")
    wt = synth.make_weights(cfg)
    wt = {**wt, "ln1_g": np.ones(cfg.C), "ln1_b": np.zeros(cfg.C)}
    rng = np.random.default_rng(5)
    base = rng.standard_normal(cfg.C)
    base = (base - base.mean()) / base.std()
    p = oracle.layer_norm(base, wt["ln1_g"], wt["ln1_b"], cfg.ln_eps)
    wt["pad"] = p
    x = np.broadcast_to(base, (1, 16, 16, cfg.C)).copy()
    C = cfg.C
    v_p = p @ wt["w_qkv"][2 * C:].T + wt["b_qkv"][2 * C:]
    ref = x + (v_p @ wt["w_o"].T + wt["b_o"])
    assert np.max(np.abs(oracle.attention_sublayer(x, wt, cfg) - ref)) < 1e-12


def test_P4_index_operator_route_equals_materialised_grid():
    """App. C: append p's projection at the END of the token sequence, gather with an index map
    (pad slots point at the appended row), then ONE block-diagonal attention over the packed sequence
    (App. B) — computed with torch SDPA + a block mask — must equal the oracle's materialised
    padded grid."""
    cfg = synth.tiny(H=12, W=20, window=4, shift_x=1, shift_y=3, dtype="f32")
    x, wt = synth.make_input(cfg), synth.make_weights(cfg)
    B, H, W, C = x.shape
    heads, d, w = cfg.heads, C // cfg.heads, cfg.window
    u = oracle.layer_norm(x, wt["ln1_g"], wt["ln1_b"], cfg.ln_eps)
    seq = np.concatenate([(u @ wt["w_qkv"].T + wt["b_qkv"]).reshape(B, H * W, 3 * C),
                          np.broadcast_to(wt["pad"] @ wt["w_qkv"].T + wt["b_qkv"], (B, 1, 3 * C))], axis=1)
    # independent enumeration of the padded layout: pad left/top = w - s, complete windows
    pl, pt = w - cfg.shift_x, w - cfg.shift_y
    Wp, Hp = -(-(pl + W) // w) * w, -(-(pt + H) // w) * w
    idx, coords = [], []
    for wy in range(Hp // w):
        for wx in range(Wp // w):
            for iy in range(w):
                for ix in range(w):
                    Y, X = wy * w + iy - pt, wx * w + ix - pl
                    idx.append(Y * W + X if (0 <= Y < H and 0 <= X < W) else H * W)
                    coords.append((X, Y))
    idx = np.array(idx)
    coords = np.array(coords)
    g = seq[:, idx].reshape(B, -1, 3, heads, d)
    q = oracle.rope_2d(g[:, :, 0], coords[None, :, 0, None], coords[None, :, 1, None])
    k = oracle.rope_2d(g[:, :, 1], coords[None, :, 0, None], coords[None, :, 1, None])
    v = g[:, :, 2]
    n = len(idx)
    blk = np.arange(n) // (w * w)
    mask = torch.from_numpy(blk[:, None] == blk[None, :])
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 1, 3)))
    o = F.scaled_dot_product_attention(tt(q), tt(k), tt(v), attn_mask=mask).numpy().transpose(0, 2, 1, 3)
    O = np.zeros((B, H * W, heads, d))
    real = idx < H * W
    O[:, idx[real]] = o[:, real]
    ref = x + O.reshape(B, H, W, C) @ wt["w_o"].T + wt["b_o"]
    assert np.max(np.abs(oracle.attention_sublayer(x, wt, cfg) - ref)) < 1e-12


# ------------------------------------------------------------------------------------------
# SSM pins: Eq. 3 worked value, Eq. 4 == Eq. 5 (LTI), conv, memoryless / L=1 closed forms
# ------------------------------------------------------------------------------------------

def test_zoh_worked_value():
    for a, delta, Bv, Abar, Bbar in read_golden("zoh_closed_form.txt"):
        Ab, Bb = oracle.zoh_discretize(np.array([[delta]]), np.array([[a]]), np.array([[Bv]]))
        assert abs(Ab[0, 0] - Abar) < 1e-15 and abs(Bb[0, 0] - Bbar) < 1e-15


@pytest.mark.parametrize("L", [1, 17, 256])
def test_scan_equals_convolution_lti(L):
    # Eq. 4 (recurrence) == Eq. 5 (global convolution) when Delta, B, C are input independent
    rng = np.random.default_rng(L)
    D, N = 8, 32
    A = -np.exp(rng.uniform(-1, 2, (D, N)))
    delta = np.exp(rng.uniform(-5, -1, D))
    Bv, Cv = rng.standard_normal(N), rng.standard_normal(N)
    v = rng.standard_normal((L, D))
    y = oracle.selective_scan_sequential(v, np.tile(delta, (L, 1)), A, np.tile(Bv, (L, 1)),
                                         np.tile(Cv, (L, 1)), np.zeros(D))
    Ab, Bb = oracle.zoh_discretize(delta[:, None], A, Bv[None, :])
    K = oracle.ssm_conv_kernel(Ab, Bb, Cv, L)
    conv = np.stack([np.convolve(v[:, c], K[:, c])[:L] for c in range(D)], axis=1)
    assert np.max(np.abs(y - conv)) < 1e-10 * max(1.0, np.abs(conv).max())


def test_causal_conv_vs_numpy():
    rng = np.random.default_rng(3)
    xs, w, b = rng.standard_normal((11, 5)), rng.standard_normal((5, 4)), rng.standard_normal(5)
    c = oracle.causal_conv1d(xs, w, b)
    for ch in range(5):
        ref = np.convolve(xs[:, ch], w[ch, ::-1])[:11] + b[ch]
        assert np.max(np.abs(c[:, ch] - ref)) < 1e-13


def _scan_weights(D=6, N=4, R=2, k=4, seed=0):
    rng = np.random.default_rng(seed)
    return dict(conv_w=rng.uniform(-.5, .5, (D, k)), conv_b=rng.uniform(-.5, .5, D),
                w_x=rng.standard_normal((R + 2 * N, D)) * 0.5, w_dt=rng.uniform(-.7, .7, (D, R)),
                b_dt=rng.uniform(-4, -1, D), a_log=np.log(np.tile(np.arange(1, N + 1.0), (D, 1))),
                d_skip=rng.uniform(0.5, 1.5, D))


def test_cycle_scan_memoryless_limit():
    # A -> -inf: A_bar = 0, B_bar = -B/A ~ 0 => y_j = D v_j; 3 copies sum to (v^1 + 2 v^2) D where v^1
    # differs from v^2 only on the first k-1 tokens (zero conv history, reading Q10).
    wt = _scan_weights()
    wt["a_log"] = np.full_like(wt["a_log"], 40.0)
    rng = np.random.default_rng(1)
    L, D = 9, 6
    xin, z = rng.standard_normal((1, L, D)), rng.standard_normal((1, L, D))
    g = oracle.cycle_scan(xin, z, wt, 3, 3)
    s = xin[0]
    v1 = oracle.silu(oracle.causal_conv1d(s, wt["conv_w"], wt["conv_b"]))
    ext = np.concatenate([s[-3:], s])
    v2 = oracle.silu(oracle.causal_conv1d(ext, wt["conv_w"], wt["conv_b"]))[3:]
    ref = (v1 + 2 * v2) * wt["d_skip"] * oracle.silu(z[0])
    assert np.max(np.abs(g[0] - ref)) < 1e-12


def test_cycle_scan_single_token():
    # L = 1: the cycled sequence is [x, x, x]; conv windows see [0,0,0,x], [0,0,x,x], [0,x,x,x].
    wt = _scan_weights(D=3, N=2, R=1)
    rng = np.random.default_rng(2)
    xin, z = rng.standard_normal((1, 1, 3)), rng.standard_normal((1, 1, 3))
    g = oracle.cycle_scan(xin, z, wt, 1, 1)
    x = xin[0, 0]
    A = -np.exp(wt["a_log"])
    h = np.zeros((3, 2))
    tot = np.zeros(3)
    for j in range(3):
        c = wt["conv_b"] + x * wt["conv_w"][:, 3 - j:].sum(axis=1)
        v = c / (1 + np.exp(-c))
        dbc = v @ wt["w_x"].T
        dt = np.log1p(np.exp(dbc[:1] @ wt["w_dt"].T + wt["b_dt"]))
        Ab = np.exp(dt[:, None] * A)
        h = Ab * h + (Ab - 1) / A * dbc[None, 1:3] * v[:, None]
        tot += h @ dbc[3:5] + wt["d_skip"] * v
    assert np.max(np.abs(g[0, 0] - tot * z[0, 0] / (1 + np.exp(-z[0, 0])))) < 1e-12


def _closed_form_cycle(xin_seq, z_seq, wt, k=4):
    """Independent route (SURVEY Appendix A / DESIGN.md "Cycle-scan closed form"): per-copy prefix of
    k-1 tokens, then ONE pass of the summed state H_t = A_t H_{t-1} + 3 B_t v_t, y = C.H + 3 D v."""
    L, D = xin_seq.shape
    P = k - 1
    R = wt["w_dt"].shape[1]
    N = wt["a_log"].shape[1]
    A = -np.exp(wt["a_log"])

    def params(v):
        dbc = v @ wt["w_x"].T
        dt = np.logaddexp(0, dbc[:, :R] @ wt["w_dt"].T + wt["b_dt"])
        Ab = np.exp(dt[:, :, None] * A)
        Bv = np.expm1(dt[:, :, None] * A) / A * dbc[:, None, R:R + N] * v[:, :, None]
        return Ab, Bv, dbc[:, R + N:]

    v1 = oracle.silu(oracle.causal_conv1d(xin_seq, wt["conv_w"], wt["conv_b"]))
    v2 = oracle.silu(oracle.causal_conv1d(np.concatenate([xin_seq[L - P:], xin_seq]), wt["conv_w"], wt["conv_b"]))[P:]
    A1, B1, C1 = params(v1)
    A2, B2, C2 = params(v2)
    Abody, Bbody = np.ones((D, N)), np.zeros((D, N))
    for t in range(P, L):
        Abody, Bbody = A2[t] * Abody, A2[t] * Bbody + B2[t]

    def prefix(Aa, Bb, c):
        hs = []
        for t in range(P):
            c = Aa[t] * c + Bb[t]
            hs.append(c)
        return c, hs

    e1, h1 = prefix(A1, B1, np.zeros((D, N)))
    c2 = Abody * e1 + Bbody
    e2, h2 = prefix(A2, B2, c2)
    c3 = Abody * e2 + Bbody
    e3, h3 = prefix(A2, B2, c3)
    y = np.empty((L, D))
    for t in range(P):
        y[t] = ((h1[t] * C1[t]).sum(-1) + (h2[t] * C2[t]).sum(-1) + (h3[t] * C2[t]).sum(-1)
                + wt["d_skip"] * (v1[t] + 2 * v2[t]))
    H = e1 + e2 + e3
    for t in range(P, L):
        H = A2[t] * H + 3 * B2[t]
        y[t] = (H * C2[t]).sum(-1) + 3 * wt["d_skip"] * v2[t]
    return y * oracle.silu(z_seq)


@pytest.mark.parametrize("L,seed", [(7, 0), (16, 1), (40, 2), (3, 3)])
def test_cycle_scan_literal_equals_closed_form(L, seed):
    wt = _scan_weights(seed=seed)
    rng = np.random.default_rng(seed + 10)
    xin, z = rng.standard_normal((1, L, 6)), rng.standard_normal((1, L, 6))
    g = oracle.cycle_scan(xin, z, wt, 1, L)
    ref = _closed_form_cycle(xin[0], z[0], wt)
    assert np.max(np.abs(g[0] - ref)) < 1e-12 * max(1.0, np.abs(ref).max())


def test_cycle_scan_channel_permutation_equivariance():
    # channels are independent: permuting the D channels of xin, z and every per-channel
    # parameter permutes the output (shared B, C projections permute their input columns).
    wt = _scan_weights(seed=4)
    rng = np.random.default_rng(4)
    xin, z = rng.standard_normal((1, 10, 6)), rng.standard_normal((1, 10, 6))
    perm = rng.permutation(6)
    wp = dict(wt, conv_w=wt["conv_w"][perm], conv_b=wt["conv_b"][perm], w_x=wt["w_x"][:, perm],
              w_dt=wt["w_dt"][perm], b_dt=wt["b_dt"][perm], a_log=wt["a_log"][perm], d_skip=wt["d_skip"][perm])
    a = oracle.cycle_scan(xin, z, wt, 2, 5)
    b = oracle.cycle_scan(xin[..., perm], z[..., perm], wp, 2, 5)
    assert np.max(np.abs(a[..., perm] - b)) < 1e-13


def test_euler_close_to_zoh_for_small_delta():
    rng = np.random.default_rng(6)
    A = -np.exp(rng.uniform(0, 1, (4, 3)))
    d = np.full((4, 1), 1e-6)
    Bm = rng.standard_normal((1, 3))
    _, bz = oracle.zoh_discretize(d, A, Bm, oracle.BBAR_ZOH)
    _, be = oracle.zoh_discretize(d, A, Bm, oracle.BBAR_EULER)
    assert np.max(np.abs(bz - be)) < 1e-11


def test_module_equals_abi_scan_composition():
    # cycle_scan_module applies W_in to all 3L tokens (literal); by linearity it must equal
    # x + (ABI cycle_scan of in_proj(LN(x)) computed once on L tokens) W_out^T.
    cfg = synth.tiny(cycle_scan=1, H=8, W=6, dtype="f32")
    x, wt = synth.make_input(cfg), synth.make_weights(cfg)
    out = oracle.cycle_scan_module(x, wt, cfg)
    u0 = oracle.layer_norm(x, wt["lns_g"], wt["lns_b"], cfg.ln_eps).reshape(1, 48, cfg.C)
    xz = u0 @ wt["w_in"].T
    g = oracle.cycle_scan(xz[..., :cfg.D], xz[..., cfg.D:], wt, 8, 6)
    ref = x + (g @ wt["w_out"].T).reshape(x.shape)
    assert np.max(np.abs(out - ref)) < 1e-12


@pytest.mark.parametrize("order", [synth.SCAN_COL_MAJOR, synth.SCAN_WINDOW_MAJOR])
def test_scan_orders_are_permutations(order):
    pi = oracle.scan_permutation(8, 12, order, 4)
    assert np.array_equal(np.sort(pi), np.arange(96))
    if order == synth.SCAN_COL_MAJOR:
        assert list(pi[:3]) == [0, 12, 24]
    else:
        assert list(pi[:6]) == [0, 1, 2, 3, 12, 13]


# ------------------------------------------------------------------------------------------
# FFN sub-layer (NEXT-2): library routines and GELU closed forms
# ------------------------------------------------------------------------------------------

def test_gelu_closed_forms():
    x = np.array([0.0, 1.0, -1.0, 3.0, -7.5, 40.0])
    g = oracle.gelu(x)
    assert g[0] == 0.0 and abs(g[-1] - 40.0) < 1e-12           # GELU(0) = 0, GELU(x) -> x
    assert np.max(np.abs(g - oracle.gelu(-x) - x)) < 1e-15     # x Phi(x) - (-x) Phi(-x) = x
    assert abs(g[1] - 0.8413447460685429) < 1e-15              # Phi(1) (normal table)
    ref = F.gelu(torch.from_numpy(x)).numpy()                   # exact (erf) GELU of the library
    assert np.max(np.abs(g - ref)) < 1e-14


def test_ffn_sublayer_vs_torch():
    cfg = synth.tiny(mlp_hidden=256, dtype="f32")
    x, wt = synth.make_input(cfg), synth.make_weights(cfg)
    t = {k: torch.from_numpy(v) for k, v in wt.items()}
    xt = torch.from_numpy(x)
    u = F.layer_norm(xt, (cfg.C,), t["ln2_g"], t["ln2_b"], cfg.ln_eps)
    ref = xt + F.linear(F.gelu(F.linear(u, t["w_fc1"], t["b_fc1"])), t["w_fc2"], t["b_fc2"])
    assert np.max(np.abs(oracle.ffn_sublayer(x, wt, cfg) - ref.numpy())) < 1e-12
    # the layer applies it after attention
    assert np.array_equal(oracle.pscwin_layer(x, wt, cfg),
                          oracle.ffn_sublayer(oracle.attention_sublayer(x, wt, cfg), wt, cfg))


def test_global_attention_rows_vs_sdpa():
    # the Table 3 "Global" comparator: sampled query rows of Eq. 1 over ALL keys equal torch fp64 SDPA
    # on the RoPE'd sequence (library routine), and the window = grid case of the window oracle
    cfg = synth.tiny(H=12, W=8, window=4, shift_x=0, shift_y=0, dtype="f32")
    qkv = synth.make_qkv(cfg)
    H, W, heads, C = 12, 8, cfg.heads, cfg.C
    d = C // heads
    toks = [0, 17, 95]
    got = oracle.global_attention_rows(qkv, H, W, heads, toks, 1)
    g = qkv[0].reshape(H * W, 3, heads, d)
    Y, X = np.divmod(np.arange(H * W), W)
    q = oracle.rope_2d(g[:, 0], X[:, None].astype(float), Y[:, None].astype(float))
    k = oracle.rope_2d(g[:, 1], X[:, None].astype(float), Y[:, None].astype(float))
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(1, 0, 2)))
    ref = F.scaled_dot_product_attention(tt(q), tt(k), tt(g[:, 2])).numpy().transpose(1, 0, 2).reshape(H * W, C)
    assert np.max(np.abs(got - ref[toks])) < 1e-12
