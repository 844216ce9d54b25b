"""PSCWin oracle: a plain, slow, fp64 CPU implementation of HRSAM's PSCWin layer.

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and bench.py's
`cpu_baseline` / `--impl reference` legs may import this module. The product path
(`paper_2407_02109_b200/`) never imports it and shares no code with it.

Citations: P:Lx = /root/reference/PAPER.md line x (section / equation given alongside);
Qn = the reading of a paper silence listed in DESIGN.md ("Readings").

Everything is computed in float64 with no intermediate rounding (Q16). The oracle is the
plain definition of what the layer computes: it MATERIALISES what the GPU avoids — the
padded grid filled with copies of the projected pad token, the full w^2 x w^2
softmax per window, and the literal 3L cycled sequence with a strictly
sequential recurrence (Eq. 4).
"""
from __future__ import annotations

import math
from typing import Dict, Optional, Tuple

import numpy as np

PAD = 0xFFFFFFFF  # index-map sentinel = max index value

PAD_LEARNABLE = 0
PAD_MASKED = 1
SCAN_ROW_MAJOR = 0
SCAN_COL_MAJOR = 1
SCAN_WINDOW_MAJOR = 2
BBAR_ZOH = 0
BBAR_EULER = 1


# =============================================================================================
# §3.2 window geometry: plain windows and padding shifted windows
# =============================================================================================

def shifted_geometry(H: int, W: int, w: int, sx: int, sy: int) -> Tuple[int, int, int, int]:
    """Padding of the padding-shifted window: "padding of w - S_x units on the left
    ... and w - S_y units on the top"; "additional padding ... to the opposite sides as necessary
    to ensure a complete number of windows". Reading Q7: pad = (w - s) mod w so shift 0 = plain.
    Returns (pad_top, pad_left, pad_bottom, pad_right)."""
    if not (0 <= sx < w and 0 <= sy < w):
        raise ValueError("shift must lie in [0, window)")
    pl = (w - sx) % w
    pt = (w - sy) % w
    pr = (-(pl + W)) % w
    pb = (-(pt + H)) % w
    return pt, pl, pb, pr


def window_count(H: int, W: int, w: int, sx: int = 0, sy: int = 0) -> int:
    if sx == 0 and sy == 0 and (H % w or W % w):
        raise ValueError("plain windows need H, W divisible by the window (P:L598)")
    pt, pl, pb, pr = shifted_geometry(H, W, w, sx, sy)
    return ((pt + H + pb) // w) * ((pl + W + pr) // w)


def index_map(H: int, W: int, w: int, sx: int = 0, sy: int = 0) -> np.ndarray:
    """Destination slot -> source token (row-major y*W+x) or PAD (App. C).
    Windows row-major over (wy, wx), slots row-major over (iy, ix) (reading Q4)."""
    n = window_count(H, W, w, sx, sy)
    pt, pl, pb, pr = shifted_geometry(H, W, w, sx, sy)
    nwx = (pl + W + pr) // w
    out = np.empty(n * w * w, dtype=np.uint64)
    k = 0
    for win in range(n):
        wy, wx = divmod(win, nwx)
        for iy in range(w):
            for ix in range(w):
                y = wy * w + iy - pt
                x = wx * w + ix - pl
                out[k] = y * W + x if (0 <= y < H and 0 <= x < W) else PAD
                k += 1
    return out.astype(np.uint32)


def window_partition(x: np.ndarray, w: int) -> np.ndarray:
    """Plain window partition F -> F_w: [B,H,W,Cx] -> [B*nW, w*w, Cx]."""
    return shifted_pad_partition(x, None, w, 0, 0)


def shifted_pad_partition(x: np.ndarray, pad_row: Optional[np.ndarray], w: int, sx: int, sy: int) -> np.ndarray:
    """Gather by the index map; PAD slots take pad_row ("(Q,K,V) of p are replicated")."""
    B, H, W, Cx = x.shape
    m = index_map(H, W, w, sx, sy)
    flat = x.reshape(B, H * W, Cx)
    out = np.empty((B, m.size, Cx), dtype=x.dtype)
    real = m != PAD
    if (~real).any():
        if pad_row is None:
            raise ValueError("shifted partition with pad slots needs pad_row (SPEC S:L249)")
        out[:, ~real] = pad_row
    out[:, real] = flat[:, m[real].astype(np.int64)]
    return out.reshape(B * (m.size // (w * w)), w * w, Cx)


def window_merge(win: np.ndarray, B: int, H: int, W: int, w: int, sx: int, sy: int,
                 residual: Optional[np.ndarray] = None) -> np.ndarray:
    """Inverse of the partition: scatter real slots back to the grid, drop pads
    ("the paddings are discarded, retaining only the region corresponding to F");
    optionally add a residual [B,H,W,Cx]."""
    m = index_map(H, W, w, sx, sy)
    Cx = win.shape[-1]
    src = win.reshape(B, m.size, Cx)
    out = np.zeros((B, H * W, Cx), dtype=win.dtype)
    real = m != PAD
    out[:, m[real].astype(np.int64)] = src[:, real]
    out = out.reshape(B, H, W, Cx)
    if residual is not None:
        out = out + residual
    return out


# =============================================================================================
# LayerNorm (ViT pre-norm; eps 1e-6, reading Q15)
# =============================================================================================

def layer_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float) -> np.ndarray:
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


# =============================================================================================
# RoPE ("replaces SAM's relative encoding with RoPE"; concrete form = reading Q6)
# =============================================================================================

def rope_2d(t: np.ndarray, X: np.ndarray, Y: np.ndarray, base: float = 10000.0) -> np.ndarray:
    """Axial 2-D rotary embedding on the last axis (size d, d % 4 == 0).
    Channels [0, d/2) rotate by X * theta_j, [d/2, d) by Y * theta_j, theta_j = base^(-4j/d),
    j < d/4; rotation planes are the interleaved pairs (2j, 2j+1) inside each half.
    X, Y broadcast against t[..., 0]."""
    d = t.shape[-1]
    q = d // 4
    theta = base ** (-4.0 * np.arange(q) / d)
    out = t.copy()
    for half, pos in ((0, X), (1, Y)):
        ang = np.asarray(pos, dtype=np.float64)[..., None] * theta  # [..., q]
        c, s = np.cos(ang), np.sin(ang)
        i0 = half * (d // 2) + 2 * np.arange(q)
        a = t[..., i0]
        b = t[..., i0 + 1]
        out[..., i0] = a * c - b * s
        out[..., i0 + 1] = a * s + b * c
    return out


# =============================================================================================
# App. A: softmax forms and attention
# =============================================================================================

def stable_softmax(x: np.ndarray, axis: int = -1) -> np.ndarray:
    """softmax(x_i) = exp(x_i - max_k x_k) / sum_j exp(x_j - max_k x_k)."""
    m = np.max(x, axis=axis, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=axis, keepdims=True)


def online_softmax_3pass(x: np.ndarray) -> np.ndarray:
    """Three-pass online softmax, literal loops (small inputs only)."""
    n = len(x)
    m = -math.inf
    for i in range(n):
        m = max(m, x[i])
    d = 0.0
    for i in range(n):
        d = d + math.exp(x[i] - m)
    return np.array([math.exp(x[i] - m) / d for i in range(n)])


def online_softmax_2pass(x: np.ndarray) -> np.ndarray:
    """Two-pass online softmax with the d'_i recurrence."""
    n = len(x)
    m_prev, d = -math.inf, 0.0
    for i in range(n):
        m_i = max(m_prev, x[i])
        d = math.exp(m_prev - m_i) * d + math.exp(x[i] - m_i)
        m_prev = m_i
    return np.array([math.exp(x[i] - m_prev) / d for i in range(n)])


def attention_naive(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float,
                    key_valid: Optional[np.ndarray] = None) -> np.ndarray:
    """softmax(scale * q k^T) v over the last two axes (Eq. 1, with the pre-softmax
    1/sqrt(d) of reading Q1). key_valid (broadcast over [..., Lk]) masks keys to -inf."""
    logits = scale * np.einsum("...qd,...kd->...qk", q, k)
    if key_valid is not None:
        logits = np.where(key_valid[..., None, :], logits, -np.inf)
    return np.einsum("...qk,...kd->...qd", stable_softmax(logits, -1), v)


def flash_attention_tiled(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float, b: int) -> np.ndarray:
    """Tiled one-pass flash attention, App. A.5, all rows at once:
    m_i = max(m_{i-1}, m_i^local); d'_i = d'_{i-1} e^{m_{i-1}-m_i} + sum_j e^{x_i[j]-m_i};
    o'_i = o'_{i-1} (d'_{i-1}/d'_i) e^{m_{i-1}-m_i} + sum_j e^{x_i[j]-m_i}/d'_i V[j+(i-1)b]."""
    Lq, Lk = q.shape[-2], k.shape[-2]
    m = np.full(q.shape[:-1], -np.inf)
    dd = np.zeros(q.shape[:-1])
    o = np.zeros(q.shape[:-1] + (v.shape[-1],))
    for start in range(0, Lk, b):
        kt, vt = k[..., start:start + b, :], v[..., start:start + b, :]
        x = scale * np.einsum("...qd,...kd->...qk", q, kt)
        m_new = np.maximum(m, x.max(-1))
        corr = np.exp(m - m_new)
        p = np.exp(x - m_new[..., None])
        d_new = dd * corr + p.sum(-1)
        o = o * ((dd / d_new) * corr)[..., None] + np.einsum("...qk,...kd->...qd", p / d_new[..., None], vt)
        m, dd = m_new, d_new
    return o


# =============================================================================================
# Attention sub-layer: steps a4-a7; plain / padded-shift windows
# =============================================================================================

def attention_core_padded(qkv: np.ndarray, qkv_p: np.ndarray, H: int, W: int, heads: int, w: int,
                          sx: int, sy: int, pad_mode: int, rope: int, window_rows=None) -> np.ndarray:
    """Window attention over the materialised padded grid (a5 + a6 + crop of a7).

    qkv  [B,H,W,3C] projected tokens (Q = cols [0,C), K = [C,2C), V = [2C,3C); head-contiguous, Q3)
    qkv_p [3C]      projected learnable pad token p ("F and p are both projected")
    Builds the padded grid whose pad cells hold COPIES of qkv_p ("replicated"), applies RoPE at
    every cell's global coordinate (pad cells at their geometric coordinates, Q6), runs softmax attention
    inside every w x w window over all w^2 keys (LEARNABLE) or over real keys only (MASKED, Q5), and keeps
    only real cells ("the paddings are discarded"). Returns O [B,H,W,C].
    window_rows: optional subset of padded-grid window rows to evaluate (sampling at full size; the other
    cells are NaN). Each window depends only on its own cells, so a subset is exact for those windows."""
    B = qkv.shape[0]
    C3 = qkv.shape[-1]
    C = C3 // 3
    d = C // heads
    pt, pl, pb, pr = shifted_geometry(H, W, w, sx, sy)
    if sx == 0 and sy == 0 and (H % w or W % w):
        raise ValueError("plain windows need H, W divisible by the window")
    Hp, Wp = pt + H + pb, pl + W + pr
    grid = np.empty((B, Hp, Wp, C3))
    grid[:] = qkv_p
    grid[:, pt:pt + H, pl:pl + W] = qkv
    valid = np.zeros((Hp, Wp), dtype=bool)
    valid[pt:pt + H, pl:pl + W] = True
    Y = (np.arange(Hp) - pt)[:, None] * np.ones((1, Wp))
    X = np.ones((Hp, 1)) * (np.arange(Wp) - pl)[None, :]
    g = grid.reshape(B, Hp, Wp, 3, heads, d)
    q, k, v = g[:, :, :, 0], g[:, :, :, 1], g[:, :, :, 2]   # [B,Hp,Wp,heads,d]
    if rope:
        q = rope_2d(q, X[None, :, :, None], Y[None, :, :, None])
        k = rope_2d(k, X[None, :, :, None], Y[None, :, :, None])
    nwy, nwx = Hp // w, Wp // w
    out = np.full((B, Hp, Wp, heads, d), np.nan)
    scale = 1.0 / math.sqrt(d)
    for wy in (range(nwy) if window_rows is None else window_rows):  # one window row at a time bounds memory
        ys = slice(wy * w, (wy + 1) * w)

        def win(t):  # [B, w, Wp, heads, d] -> [B, nwx, heads, w*w, d]
            t = t[:, ys].reshape(B, w, nwx, w, heads, d)
            return t.transpose(0, 2, 4, 1, 3, 5).reshape(B, nwx, heads, w * w, d)

        kv_valid = valid[ys].reshape(w, nwx, w).transpose(1, 0, 2).reshape(nwx, 1, w * w)
        kmask = kv_valid[None] if pad_mode == PAD_MASKED else None
        o = attention_naive(win(q), win(k), win(v), scale, kmask)        # [B,nwx,heads,w*w,d]
        o = o.reshape(B, nwx, heads, w, w, d).transpose(0, 3, 1, 4, 2, 5).reshape(B, w, Wp, heads, d)
        out[:, ys] = o
    return out[:, pt:pt + H, pl:pl + W].reshape(B, H, W, C)


def global_attention_rows(qkv: np.ndarray, H: int, W: int, heads: int, tokens, rope: int = 1) -> np.ndarray:
    """Global attention (Eq. 1; the Table 3 "Global" comparator) evaluated for the given
    query tokens only (y*W + x of image 0): o_t = softmax(q_t K^T / sqrt(d)) V over ALL H*W keys, RoPE at grid
    coordinates (Q6). Equals window attention with window = H = W. qkv [B,H,W,3C] unrotated. Returns [n, C]."""
    C = qkv.shape[-1] // 3
    d = C // heads
    g = qkv[0].reshape(H * W, 3, heads, d)
    Y, X = np.divmod(np.arange(H * W), W)
    q, k, v = g[:, 0], g[:, 1], g[:, 2]
    if rope:
        q = rope_2d(q, X[:, None].astype(float), Y[:, None].astype(float))
        k = rope_2d(k, X[:, None].astype(float), Y[:, None].astype(float))
    tokens = np.asarray(tokens)
    out = np.empty((len(tokens), heads, d))
    for h in range(heads):
        logits = q[tokens, h] @ k[:, h].T / math.sqrt(d)
        out[:, h] = stable_softmax(logits, axis=-1) @ v[:, h]
    return out.reshape(len(tokens), C)


def attention_sublayer(x: np.ndarray, wt: Dict[str, np.ndarray], cfg, return_parts: bool = False,
                       window_rows=None):
    """One PSCWin attention sub-layer (a4-a7), pre-LN residual:
    u = LN1(x); qkv = u W_qkv^T + b_qkv; qkv_p = p W_qkv^T + b_qkv (p not normalised, Q14);
    O = window attention (plain if shift == 0, else padded shift);
    x_out = x + O W_o^T + b_o (P:L104 outer "Linear").
    window_rows: evaluate only these padded-grid window rows (attention_core_padded); other tokens are NaN."""
    u = layer_norm(x, wt["ln1_g"], wt["ln1_b"], cfg.ln_eps)
    qkv = u @ wt["w_qkv"].T + wt["b_qkv"]
    qkv_p = wt["pad"] @ wt["w_qkv"].T + wt["b_qkv"]
    O = attention_core_padded(qkv, qkv_p, cfg.H, cfg.W, cfg.heads, cfg.window,
                              cfg.shift_x, cfg.shift_y, cfg.pad_mode, cfg.rope, window_rows=window_rows)
    y = O @ wt["w_o"].T + wt["b_o"]
    out = x + y
    if return_parts:
        return out, dict(u=u, qkv=qkv, qkv_p=qkv_p, O=O, y=y)
    return out


# =============================================================================================
# §3.3 SSMs (Eqs. 2-5), the Mamba selective SSM and the cycle scan
# =============================================================================================

def zoh_discretize(delta: np.ndarray, A: np.ndarray, B: np.ndarray, bbar_mode: int = BBAR_ZOH):
    """Eq. 3 for diagonal A: A_bar = e^{Delta A};
    B_bar = (Delta A)^{-1} (e^{Delta A} - I) Delta B = (e^{Delta A} - 1)/A * B  (ZOH, reading Q11);
    EULER (Mamba kernel rule): B_bar = Delta B. delta [...,D,1]/[...,D], A [D,N], B [...,1,N]."""
    dA = delta * A
    A_bar = np.exp(dA)
    if bbar_mode == BBAR_ZOH:
        B_bar = np.expm1(dA) / A * B
    else:
        B_bar = delta * B
    return A_bar, B_bar


def selective_scan_sequential(v: np.ndarray, delta: np.ndarray, A: np.ndarray, Bm: np.ndarray,
                              Cm: np.ndarray, d_skip: np.ndarray, bbar_mode: int = BBAR_ZOH) -> np.ndarray:
    """Eq. 4, strictly sequential over the given sequence, every channel independently
    (P:L161): h_0 = 0; h_j = A_bar_j h_{j-1} + B_bar_j v_j; y_j = C_j . h_j + D_skip v_j.
    v, delta [S, D]; A [D, N]; Bm, Cm [S, N]. Returns y [S, D]."""
    S, D = v.shape
    N = A.shape[1]
    h = np.zeros((D, N))
    y = np.empty((S, D))
    for j in range(S):
        A_bar, B_bar = zoh_discretize(delta[j][:, None], A, Bm[j][None, :], bbar_mode)
        h = A_bar * h + B_bar * v[j][:, None]
        y[j] = h @ Cm[j] + d_skip * v[j]
    return y


def ssm_conv_kernel(A_bar: np.ndarray, B_bar: np.ndarray, C: np.ndarray, L: int) -> np.ndarray:
    """Eq. 5, LTI only: K = (C B, C A B, ..., C A^{L-1} B) per channel.
    A_bar, B_bar [D, N]; C [N]. Returns K [L, D]."""
    K = np.empty((L, A_bar.shape[0]))
    P = np.ones_like(A_bar)
    for i in range(L):
        K[i] = (P * B_bar) @ C
        P = P * A_bar
    return K


def causal_conv1d(xs: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Depthwise causal conv (Mamba block, Q9): c_j = b + sum_{i<k} w[:, i] * x_{j-k+1+i}; indices
    below 0 contribute 0 (Q10: applied to the literal 3L sequence). xs [S, D], w [D, k]."""
    S, D = xs.shape
    k = w.shape[1]
    c = np.tile(b, (S, 1)).astype(np.float64)
    for i in range(k):
        shift = k - 1 - i
        if shift == 0:
            c += w[:, i] * xs
        elif shift < S:
            c[shift:] += w[:, i] * xs[:S - shift]
    return c


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def softplus(x: np.ndarray) -> np.ndarray:
    return np.logaddexp(0.0, x)


def scan_permutation(H: int, W: int, order: int, window: int = 0) -> np.ndarray:
    """pi: scan position t -> grid token y*W+x (reading Q13; default row-major raster)."""
    idx = np.arange(H * W).reshape(H, W)
    if order == SCAN_ROW_MAJOR:
        return idx.reshape(-1)
    if order == SCAN_COL_MAJOR:
        return idx.T.reshape(-1)
    if order == SCAN_WINDOW_MAJOR:
        w = window
        return idx.reshape(H // w, w, W // w, w).transpose(0, 2, 1, 3).reshape(-1)
    raise ValueError(order)


def cycle_ssm_3L(xin3: np.ndarray, z3: Optional[np.ndarray], wt: Dict[str, np.ndarray], bbar_mode: int,
                 channels=None, z_sampled: bool = False) -> np.ndarray:
    """The Mamba SSM operator over the literal cycled sequence of 3L tokens ("repeats the image
    token sequence three times and connects them sequentially. The Mamba SSM operator then scans the
    tokens in this order"). Mamba-1 block internals per reading Q9:
      v = SiLU(causal_conv(xin));  (delta_low, B, C) = v W_x^T;  Delta = softplus(delta_low W_dt^T + b_dt);
      A = -exp(A_log);  y = selective scan (Eqs. 3-4) + D_skip v;  g = y * SiLU(z)  (no gate if z3 is None).
    xin3, z3 [3L, D]. Returns g3 [3L, D] (or [3L, len(channels)]: channels are independent, so a
    subset is exact for those channels — used to sample full-size cases). z_sampled: z3 holds only the
    sampled channels' columns [3L, len(channels)]."""
    R = wt["w_dt"].shape[1]
    N = wt["a_log"].shape[1]
    v = silu(causal_conv1d(xin3, wt["conv_w"], wt["conv_b"]))
    dbc = v @ wt["w_x"].T
    delta_low, Bm, Cm = dbc[:, :R], dbc[:, R:R + N], dbc[:, R + N:R + 2 * N]
    ch = slice(None) if channels is None else np.asarray(channels)
    delta = softplus(delta_low @ wt["w_dt"][ch].T + wt["b_dt"][ch])
    A = -np.exp(wt["a_log"][ch])
    y = selective_scan_sequential(v[:, ch], delta, A, Bm, Cm, wt["d_skip"][ch], bbar_mode)
    return y if z3 is None else y * silu(z3 if z_sampled else z3[:, ch])


def cycle_scan(xin: np.ndarray, z: Optional[np.ndarray], wt: Dict[str, np.ndarray], H: int, W: int,
               scan_order: int = SCAN_ROW_MAJOR, bbar_mode: int = BBAR_ZOH, window: int = 0,
               channels=None) -> np.ndarray:
    """ABI-level cycle scan (pscwin_cycle_scan): xin, z [B,L,D] in grid (row-major token) order.
    Per image: flatten in scan order, replicate three times, run the SSM over 3L (cycle_ssm_3L),
    "split into the corresponding three sequences and ... merged through summation".
    z None => no SiLU(z) gate. Returns g [B,L,D] (or [B,L,len(channels)]) in grid order."""
    B, L, D = xin.shape
    pi = scan_permutation(H, W, scan_order, window)
    nd = D if channels is None else len(channels)
    out = np.empty((B, L, nd))
    for b in range(B):
        s = xin[b][pi]
        z3 = None if z is None else np.concatenate([z[b][pi]] * 3)
        g3 = cycle_ssm_3L(np.concatenate([s, s, s]), z3, wt, bbar_mode, channels)
        out[b][pi] = g3[:L] + g3[L:2 * L] + g3[2 * L:]
    return out


def cycle_scan_module(x: np.ndarray, wt: Dict[str, np.ndarray], cfg, return_parts: bool = False,
                      channels=None):
    """Cycle-scan module before the attention block (a1-a3; SURVEY §8c oracle step 1):
    u0 = LN_s(x); flatten in scan order; MATERIALISE X3_j = s_{j mod L} (j < 3L); [xin, z] = X3 W_in^T
    (W_in applied to all 3L tokens); g3 = SSM(X3); o = g3 W_out^T; out_t = o_t + o_{L+t} + o_{2L+t};
    x[pi(t)] += out_t (pre-LN residual, Q13).
    channels: full-size sampling. Valid only for weights whose W_out columns outside `channels` are zero:
    then o = g[:, channels] W_out[:, channels]^T exactly, and the SSM runs on those channels alone (channels
    are independent given v, Delta, B, C)."""
    B, H, W, C = x.shape
    D = cfg.D
    L = H * W
    if channels is not None:
        ch = np.asarray(channels)
        rest = np.ones(D, dtype=bool)
        rest[ch] = False
        if np.any(wt["w_out"][:, rest] != 0):
            raise ValueError("channel sampling needs W_out to be zero outside the sampled channels")
    u0 = layer_norm(x, wt["lns_g"], wt["lns_b"], cfg.ln_eps).reshape(B, L, C)
    pi = scan_permutation(H, W, cfg.scan_order, cfg.window)
    out = x.reshape(B, L, C).copy()
    parts = []
    for b in range(B):
        s = u0[b][pi]
        X3 = np.concatenate([s, s, s])
        if channels is None:
            xz = X3 @ wt["w_in"].T
            g3 = cycle_ssm_3L(xz[:, :D], xz[:, D:], wt, cfg.bbar_mode)
            o3 = g3 @ wt["w_out"].T
        else:  # xin on every channel (conv, x_proj need them), z only on the sampled ones (row subset of W_in)
            xin3 = X3 @ wt["w_in"][:D].T
            z3 = X3 @ wt["w_in"][D + ch].T
            g3 = cycle_ssm_3L(xin3, z3, wt, cfg.bbar_mode, channels=ch, z_sampled=True)
            o3 = g3 @ wt["w_out"][:, ch].T
        o = o3[:L] + o3[L:2 * L] + o3[2 * L:]
        out[b][pi] += o
        parts.append(dict(g=(g3[:L] + g3[L:2 * L] + g3[2 * L:])))
    out = out.reshape(B, H, W, C)
    if return_parts:
        return out, parts
    return out


def gelu(x: np.ndarray) -> np.ndarray:
    """Exact GELU, x * Phi(x) = 0.5 x (1 + erf(x / sqrt 2)) (ViT / MAE FFN activation; reading Q21)."""
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def ffn_sublayer(x: np.ndarray, wt: Dict[str, np.ndarray], cfg) -> np.ndarray:
    """The ViT block's FFN ("the typical FFN has a hidden layer dimension of 768x4"), pre-LN residual
    (reading Q21): x + GELU(LN2(x) W_fc1^T + b_fc1) W_fc2^T + b_fc2."""
    u = layer_norm(x, wt["ln2_g"], wt["ln2_b"], cfg.ln_eps)
    h = gelu(u @ wt["w_fc1"].T + wt["b_fc1"])
    return x + h @ wt["w_fc2"].T + wt["b_fc2"]


def pscwin_layer(x: np.ndarray, wt: Dict[str, np.ndarray], cfg, window_rows=None, channels=None) -> np.ndarray:
    """One PSCWin layer: optional cycle-scan module ("prior to the final block of each stage")
    followed by the plain or padded-shift attention sub-layer, then (cfg.mlp_hidden > 0) the FFN sub-layer.
    Full-size sampling (exact for what it evaluates): window_rows = padded-grid window rows of the attention
    sub-layer (other tokens NaN); channels = SSM channels of the cycle-scan module (cycle_scan_module)."""
    if cfg.cycle_scan:
        x = cycle_scan_module(x, wt, cfg, channels=channels)
    x = attention_sublayer(x, wt, cfg, window_rows=window_rows)
    if getattr(cfg, "mlp_hidden", 0):
        x = ffn_sublayer(x, wt, cfg)
    return x


# =============================================================================================
# §3.4 Multi-scale fusion (HRSAM++): packed multi-scale token sequences
# =============================================================================================
# Packing (reading Q20): the token grids of all scales are flattened row-major and concatenated
# ("patchified and concatenated to form a sequence of image tokens with a length of
# (HW + H_sW_s)/16^2"). With a batch of B samples the scale is the OUTERMOST axis: scale s occupies
# packed rows [B*off_s, B*off_{s+1}) as a [B, H_s, W_s, C] block (off_s = sum of the earlier scales'
# H*W). For B = 1 this is exactly the paper's per-sample concatenation.

CS_NONE = 0
CS_SINGLE_SCALE = 1
CS_MULTI_SCALE = 2


def ms_offsets(scales) -> np.ndarray:
    """Per-sample token offsets of each scale segment: [0, L_0, L_0+L_1, ...] (SPEC S:L368 bounds)."""
    return np.concatenate([[0], np.cumsum([h * w for h, w in scales])]).astype(np.int64)


def ms_pack(grids) -> np.ndarray:
    """[B, H_s, W_s, C] per scale -> packed [B * sum L_s, C] (scale outermost, Q20)."""
    C = grids[0].shape[-1]
    if any(g.shape[-1] != C for g in grids):
        raise ValueError("all scales must share C")
    return np.concatenate([g.reshape(-1, C) for g in grids], axis=0)


def ms_unpack(xp: np.ndarray, B: int, scales):
    """Inverse of ms_pack: packed [B * sum L_s, C] -> list of [B, H_s, W_s, C]."""
    off = ms_offsets(scales)
    C = xp.shape[-1]
    return [xp[B * off[i]:B * off[i + 1]].reshape(B, h, w, C) for i, (h, w) in enumerate(scales)]


def ms_index_map(scales, w: int, sx: int = 0, sy: int = 0) -> np.ndarray:
    """Multi-scale indexing operator (App. C; "reorganized by indexing to ensure
    tokens within the same window are sequential and tokens from the same scale remain contiguous"):
    destination = the windows of scale 0 (row-major, slots row-major) then those of scale 1, ...;
    value = source position in the packed single-sample sequence, or PAD."""
    off = ms_offsets(scales)
    maps = []
    for i, (h, ww) in enumerate(scales):
        m = index_map(h, ww, w, sx, sy).astype(np.int64)
        maps.append(np.where(m == PAD, PAD, m + off[i]))
    return np.concatenate(maps).astype(np.uint32)


def ms_attention_sublayer(xp: np.ndarray, wt: Dict[str, np.ndarray], cfg, scales, window_rows=None) -> np.ndarray:
    """Multi-scale attention: "computationally equivalent to performing attention on isolated
    windows" — every scale's grid gets its own (plain / padded-shift) windows with the layer's window,
    shift and pad token, RoPE at the scale's own grid coordinates (reading Q20); no window spans two
    scales (block-diagonal mask). xp packed [B * sum L_s, C].
    window_rows: per scale, the padded-grid window rows to evaluate (None = all; sampling, other tokens NaN)."""
    B = xp.shape[0] // int(ms_offsets(scales)[-1])
    outs = []
    for i, (g, (h, w)) in enumerate(zip(ms_unpack(xp, B, scales), scales)):
        rows = None if window_rows is None else window_rows[i]
        outs.append(attention_sublayer(g, wt, cfg.replace(B=B, H=h, W=w), window_rows=rows))
    return ms_pack(outs)


def ms_cycle_scan_module(xp: np.ndarray, wt: Dict[str, np.ndarray], cfg, scales, mode: int,
                         channels=None) -> np.ndarray:
    """Cycle-scan module over a packed multi-scale sequence:
    SINGLE-SCALE "first splits the tokens by scale, scan each scale's tokens separately by the SSM, and
    then concatenates them" -> the single-scale module on every scale grid;
    MULTI-SCALE "directly performs the SSM across the tokens from all the scales": per sample, the
    scan-order sequences of all scales are concatenated (scale order) into ONE sequence of sum L_s tokens,
    which is cycled three times, scanned, split and summed like a single-scale sequence.
    Pre-LN residual (Q13). xp packed [B * sum L_s, C].
    channels: SSM channel sampling, valid when W_out is zero outside them (see cycle_scan_module)."""
    off = ms_offsets(scales)
    B = xp.shape[0] // int(off[-1])
    grids = ms_unpack(xp, B, scales)
    if mode == CS_SINGLE_SCALE:
        return ms_pack([cycle_scan_module(g, wt, cfg.replace(B=B, H=h, W=w), channels=channels)
                        for g, (h, w) in zip(grids, scales)])
    if mode != CS_MULTI_SCALE:
        raise ValueError(mode)
    D, C, Ltot = cfg.D, cfg.C, int(off[-1])
    outs = [g.reshape(B, -1, C).copy() for g in grids]
    for b in range(B):
        seq, pis = [], []
        for g, (h, w) in zip(grids, scales):
            pi = scan_permutation(h, w, cfg.scan_order, cfg.window)
            u0 = layer_norm(g[b].reshape(h * w, C), wt["lns_g"], wt["lns_b"], cfg.ln_eps)
            seq.append(u0[pi])
            pis.append(pi)
        s = np.concatenate(seq)
        X3 = np.concatenate([s, s, s])
        if channels is None:
            xz = X3 @ wt["w_in"].T
            g3 = cycle_ssm_3L(xz[:, :D], xz[:, D:], wt, cfg.bbar_mode)
            o3 = g3 @ wt["w_out"].T
        else:
            ch = np.asarray(channels)
            rest = np.ones(D, dtype=bool)
            rest[ch] = False
            if np.any(wt["w_out"][:, rest] != 0):
                raise ValueError("channel sampling needs W_out to be zero outside the sampled channels")
            xin3 = X3 @ wt["w_in"][:D].T
            z3 = X3 @ wt["w_in"][D + ch].T
            g3 = cycle_ssm_3L(xin3, z3, wt, cfg.bbar_mode, channels=ch, z_sampled=True)
            o3 = g3 @ wt["w_out"][:, ch].T
        o = o3[:Ltot] + o3[Ltot:2 * Ltot] + o3[2 * Ltot:]
        for i, pi in enumerate(pis):
            outs[i][b][pi] += o[off[i]:off[i + 1]]
    return ms_pack(outs)


def ms_layer(xp: np.ndarray, wt: Dict[str, np.ndarray], cfg, scales, attention: int = 1,
             cycle_scan: int = CS_NONE, window_rows=None, channels=None) -> np.ndarray:
    """One HRSAM++ layer over a packed multi-scale sequence: optional cycle-scan module (single- or
    multi-scale) followed (attention = 1) by the multi-scale window-attention sub-layer.
    window_rows (per scale) / channels: full-size sampling as in pscwin_layer."""
    if cycle_scan:
        xp = ms_cycle_scan_module(xp, wt, cfg, scales, cycle_scan, channels=channels)
    if attention:
        xp = ms_attention_sublayer(xp, wt, cfg, scales, window_rows=window_rows)
        if getattr(cfg, "mlp_hidden", 0):
            xp = ffn_sublayer(xp, wt, cfg)
    return xp


# =============================================================================================
# Encoder ends (reading Q22)
# =============================================================================================

def patch_embed(img: np.ndarray, w: np.ndarray, b: np.ndarray, p: int = 16) -> np.ndarray:
    """ViT patch embedding ("image encoder ... ViT"; 1024^2 -> 64 x 64 tokens): a p x p convolution
    with stride p, written out as its definition. img [B, 3, pH, pW]; w [C, 3, p, p]; b [C]. Returns [B, H, W, C]
    (no absolute position embedding: positions enter through RoPE, reading Q22)."""
    B, Ci, Hi, Wi = img.shape
    H, W = Hi // p, Wi // p
    patches = img.reshape(B, Ci, H, p, W, p).transpose(0, 2, 4, 1, 3, 5).reshape(B, H, W, Ci * p * p)
    return patches @ w.reshape(w.shape[0], -1).T + b


def conv3x3(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """3 x 3 convolution, stride 1, zero padding 1, no bias, channels-last: out[b,y,x,o] =
    sum_{dy,dx,i} x[b, y+dy-1, x+dx-1, i] w[o, i, dy, dx]. x [B,H,W,Ci]; w [Co, Ci, 3, 3]."""
    B, H, W, Ci = x.shape
    xp = np.zeros((B, H + 2, W + 2, Ci))
    xp[:, 1:H + 1, 1:W + 1] = x
    out = np.zeros((B, H, W, w.shape[0]))
    for dy in range(3):
        for dx in range(3):
            out += xp[:, dy:dy + H, dx:dx + W] @ w[:, :, dy, dx].T
    return out


def encoder_neck(stage_outs, wt: Dict[str, np.ndarray], eps: float = 1e-6) -> np.ndarray:
    """HRSAM's output fusion ("fusing outputs from all four stages through summation, followed by a
    convolutional block"; "the output dimension of each stage is 256"), reading Q22: each stage output is
    projected to 256 channels (1x1 conv, no bias), the projections are summed, and the sum passes SAM's neck
    block LN2d -> conv3x3 (no bias) -> LN2d. stage_outs: list of [B,H,W,C]. Returns [B,H,W,256]."""
    f = sum(s @ wt[f"w_stage{i}"].T for i, s in enumerate(stage_outs))
    f = layer_norm(f, wt["neck_ln1_g"], wt["neck_ln1_b"], eps)
    f = conv3x3(f, wt["w_neck_conv"])
    return layer_norm(f, wt["neck_ln2_g"], wt["neck_ln2_b"], eps)


def resize_bilinear(x: np.ndarray, H: int, W: int) -> np.ndarray:
    """Bilinear resize, align_corners = False (half-pixel centres; reading Q22), channels-last [B,h,w,C] ->
    [B,H,W,C]: source coordinate s = (d + 0.5) * in / out - 0.5 clamped at 0, linear weights between floor(s)
    and floor(s) + 1 (clamped to the last row / column). HRSAM++ resizes the overview scale's outputs to the main
    grid (Fig. 4 caption)."""
    B, h, w, C = x.shape

    def axis(n_out, n_in):
        s = np.maximum((np.arange(n_out) + 0.5) * n_in / n_out - 0.5, 0.0)
        i0 = np.minimum(np.floor(s).astype(int), n_in - 1)
        i1 = np.minimum(i0 + 1, n_in - 1)
        return i0, i1, s - i0

    y0, y1, fy = axis(H, h)
    x0, x1, fx = axis(W, w)
    top = x[:, y0][:, :, x0] * (1 - fx)[None, None, :, None] + x[:, y0][:, :, x1] * fx[None, None, :, None]
    bot = x[:, y1][:, :, x0] * (1 - fx)[None, None, :, None] + x[:, y1][:, :, x1] * fx[None, None, :, None]
    return top * (1 - fy)[None, :, None, None] + bot * fy[None, :, None, None]
