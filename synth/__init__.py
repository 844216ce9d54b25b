"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no LayerNorm, projection, RoPE,
attention or scan). It only draws numbers and rounds them to the storage
precision both sides consume, so that `oracle/` and the CUDA path see
bit-identical inputs (SURVEY.md §8(d) "Inputs").

Generator: a counter-based splitmix64 stream ("splitmix-style
update ... so alternates reproduce streams"): value i of stream s is
splitmix64(s * GOLDEN + (i + 1) * GOLDEN). Uniforms take the top 53 bits;
normals use Box-Muller on consecutive uniform pairs.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

PAD_LEARNABLE = 0
PAD_MASKED = 1
SCAN_ROW_MAJOR = 0
SCAN_COL_MAJOR = 1
SCAN_WINDOW_MAJOR = 2
BBAR_ZOH = 0
BBAR_EULER = 1


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z.copy()
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def stream_seed(*parts: int) -> int:
    """Fold a tuple of small ints into one 64-bit stream id."""
    s = np.uint64(0x243F6A8885A308D3)
    for p in parts:
        with np.errstate(over="ignore"):
            s = _splitmix64(np.array([s ^ np.uint64(p & 0xFFFFFFFFFFFFFFFF)], dtype=np.uint64))[0]
    return int(s)


def uniform(seed: int, n: int) -> np.ndarray:
    """n uniforms in [0, 1) from stream `seed` (float64)."""
    i = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) * GOLDEN + i * GOLDEN
    r = _splitmix64(z) >> np.uint64(11)
    return r.astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed: int, n: int) -> np.ndarray:
    """n standard normals (Box-Muller over consecutive uniform pairs)."""
    m = (n + 1) // 2
    u = uniform(seed, 2 * m)
    u1 = 1.0 - u[0::2]  # (0, 1]
    u2 = u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    out = np.empty(2 * m)
    out[0::2] = r * np.cos(2.0 * math.pi * u2)
    out[1::2] = r * np.sin(2.0 * math.pi * u2)
    return out[:n]


# ----------------------------------------------------------------------------------------------
# Storage rounding (not method arithmetic: it fixes the bytes both sides read)
# ----------------------------------------------------------------------------------------------

def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float64 -> float32 -> bf16 (round-to-nearest-even); returns uint16 bits."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    b = (b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)
    return b.astype(np.uint16)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def round_bf16(x: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f64(to_bf16_bits(x)).reshape(np.shape(x))


def round_f32(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, dtype=np.float32).astype(np.float64)


# ----------------------------------------------------------------------------------------------
# Layer configuration (mirrors pscwin_layer_desc in include/pscwin.h)
# ----------------------------------------------------------------------------------------------

@dataclasses.dataclass(frozen=True)
class LayerConfig:
    B: int
    H: int
    W: int
    C: int
    heads: int
    window: int
    shift_x: int = 0
    shift_y: int = 0
    pad_mode: int = PAD_LEARNABLE
    rope: int = 1
    cycle_scan: int = 0
    ssm_state: int = 32
    ssm_expand: int = 2
    ssm_dt_rank: int = 0          # 0 => ceil(C / 16) (Mamba default)
    ssm_conv: int = 4
    scan_order: int = SCAN_ROW_MAJOR
    bbar_mode: int = BBAR_ZOH
    dtype: str = "bf16"           # "bf16" or "f32"
    ln_eps: float = 1e-6
    mlp_hidden: int = 0           # FFN hidden width (768 x 4); 0 = no FFN sub-layer

    @property
    def d_head(self) -> int:
        return self.C // self.heads

    @property
    def D(self) -> int:
        return self.ssm_expand * self.C

    @property
    def R(self) -> int:
        return self.ssm_dt_rank if self.ssm_dt_rank > 0 else -(-self.C // 16)

    @property
    def N(self) -> int:
        return self.ssm_state

    @property
    def L(self) -> int:
        return self.H * self.W

    def replace(self, **kw) -> "LayerConfig":
        return dataclasses.replace(self, **kw)


def tiny(**kw) -> LayerConfig:
    """configs[0]: 1 image, 16x16 grid, dim 64, 2 heads, window 8, shift 4, state 16 (BASELINE.json)."""
    base = dict(B=1, H=16, W=16, C=64, heads=2, window=8, shift_x=4, shift_y=4,
                ssm_state=16, ssm_dt_rank=4)
    base.update(kw)
    return LayerConfig(**base)


def vitb(side_tokens: int, B: int = 1, **kw) -> LayerConfig:
    """ViT-B PSCWin layer on a side_tokens^2 grid (1024^2 -> 64, 2048^2 -> 128, 4096^2 -> 256)."""
    base = dict(B=B, H=side_tokens, W=side_tokens, C=768, heads=12, window=16, shift_x=8, shift_y=8,
                ssm_state=32, ssm_expand=2, ssm_conv=4)
    base.update(kw)
    return LayerConfig(**base)


def stack_layer_kind(i: int):
    """Global-alternation stack: layer i plain if even, shifted if odd;
    a cycle-scan module precedes layers 2, 5, 8, 11. Returns (shifted, cycle_scan)."""
    return (i % 2 == 1), (i % 3 == 2)


# ----------------------------------------------------------------------------------------------
# Inputs and weights
# ----------------------------------------------------------------------------------------------

def _store(x: np.ndarray, kind: str, cfg: LayerConfig) -> np.ndarray:
    """kind 'mat' = tensor stored in the activation/GEMM dtype; 'f32' = always-f32 parameter."""
    if kind == "mat" and cfg.dtype == "bf16":
        return round_bf16(x)
    return round_f32(x)


def make_input(cfg: LayerConfig, layer: int = 0, scale: float = 1.0) -> np.ndarray:
    """x ~ N(0, scale^2), shape [B,H,W,C] (seed 1 + layer). The layer-level parity gates use a small residual
    stream (scale 0.02): LayerNorm makes every sub-layer's increment independent of the scale of x, so the
    increment dominates x_out and a layer that returns its input (or drops a sub-layer) fails the gate."""
    n = cfg.B * cfg.H * cfg.W * cfg.C
    return _store(scale * normal(stream_seed(1 + layer, 0), n).reshape(cfg.B, cfg.H, cfg.W, cfg.C), "mat", cfg)


def make_weights(cfg: LayerConfig, layer: int = 0, peaky: bool = False,
                 scan_params: str = "varied") -> Dict[str, np.ndarray]:
    """Weights of one PSCWin layer (SURVEY §8(d) recipe). Linear weights are nn.Linear-style [out, in].

    GEMM matrices and the pad token p are stored in the activation dtype; LN parameters, biases,
    conv, dt_proj, A_log and D_skip are f32.

    scan_params: "varied" (default) draws channel-dependent SSM parameters, A_log[d,n] = log(n+1) + U(-0.5, 0.5)
    and D_skip[d] ~ U(0.5, 1.5), so a kernel that indexes them by the wrong channel fails parity; "mamba" is the
    channel-uniform S4D-real init (A_log = log(n+1), D_skip = 1) of round 1."""
    C, D, N, R, K = cfg.C, cfg.D, cfg.N, cfg.R, cfg.ssm_conv
    s = 100 + layer
    g = lambda idx, n: normal(stream_seed(s, idx), n)
    u = lambda idx, n: uniform(stream_seed(s, idx), n)
    w: Dict[str, np.ndarray] = {}
    w["ln1_g"] = _store(1.0 + 0.1 * g(1, C), "f32", cfg)
    w["ln1_b"] = _store(0.02 * g(2, C), "f32", cfg)
    wq = 0.02 * g(3, 3 * C * C).reshape(3 * C, C)
    if peaky:
        wq[:C] *= 8.0
    w["w_qkv"] = _store(wq, "mat", cfg)
    w["b_qkv"] = _store(0.02 * g(4, 3 * C), "f32", cfg)
    w["pad"] = _store(g(5, C), "mat", cfg)
    w["w_o"] = _store(0.02 * g(6, C * C).reshape(C, C), "mat", cfg)
    w["b_o"] = _store(0.02 * g(7, C), "f32", cfg)
    # cycle-scan (Mamba-1 block)
    w["lns_g"] = _store(1.0 + 0.1 * g(11, C), "f32", cfg)
    w["lns_b"] = _store(0.02 * g(12, C), "f32", cfg)
    w["w_in"] = _store(0.02 * g(13, 2 * D * C).reshape(2 * D, C), "mat", cfg)
    bound = 1.0 / math.sqrt(K)
    w["conv_w"] = _store((2.0 * u(14, D * K) - 1.0).reshape(D, K) * bound, "f32", cfg)
    w["conv_b"] = _store((2.0 * u(15, D) - 1.0) * bound, "f32", cfg)
    w["w_x"] = _store(0.02 * g(16, (R + 2 * N) * D).reshape(R + 2 * N, D), "mat", cfg)
    w["w_dt"] = _store((2.0 * u(17, D * R) - 1.0).reshape(D, R) / math.sqrt(R), "f32", cfg)
    dt0 = np.exp(math.log(1e-3) + u(18, D) * (math.log(1e-1) - math.log(1e-3)))
    w["b_dt"] = _store(dt0 + np.log(-np.expm1(-dt0)), "f32", cfg)  # softplus^{-1}(dt0)
    a_log = np.log(np.tile(np.arange(1, N + 1, dtype=np.float64), (D, 1)))
    if scan_params == "varied":
        w["a_log"] = _store(a_log + (u(27, D * N).reshape(D, N) - 0.5), "f32", cfg)
        w["d_skip"] = _store(0.5 + u(28, D), "f32", cfg)
    elif scan_params == "mamba":
        w["a_log"] = _store(a_log, "f32", cfg)
        w["d_skip"] = _store(np.ones(D), "f32", cfg)
    else:
        raise ValueError(scan_params)
    w["w_out"] = _store(0.02 * g(19, C * D).reshape(C, D), "mat", cfg)
    # FFN sub-layer ("the typical FFN has a hidden layer dimension of 768x4"; reading Q21)
    Hd = cfg.mlp_hidden if cfg.mlp_hidden > 0 else 4 * C
    w["ln2_g"] = _store(1.0 + 0.1 * g(21, C), "f32", cfg)
    w["ln2_b"] = _store(0.02 * g(22, C), "f32", cfg)
    w["w_fc1"] = _store(0.02 * g(23, Hd * C).reshape(Hd, C), "mat", cfg)
    w["b_fc1"] = _store(0.02 * g(24, Hd), "f32", cfg)
    w["w_fc2"] = _store(0.02 * g(25, C * Hd).reshape(C, Hd), "mat", cfg)
    w["b_fc2"] = _store(0.02 * g(26, C), "f32", cfg)
    return w


def make_qkv(cfg: LayerConfig, seed: int = 7) -> np.ndarray:
    """Standalone QKV buffer [B,H,W,3C] (~N(0, 0.5^2)) for the attention-core ABI tests."""
    n = cfg.B * cfg.H * cfg.W * 3 * cfg.C
    return _store(0.5 * normal(stream_seed(seed, 1), n).reshape(cfg.B, cfg.H, cfg.W, 3 * cfg.C), "mat", cfg)


def make_pad_qkv(cfg: LayerConfig, seed: int = 7) -> np.ndarray:
    return _store(0.5 * normal(stream_seed(seed, 2), 3 * cfg.C), "mat", cfg)


def make_image(B: int, H: int, W: int, seed: int = 50) -> np.ndarray:
    """Synthetic input image [B, 3, 16H, 16W] ~ N(0,1) (normalised pixels), stored in bf16."""
    n = B * 3 * 16 * H * 16 * W
    return round_bf16(normal(stream_seed(seed, B, H, W), n).reshape(B, 3, 16 * H, 16 * W))


def make_ends_weights(C: int = 768, C_out: int = 256, n_stages: int = 4, seed: int = 300) -> Dict[str, np.ndarray]:
    """Encoder-end weights (reading Q22): patch embedding conv [C, 3, 16, 16] + bias, per-stage 1x1 projections
    [C_out, C], neck LN2d / conv3x3 [C_out, C_out, 3, 3] / LN2d. Matrices bf16, LN params / bias f32."""
    g = lambda idx, n: normal(stream_seed(seed, idx), n)
    w: Dict[str, np.ndarray] = {}
    w["w_patch"] = round_bf16(0.02 * g(1, C * 768).reshape(C, 3, 16, 16))
    w["b_patch"] = round_f32(0.02 * g(2, C))
    for i in range(n_stages):
        w[f"w_stage{i}"] = round_bf16(0.02 * g(10 + i, C_out * C).reshape(C_out, C))
    w["neck_ln1_g"] = round_f32(1.0 + 0.1 * g(20, C_out))
    w["neck_ln1_b"] = round_f32(0.02 * g(21, C_out))
    w["w_neck_conv"] = round_bf16(0.02 * g(22, C_out * C_out * 9).reshape(C_out, C_out, 3, 3))
    w["neck_ln2_g"] = round_f32(1.0 + 0.1 * g(23, C_out))
    w["neck_ln2_b"] = round_f32(0.02 * g(24, C_out))
    return w
