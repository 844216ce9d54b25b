"""Helpers for the GPU parity tests: move synth (fp64, storage-exact) arrays to the device in the dtype the
ABI expects, and the error metric of DESIGN.md "Tolerances" (reading Q17)."""
import numpy as np

F32_KEYS = {"ln1_g", "ln1_b", "b_qkv", "b_o", "lns_g", "lns_b", "conv_w", "conv_b", "w_dt", "b_dt", "a_log",
            "d_skip", "ln2_g", "ln2_b", "b_fc1", "b_fc2"}


def dev(a, dtype="bf16"):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    t = t.to(torch.bfloat16) if dtype == "bf16" else t
    return t.cuda().contiguous()


def host(t):
    import torch
    return t.detach().to(torch.float64).cpu().numpy()


def dev_weights(w, cfg):
    return {k: dev(v, "f32" if (k in F32_KEYS or cfg.dtype == "f32") else "bf16") for k, v in w.items()}


def rel_err(got, ref):
    """max |g - o| / max |o|  (reading Q17)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    assert np.all(np.isfinite(got)), "non-finite GPU output"
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-30))


BF16_TOL = 2e-2   # north star: bf16 inputs, fp32 accumulate
F32_TOL = 1e-4    # north star: fp32 path


X_SCALE = 0.02    # residual-stream scale of the layer-level parity cases (synth.make_input(scale=...))


def layer_gate(got, x, ref, n_res, tol=BF16_TOL, storage="bf16"):
    """Layer-level parity gate on the sub-layer INCREMENT: a layer computes
    x_out = x + inc, and on a realistic residual stream max|x| >> max|inc|, so a gate on x_out alone passes a layer
    that returns its input. This gate bounds the increment error by the tolerance times the increment's own
    magnitude, plus one storage half-ulp (<= 2^-8 relative for bf16, 2^-24 for f32) of x_out per residual store
    (Q16: cycle-scan module, attention, FFN). Returns err / bound (the gate passes below 1)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64).reshape(ref.shape)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    assert np.all(np.isfinite(got)), "non-finite GPU output"
    inc = ref - x
    half_ulp = 2.0 ** -8 if storage == "bf16" else 2.0 ** -24
    bound = tol * np.max(np.abs(inc)) + n_res * half_ulp * np.max(np.abs(ref))
    return float(np.max(np.abs(got - ref)) / bound)


def n_residual(cfg, attention=1, cs=None):
    """Residual stores of x in one layer: cycle-scan module, attention sub-layer, FFN sub-layer."""
    cs = cfg.cycle_scan if cs is None else cs
    return int(bool(cs)) + attention + int(attention and cfg.mlp_hidden > 0)


def masked_w_out(w, channels):
    """Weights with W_out zero outside the sampled SSM channels: full-size cycle-scan parity cases run every channel
    on the GPU while the oracle evaluates only `channels` (exact for this weight pattern; oracle.cycle_scan_module)."""
    m = np.zeros_like(w["w_out"])
    m[:, channels] = w["w_out"][:, channels]
    return dict(w, w_out=m)


def sampled_gate(got, x, ref, n_res, tol=BF16_TOL):
    """layer_gate restricted to the tokens the sampled oracle evaluated (the others are NaN in ref)."""
    sel = ~np.isnan(np.asarray(ref))
    assert sel.sum() > 0
    g = np.asarray(got, dtype=np.float64)
    assert np.all(np.isfinite(g)), "non-finite GPU output"
    return layer_gate(g[sel], np.asarray(x, dtype=np.float64).reshape(g.shape)[sel], np.asarray(ref)[sel], n_res, tol)
