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
