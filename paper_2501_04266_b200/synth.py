"""Seeded synthetic inputs shared by the tests, the oracle runs and bench.py.

This module holds NO arithmetic of the method (no quantization, no partition
map, no reduction).  It only draws numbers: GPT-shaped parameter / gradient
tensors with the value distributions of DESIGN.md §4 and a set of hand-placed
special blocks that exercise the quantizer's edge cases (zero block, constant
block, exact rounding ties, outliers, subnormal-only and tiny-normal blocks).

NumPy generators (``np.random.default_rng(seed)``) are used for everything the
CPU oracle also consumes; ``torch_*`` helpers draw the large bench tensors on
the GPU with ``torch.Generator(device).manual_seed``.
"""

import math

import numpy as np

# GPT shapes (external to the paper: GPT-3 table and the GPT-NeoX-20B config;
# see DESIGN.md §4).  Per layer: 12 h^2 + 13 h parameters.
GPT_CONFIGS = {
    "gpt1.3b": {"layers": 24, "hidden": 2048, "vocab": 50304, "embeddings": 1},
    "gpt6.7b": {"layers": 32, "hidden": 4096, "vocab": 50304, "embeddings": 1},
    "neox20b": {"layers": 44, "hidden": 6144, "vocab": 50432, "embeddings": 2},
}


def layer_numel(hidden):
    return 12 * hidden * hidden + 13 * hidden


def model_tensors(name):
    """List of (label, numel) flat buffers of one model: every transformer layer, then
    the embedding matrix (matrices)."""
    c = GPT_CONFIGS[name]
    out = [(f"layer{i}", layer_numel(c["hidden"])) for i in range(c["layers"])]
    for e in range(c["embeddings"]):
        out.append((f"embed{e}", c["vocab"] * c["hidden"]))
    return out


def special_blocks(block, bits_for_ties=(8, 4), rng=None):
    """A list of hand-made blocks (each ``block`` fp32 values) that hit quantizer edge cases."""
    rng = rng or np.random.default_rng(7)
    out = []
    out.append(np.zeros(block, np.float32))                                 # all zero
    b = np.full(block, 0.75, np.float32)
    b[1::2] = -0.75
    out.append(b)                                                           # constant +-absmax
    for qmax in (127 if 8 in bits_for_ties else None, 7 if 4 in bits_for_ties else None):
        if qmax is None:
            continue
        # absmax = qmax * 2^-3 makes qmax/absmax = 2^3 exactly, so x = (k + 0.5) * 2^-3
        # lands exactly on a rounding tie k + 0.5 after the multiply.
        k = rng.integers(-qmax, qmax, size=block).astype(np.float32)
        t = ((k + 0.5) * 0.125).astype(np.float32)
        t[0] = qmax * 0.125
        out.append(t)
    out.append((rng.standard_normal(block) * 1e-40).astype(np.float32))    # subnormal only
    out.append((rng.standard_normal(block) * 1.2e-38).astype(np.float32))  # tiny normal (< 2^-100)
    b = (rng.uniform(-1, 1, block) * 2.0 ** -100).astype(np.float32)
    b[3] = np.float32(2.0 ** -100) * np.float32(1.5)                        # absmax just above 2^-100
    out.append(b)
    b = (rng.standard_normal(block) * 1e-3).astype(np.float32)
    b[block // 2] = np.float32(1e-3 * 64)                                   # single big outlier
    out.append(b)
    return out


def gradient_like(n, seed, block=256, specials=True, std=1e-3, zero_block_frac=0.01,
                  outlier_every=1024):
    """fp32 gradient-like vector: N(0, std^2), 1/outlier_every elements scaled x64,
    ~1 % all-zero blocks, special blocks at the start (if they fit)."""
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(n) * std).astype(np.float32)
    if outlier_every:
        idx = rng.integers(0, n, size=max(1, n // outlier_every)) if n else np.zeros(0, int)
        x[idx] *= np.float32(64)
    nb = n // block
    if zero_block_frac and nb:
        zb = rng.choice(nb, size=max(1, int(nb * zero_block_frac)), replace=False)
        for b in zb:
            x[b * block:(b + 1) * block] = 0
    if specials:
        sp = special_blocks(block, rng=rng)
        for i, b in enumerate(sp):
            if (i + 1) * block <= n:
                x[i * block:(i + 1) * block] = b * (std / 1e-3) if i == 1 else b
    return x


def params_like(n, seed, block=256, specials=True, std=0.02):
    """fp32 parameter-like vector N(0, std^2) with the special blocks at the start."""
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(n) * std).astype(np.float32)
    if specials:
        sp = special_blocks(block, rng=rng)
        for i, b in enumerate(sp):
            if (i + 1) * block <= n:
                x[i * block:(i + 1) * block] = b
    return x


def to_bf16_bits(x):
    """Round an fp32 array to bf16 (RNE) and return it as ml_dtypes.bfloat16.
    Input generation only: the bench and tests feed bf16 tensors."""
    import ml_dtypes
    return np.asarray(x, np.float32).astype(ml_dtypes.bfloat16)


# ---------------------------------------------------------------- torch (GPU) side
def torch_normal(n, seed, std, dtype, device, outlier_every=1024):
    """Large bench tensors drawn on the device (no host round trip)."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    x = torch.randn(n, generator=gen, device=device, dtype=torch.float32).mul_(std)
    if outlier_every:
        k = max(1, n // outlier_every)
        idx = torch.randint(0, n, (k,), generator=gen, device=device)
        x[idx] *= 64
    return x.to(dtype)


def sample_blocks(nblocks, chunk_bounds, every=997):
    """Block indices for sampled parity at full size: every ``every``-th block plus both
    edge blocks of each chunk boundary (block offsets in ``chunk_bounds``)."""
    s = set(range(0, nblocks, every))
    s.add(nblocks - 1)
    for b in chunk_bounds:
        for v in (b - 1, b):
            if 0 <= v < nblocks:
                s.add(v)
    return np.array(sorted(s), dtype=np.int64)


def ceil_div(a, b):
    return -(-a // b)


__all__ = ["GPT_CONFIGS", "layer_numel", "model_tensors", "special_blocks", "gradient_like",
           "params_like", "to_bf16_bits", "torch_normal", "sample_blocks", "ceil_div", "math"]
