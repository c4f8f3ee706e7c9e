"""O4-O6: symmetric absmax block quantization, int4 packing, dequantization.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Paper: "ZeRO++ utilizes block-based quantization, which quantizes blocks of FP16
data into INT8 or INT4 blocks"; weights INT8, gradients INT4
(P:122).  The paper fixes neither the formula nor the rounding; the readings
used here (R1-R5) are:

  R1  symmetric absmax per block, no zero point; qmax = 127 (int8) / 7 (int4);
      the most-negative code (-128 / -8) is never emitted.
  R2  fp32 arithmetic: x widened exactly to fp32 (bf16/fp16 -> fp32 is exact),
        am    = max_i |x_i|                      (exact)
        scale = fl32(am / qmax)
        inv   = fl32(qmax / am)
        code  = clamp(rne(fl32(x_i * inv)), -qmax, qmax)
      Multiplying by ``inv`` (not dividing by ``scale``) is the only fp32 form
      that reproduces SPEC's worked example [8,-8,4,2] -> [7,-7,4,2]
      (tests/golden/quant_examples.json).
  R3  a block whose am < 2**-100 (zero, subnormal, tiny) gets scale 0, codes 0.
  R4  int4 packing: byte j = (c[2j] & 0xF) | ((c[2j+1] & 0xF) << 4).
  R5  dequantize: x_hat = fl32(code * scale); bf16 output is RNE of x_hat.

Layout (R6): one global codes array (unpacked int8 codes here; ``pack_int4``
gives the wire bytes) and one global fp32 scales array, block k at index k.
"""

import numpy as np
import ml_dtypes

TINY = np.float32(2.0 ** -100)          # R3
QMAX = {8: 127, 4: 7}                   # R1


def qmax_of(bits):
    if bits not in QMAX:
        raise ValueError(f"bits must be 4 or 8, got {bits}")
    return QMAX[bits]


def to_f32(x):
    """Exact widening of bf16 / fp16 / fp32 input to fp32 (R2)."""
    x = np.asarray(x)
    if x.dtype == np.float64:
        raise TypeError("oracle inputs are bf16/fp16/fp32; fp64 would round on widening")
    return x.astype(np.float32)


def quantize(x, bits, block):
    """O4.  x: 1-D bf16/fp16/fp32 with len(x) % block == 0.

    Returns (codes int8[n] (logical, unpacked), scales float32[n // block]).
    Follows R1-R3 step by step, one block at a time in vectorised form
    (blocks are independent, so the row-wise form is the definition).
    """
    qmax = np.float32(qmax_of(bits))
    x32 = to_f32(x)
    n = x32.shape[0]
    if n % block:
        raise ValueError("len(x) must be a multiple of block")
    xb = x32.reshape(n // block, block)
    am = np.max(np.abs(xb), axis=1) if n else np.zeros(0, np.float32)
    is_tiny = am < TINY
    am_safe = np.where(is_tiny, np.float32(1), am).astype(np.float32)
    scale = np.where(is_tiny, np.float32(0), am_safe / qmax).astype(np.float32)
    inv = np.where(is_tiny, np.float32(0), qmax / am_safe).astype(np.float32)
    prod = (xb * inv[:, None]).astype(np.float32)        # fl32(x * inv)
    codes = np.rint(prod)                                # round half to even
    codes = np.clip(codes, -qmax, qmax).astype(np.int8)
    return codes.reshape(n), scale


def dequantize(codes, scales, block, out="f32"):
    """O6.  x_hat = fl32(code * scale); out in {"f32", "bf16", "f16"} (RNE narrowing)."""
    c = np.asarray(codes).astype(np.float32).reshape(-1, block)
    s = np.asarray(scales, dtype=np.float32)
    xh = (c * s[:, None]).astype(np.float32).reshape(-1)
    if out == "f32":
        return xh
    if out == "bf16":
        return xh.astype(ml_dtypes.bfloat16)
    if out == "f16":
        return xh.astype(np.float16)                     # IEEE RNE
    raise ValueError(out)


def pack_int4(codes):
    """R4: two signed 4-bit codes per byte, even element in the low nibble."""
    c = np.asarray(codes).astype(np.int16)
    if c.shape[0] % 2:
        raise ValueError("int4 packing needs an even count")
    lo = c[0::2] & 0xF
    hi = c[1::2] & 0xF
    return (lo | (hi << 4)).astype(np.uint8)


def unpack_int4(packed):
    """Inverse of R4 with sign extension."""
    b = np.asarray(packed, dtype=np.uint8).astype(np.int16)
    lo = b & 0xF
    hi = (b >> 4) & 0xF
    lo = np.where(lo >= 8, lo - 16, lo)
    hi = np.where(hi >= 8, hi - 16, hi)
    out = np.empty(b.shape[0] * 2, np.int8)
    out[0::2] = lo
    out[1::2] = hi
    return out


def wire_codes(codes, bits):
    """The byte array a rank puts on the wire for ``codes`` (R4 / two's complement)."""
    if bits == 8:
        return np.asarray(codes, dtype=np.int8).view(np.uint8)
    return pack_int4(codes)


def from_wire(buf, bits):
    if bits == 8:
        return np.asarray(buf, dtype=np.uint8).view(np.int8)
    return unpack_int4(buf)


def quantized_size_bytes(n, bits, block, scale_bytes=4):
    """SPEC quantized_size_bytes with our 4-byte fp32 scales."""
    nblocks = -(-n // block)
    return -(-n * bits // 8) + nblocks * scale_bytes
