"""Pins for oracle/quant.py (O4-O6) against SPEC worked examples, exact rational
brute force, and properties that any correct symmetric absmax quantizer has.
None of these re-types the oracle's formula."""

import json
import os
from fractions import Fraction

import ml_dtypes
import numpy as np
import pytest

from oracle import quant

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def test_spec_worked_examples():
    g = _golden("quant_examples.json")
    for ex in g["quantize"]:
        x = np.array(ex["x"], np.float32)
        codes, scales = quant.quantize(x, ex["bits"], ex["block"])
        assert codes.tolist() == ex["codes"], ex["cite"]
        want = np.float32(ex["scale_num"] / ex["scale_den"])        # fl32 of the exact ratio
        assert scales[0] == want, ex["cite"]


def test_spec_sizes():
    for ex in _golden("quant_examples.json")["sizes"]:
        got = quant.quantized_size_bytes(ex["n"], ex["bits"], ex["block"], ex["scale_bytes"])
        assert got == ex["bytes"], ex["cite"]


def _rne_fraction(q):
    """Round a Fraction to the nearest integer, ties to even."""
    f = q.numerator // q.denominator
    rem = q - f
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and f % 2 == 1):
        return f + 1
    return f


@pytest.mark.parametrize("bits", [8, 4])
def test_brute_force_exact_rational(bits):
    """code_i = the integer nearest to x_i * qmax / absmax (exact rationals), clamped;
    scale = the fp32 nearest to absmax / qmax.  Skip elements whose exact value lies
    within 1e-5 of a rounding boundary (there fp32 rounding of inv may legitimately
    decide)."""
    rng = np.random.default_rng(11 + bits)
    qmax = {8: 127, 4: 7}[bits]
    checked = 0
    for trial in range(60):
        block = int(rng.choice([1, 2, 3, 8, 32]))
        x = (rng.standard_normal(block) * 10.0 ** rng.integers(-6, 6)).astype(np.float32)
        codes, scales = quant.quantize(x, bits, block)
        am = max(abs(Fraction(float(v))) for v in x)
        if am == 0:
            assert scales[0] == 0 and not codes.any()
            continue
        # scale: fp64 division then fp32 rounding is correctly rounded (53 >= 2*24+2)
        assert scales[0] == np.float32(float(am) / qmax)
        for v, c in zip(x, codes):
            exact = Fraction(float(v)) * qmax / am
            frac = exact - (exact.numerator // exact.denominator)
            if abs(frac - Fraction(1, 2)) < Fraction(1, 100000):
                continue
            want = max(-qmax, min(qmax, _rne_fraction(exact)))
            assert int(c) == want, (v, exact, c)
            checked += 1
    assert checked > 100


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("block", [1, 3, 256, 2048])
def test_roundtrip_bound(bits, block):
    """|x - dequant(quant(x))| <= scale/2, up to fp32 rounding of the
    product and of inv (relative 2^-20 slack), on ragged lengths zero padded to the block."""
    rng = np.random.default_rng(bits * 1000 + block)
    for n in (block * 7 + (block // 3 if block > 2 else 0), 1 + block):
        npad = -(-n // block) * block
        x = np.zeros(npad, np.float32)
        x[:n] = rng.standard_normal(n) * 3
        x[rng.integers(0, n, size=max(1, n // 100))] *= 64
        codes, scales = quant.quantize(x, bits, block)
        xh = quant.dequantize(codes, scales, block)
        err = np.abs(x.astype(np.float64) - xh.astype(np.float64)).reshape(-1, block)
        bound = scales.astype(np.float64)[:, None] / 2 * (1 + 2.0 ** -20) + 1e-45
        assert (err <= bound).all()


@pytest.mark.parametrize("bits", [8, 4])
def test_idempotent_and_sign(bits):
    rng = np.random.default_rng(5)
    x = (rng.standard_normal(256 * 64) * 0.02).astype(np.float32)
    c1, s1 = quant.quantize(x, bits, 256)
    xh = quant.dequantize(c1, s1, 256)
    c2, s2 = quant.quantize(xh, bits, 256)
    assert np.array_equal(c1, c2)
    assert np.array_equal(s1, s2)
    # sign preservation: sign(x_hat) in {0, sign(x)}
    sx, sh = np.sign(x), np.sign(xh)
    assert ((sh == 0) | (sh == sx)).all()


def test_codes_range_and_no_most_negative():
    rng = np.random.default_rng(3)
    x = (rng.standard_normal(256 * 32)).astype(np.float32)
    for bits, qmax in ((8, 127), (4, 7)):
        c, _ = quant.quantize(x, bits, 256)
        assert c.min() >= -qmax and c.max() <= qmax
        # absmax element of each block maps to +-qmax exactly
        cb = c.reshape(-1, 256)
        assert (np.abs(cb).max(axis=1) == qmax).all()


def test_int4_pack_bijection():
    allbytes = np.arange(256, dtype=np.uint8)
    codes = quant.unpack_int4(allbytes)
    assert codes.min() == -8 and codes.max() == 7
    assert np.array_equal(quant.pack_int4(codes), allbytes)
    # explicit nibble order (R4): low nibble = even element
    assert quant.pack_int4(np.array([1, -1], np.int8))[0] == 0xF1
    assert quant.pack_int4(np.array([-7, 7], np.int8))[0] == 0x79


@pytest.mark.parametrize("bits", [8, 4])
def test_lattice_exact(bits):
    """Vectors already on the code lattice (x = c * 2^k with max |c| = qmax) round-trip exactly."""
    qmax = {8: 127, 4: 7}[bits]
    rng = np.random.default_rng(9)
    for k in (-20, -3, 0, 5):
        c = rng.integers(-qmax, qmax + 1, size=64)
        c[7] = -qmax
        x = (c * 2.0 ** k).astype(np.float32)
        codes, scales = quant.quantize(x, bits, 64)
        assert np.array_equal(codes, c.astype(np.int8))
        assert np.array_equal(quant.dequantize(codes, scales, 64), x)


def test_tiny_and_subnormal_blocks():
    """R3: absmax < 2^-100 -> scale 0 and codes 0; just above -> finite scale, no NaN."""
    tiny = np.float32(2.0 ** -100)
    for x in (np.full(8, 1e-40, np.float32), np.full(8, 1.2e-38, np.float32),
              np.full(8, tiny * np.float32(0.75), np.float32)):
        c, s = quant.quantize(x, 8, 8)
        assert s[0] == 0 and not c.any()
    x = np.zeros(8, np.float32)
    x[2] = tiny * np.float32(1.5)
    x[5] = -tiny
    c, s = quant.quantize(x, 8, 8)
    assert s[0] > 0 and np.isfinite(s[0])
    assert c[2] == 127 and c[0] == 0
    assert np.isfinite(quant.dequantize(c, s, 8)).all()
    # FLT_MIN-scale block would overflow qmax/am if the threshold were FLT_MIN:
    x = np.zeros(8, np.float32)
    x[0] = np.float32(1.2e-38)
    c, s = quant.quantize(x, 8, 8)
    assert not np.isnan(quant.dequantize(c, s, 8)).any()


def test_bf16_output_is_rne():
    """O6 bf16 output equals a hand-written RNE of the fp32 bit pattern."""
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(4096) * 0.02).astype(np.float32)
    c, s = quant.quantize(x, 8, 256)
    f32 = quant.dequantize(c, s, 256, out="f32")
    b16 = quant.dequantize(c, s, 256, out="bf16")
    u = f32.view(np.uint32).astype(np.uint64)
    bias = 0x7FFF + ((u >> 16) & 1)
    manual = ((u + bias) >> 16).astype(np.uint16)
    assert np.array_equal(b16.view(np.uint16), manual)
    assert b16.dtype == ml_dtypes.bfloat16


def test_bf16_input_widening_is_exact():
    rng = np.random.default_rng(2)
    xb = (rng.standard_normal(1024)).astype(np.float32).astype(ml_dtypes.bfloat16)
    c1, s1 = quant.quantize(xb, 8, 256)
    c2, s2 = quant.quantize(xb.astype(np.float32), 8, 256)
    assert np.array_equal(c1, c2) and np.array_equal(s1, s2)
