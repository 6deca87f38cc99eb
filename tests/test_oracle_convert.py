"""Pins of the oracle's dtype handling against NumPy / torch conversions (independent
library routines): widening of every bf16 and fp16 bit pattern, and round-to-nearest-even
into fp32 / bf16 / fp16 (R7)."""
import numpy as np
from fractions import Fraction
import torch


def _finite_mask16(bits16, tag):
    e = (bits16 >> 10) & 0x1F if tag == 2 else (bits16 >> 7) & 0xFF
    return e != (0x1F if tag == 2 else 0xFF)


def test_widen_all_bf16_patterns(orc):
    pats = np.arange(65536, dtype=np.uint16)
    ref = torch.from_numpy(pats.view(np.int16)).view(torch.bfloat16).float().numpy()
    got = orc.widen(pats, orc.BF16)
    fin = _finite_mask16(pats.astype(np.uint32), 1)
    assert np.array_equal(got[fin].view(np.uint32), ref[fin].view(np.uint32))
    assert np.array_equal(np.isnan(got), np.isnan(ref))


def test_widen_all_f16_patterns(orc):
    pats = np.arange(65536, dtype=np.uint16)
    ref = pats.view(np.float16).astype(np.float32)
    got = orc.widen(pats, orc.F16)
    fin = _finite_mask16(pats.astype(np.uint32), 2)
    assert np.array_equal(got[fin].view(np.uint32), ref[fin].view(np.uint32))
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    assert np.array_equal(np.isinf(got), np.isinf(ref))


def _test_values(rng):
    v = list(rng.standard_normal(3000) * 10.0 ** rng.uniform(-8, 8, 3000))
    v += list(rng.uniform(-1, 1, 500) * 2.0 ** -130)  # fp32 subnormal range
    v += list(rng.uniform(-1, 1, 500) * 2.0 ** -20)   # fp16 subnormal range
    v += [0.0, -0.0, 1.0, -1.0, 65504.0, 65519.99, 65520.0, 3.4028234663852886e38,
          2.0 ** -149, 2.0 ** -150, 3 * 2.0 ** -151, 2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26]
    # exact ties: midpoints between consecutive fp32 / fp16 values
    for _ in range(200):
        f = np.float32(rng.standard_normal())
        nxt = np.nextafter(f, np.float32(np.inf))
        v.append((float(f) + float(nxt)) / 2.0)
        h = np.float16(rng.standard_normal())
        nh = np.nextafter(h, np.float16(np.inf))
        v.append((float(h) + float(nh)) / 2.0)
    return np.array(v, dtype=np.float64)


def test_round_to_f32_matches_numpy(orc):
    vals = _test_values(np.random.default_rng(1))
    ref = vals.astype(np.float32).view(np.uint32)
    got = np.array([orc.round_to_dtype(v, orc.F32) for v in vals], dtype=np.uint32)
    assert np.array_equal(got, ref)


def test_round_to_f16_matches_numpy(orc):
    vals = _test_values(np.random.default_rng(2))
    ref = vals.astype(np.float16).view(np.uint16)
    got = np.array([orc.round_to_dtype(v, orc.F16) for v in vals], dtype=np.uint16)
    assert np.array_equal(got, ref)


def test_round_to_bf16_matches_torch(orc):
    """Values exactly representable in fp32 (so torch's fp32->bf16 RNE is the single
    rounding), including every tie halfway between two bf16 values."""
    rng = np.random.default_rng(3)
    f = (rng.standard_normal(4000) * 10.0 ** rng.uniform(-30, 30, 4000)).astype(np.float32)
    ties = (rng.integers(0, 2**16, 500).astype(np.uint32) << 16) | 0x8000  # exact midpoints
    ties = ties[((ties >> 23) & 0xFF) != 0xFF].view(np.float32)
    f = np.concatenate([f, ties, np.array([0.0, -0.0, 1e-40, -3e-39], dtype=np.float32)])
    ref = torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = np.array([orc.round_to_dtype(float(v), orc.BF16) for v in f], dtype=np.uint16)
    assert np.array_equal(got, ref)


def _round_fraction_f32(F):
    """Nearest binary32 to the exact rational F, ties to even (independent of the oracle:
    candidates from NumPy's neighbours, chosen by exact Fraction distances)."""
    import numpy as np
    c = np.float32(float(F))
    cands = {np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))}
    best = sorted(cands, key=lambda v: (abs(Fraction(float(v)) - F), int(np.array(v).view(np.uint32)) & 1))
    return np.array(best[0], dtype=np.float32).view(np.uint32)


def test_dequantize_rounds_the_exact_value_once(orc):
    """R7: y = mn + q * scale rounded ONCE into the output dtype. Pins: (i) a case where
    rounding through binary64 first is wrong -- mn = 1, q = 205, scale = 5237765 * 2^-54, so
    q * scale = (2^30 + 1) 2^-54 = 2^-24 + 2^-54 and the exact value lies just above the
    binary32 tie 1 + 2^-24 (binary64 would round it onto the tie, then ties-to-even to 1):
    the answer is 1 + 2^-23; (ii) 3000 random (mn, scale, q) with large exponent gaps against
    an exact rational rounding."""
    import numpy as np
    mn = np.array([1.0], dtype=np.float32)
    sc = np.array([5237765 * 2.0 ** -54], dtype=np.float32)
    assert float(sc[0]) == 5237765 * 2.0 ** -54
    packed = orc.pack(np.array([205], dtype=np.uint8), 8)
    y = orc.unpack_dequantize(packed, mn, sc, 1, 256, 8, orc.F32)
    assert int(y[0]) == 0x3F800001
    rng = np.random.default_rng(3)
    n = 3000
    mnv = (rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, n)).astype(np.float32)
    scv = (np.abs(rng.standard_normal(n)) * np.abs(mnv) * 2.0 ** -rng.integers(8, 40, n)).astype(np.float32)
    q = rng.integers(0, 256, n).astype(np.uint8)
    ys = orc.unpack_dequantize(orc.pack(q, 8), mnv, scv, n, 1, 8, orc.F32)
    for i in range(n):
        F = Fraction(float(mnv[i])) + int(q[i]) * Fraction(float(scv[i]))
        assert int(ys[i]) == int(_round_fraction_f32(F)), i
