"""Pins of the oracle's quantizer (R1, R2, R4, R5, R7) to what the paper and
the mathematics fix, never to the oracle itself:

  * SPEC.md's worked group-statistics examples (tests/golden/spec_examples.txt);
  * group statistics recomputed with NumPy's min / max / binary32 division and an exact
    rational round-toward-zero for inv (Fractions);
  * every code recomputed as the exact real floor(d * inv + (2k+1) 2^-9) with Fractions
    (d = x - mn in binary32; product and sum exact);
  * the exact round trip on b-bit grids (P:497 idempotence, B3) for every seed;
  * Monte Carlo unbiasedness E[Q(x)] = x, per-element variance p(1-p) scale^2
    and the paper's bound 1/4 range^2 S(b) (B2), and uncorrelated elements
    (B1) — including pairs that share one Philox word.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")
LADDER = [1, 2, 4, 8]


def _golden(name):
    for line in open(GOLDEN):
        if line.startswith(name + " "):
            return [t.strip() for t in line.split(";")]
    raise KeyError(name)


def _kv(s):
    return {k: v for k, v in (p.split("=") for p in s.split())}


@pytest.mark.parametrize("name", ["group_minmax_1", "group_minmax_2", "group_minmax_3"])
def test_spec_group_minmax_examples(orc, name):
    _, inp, exp = _golden(name)
    a, e = _kv(inp), _kv(exp)
    x = np.array([float(v) for v in a["x"].split(",")], dtype=np.float32)
    mn, sc = orc.group_stats(x, orc.F32, int(a["G"]), 1)  # b=1: scale = range
    assert mn.tolist() == [float(v) for v in e["mins"].split(",")]
    assert sc.tolist() == [float(v) for v in e["ranges"].split(",")]


def _rz_div(a: float, b: float) -> np.float32:
    """Largest binary32 <= a/b for a, b > 0, by exact rational comparison."""
    q = Fraction(a) / Fraction(b)
    f = np.float32(float(q)) if float(q) < 3.4e38 else np.float32(3.4028235e38)
    while Fraction(float(f)) > q:
        f = np.nextafter(f, np.float32(0))
    while True:
        up = np.nextafter(f, np.float32(np.inf))
        if np.isinf(up) or Fraction(float(up)) > q:
            return f
        f = up


def _host_values(tag, x):
    if tag == 1:  # bf16 patterns -> f32 by definition (upper half)
        return (x.astype(np.uint32) << 16).view(np.float32)
    if tag == 2:
        return x.view(np.float16).astype(np.float32)
    return x


def _rand_input(rng, n, tag):
    v = rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3)
    v[rng.integers(0, n, size=max(1, n // 50))] = -0.0
    if tag == 0:
        return v.astype(np.float32)
    if tag == 2:
        return v.astype(np.float16).view(np.uint16)
    import torch
    return torch.from_numpy(v.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def _ref_params(vals, bits):
    """(mn, scale, inv) of one group from NumPy + exact rationals."""
    L = np.float32((1 << bits) - 1)
    mn = np.float32(np.min(vals)) + np.float32(0.0)
    mx = np.float32(np.max(vals)) + np.float32(0.0)
    rng_ = np.float32(mx - mn)
    scale = np.float32(rng_ / L)
    inv = np.float32(0.0) if rng_ == 0 else _rz_div(float(L), float(rng_))
    return mn, scale, inv


@pytest.mark.parametrize("tag", [0, 1, 2])
@pytest.mark.parametrize("G", [2, 32, 100, 256])
def test_group_stats_vs_numpy(orc, tag, G):
    rng = np.random.default_rng(10 + tag * 7 + G)
    for bits in LADDER:
        n = int(rng.integers(1, 5 * G + 3))
        x = _rand_input(rng, n, tag)
        vals = _host_values(tag, x)
        mn, sc = orc.group_stats(x, tag, G, bits)
        for g in range(len(mn)):
            rmn, rsc, _ = _ref_params(vals[g * G:(g + 1) * G], bits)
            assert mn[g].view(np.uint32) == rmn.view(np.uint32)
            assert sc[g].view(np.uint32) == rsc.view(np.uint32)


@pytest.mark.parametrize("tag", [0, 1, 2])
def test_codes_are_exact_floor_of_t_plus_u(orc, tag):
    rng = np.random.default_rng(20 + tag)
    G, seed = 64, 0xC0FFEE + tag
    for bits in LADDER:
        n = 3 * G + 17
        x = _rand_input(rng, n, tag)
        vals = _host_values(tag, x)
        q, mn, sc = orc.quantize_codes(x, tag, G, bits, seed)
        for g in range(len(mn)):
            rmn, rsc, inv = _ref_params(vals[g * G:(g + 1) * G], bits)
            for i in range(g * G, min(n, (g + 1) * G)):
                d = np.float32(vals[i] - rmn)
                k = orc.rand8(seed, i)
                exact = math.floor(Fraction(float(d)) * Fraction(float(inv)) + Fraction(2 * k + 1, 1 << 9))
                assert q[i] == exact, (bits, i)


def test_t_within_0_L_on_adversarial_ranges(orc):
    """R2: with inv = RZ(L/range) the exact transform d * inv never leaves [0, L] and codes
    never exceed L (the oracle returns EINVARIANT otherwise); ranges from subnormal to 1e38."""
    rng = np.random.default_rng(5)
    for scale in [1e-44, 1e-40, 1e-30, 1e-3, 1.0, 1e10, 1e30, 1e38]:
        for bits in LADDER:
            x = (rng.uniform(-1, 1, 4096) * scale).astype(np.float32)
            q, mn, sc = orc.quantize_codes(x, 0, 256, bits, 77)
            assert q.max() <= (1 << bits) - 1
            assert np.all(np.isfinite(sc))


@pytest.mark.parametrize("bits", LADDER)
def test_exact_grid_round_trip_every_seed(orc, bits):
    """On a b-bit grid (x = m0 + k 2^e, ends present) range = L 2^e, scale = 2^e and
    inv = 2^-e are exact, so t = k, q = k for every seed and decoding returns x bit-exactly
    (idempotence B3)."""
    rng = np.random.default_rng(bits)
    G = 256
    for trial in range(20):
        x = np.concatenate([synth.exact_grid_group(G, bits, rng) for _ in range(4)])
        for seed in [0, 1, 2**63 + trial, trial * 7919]:
            packed, mn, sc = orc.quantize_pack(x, orc.F32, G, bits, seed)
            y = orc.unpack_dequantize(packed, mn, sc, x.size, G, bits, orc.F32)
            assert np.array_equal(y, x.view(np.uint32))


def test_spec_endpoints_and_constant(orc):
    # x=[0,1], b=1, G=2 -> deterministic, decodes exactly
    x = np.array([0.0, 1.0], dtype=np.float32)
    for seed in range(50):
        p, mn, sc = orc.quantize_pack(x, orc.F32, 2, 1, seed)
        assert orc.unpack(p, 2, 1).tolist() == [0, 1]
    # constant group decodes exactly for every b
    x = np.full(300, 5.0, dtype=np.float32)
    for bits in LADDER:
        p, mn, sc = orc.quantize_pack(x, orc.F32, 256, bits, 3)
        y = orc.unpack_dequantize(p, mn, sc, 300, 256, bits, orc.F32)
        assert np.array_equal(y.view(np.float32), x)
        assert sc.tolist() == [0.0, 0.0]


def test_spec_bernoulli_frequency(orc):
    """x = 0.3 in a group with min 0, range 1, b = 1: decodes to 1 with frequency
    0.3 +- 0.014 over 10^4 draws."""
    x = np.array([0.0, 0.3, 1.0], dtype=np.float32)
    ups = 0
    for seed in range(10_000):
        q, _, _ = orc.quantize_codes(x, orc.F32, 3, 1, seed)
        ups += int(q[1])
    assert abs(ups / 10_000 - 0.3) <= 0.014


def _mc(orc, x, G, bits, seeds):
    qs = []
    for s in seeds:
        q, mn, sc = orc.quantize_codes(x, orc.F32, G, bits, s)
        qs.append(q.astype(np.float64))
    return np.array(qs), mn.astype(np.float64), sc.astype(np.float64)


@pytest.mark.parametrize("bits", LADDER)
def test_unbiased_variance_bound_uncorrelated(orc, bits):
    """Monte Carlo over 20000 seeds on 64 elements (2 groups of 32):
    E[q] = frac-rounded t within 4 sigma + 2^-9 (E_Q[Q(x)] = x up to the 8-bit lattice,
    R4), E[y] = x within
    the same bound scaled by `scale` plus binary32 transform rounding;
    Var[q] = p(1-p) within 25% (and never above 1/4: B2, Var[y] <= 1/4 range^2 S(b));
    pairwise correlations of neighbours (same Philox word) ~ 0 (B1)."""
    rng = np.random.default_rng(100 + bits)
    G, n, N = 32, 64, 20_000
    x = rng.standard_normal(n).astype(np.float32)
    qs, mn, sc = _mc(orc, x, G, bits, range(1000 * bits, 1000 * bits + N))
    L = (1 << bits) - 1
    for g in range(2):
        vals = x[g * G:(g + 1) * G]
        rmn, rsc, inv = _ref_params(vals, bits)
        t = np.array([float(np.float32(np.float32(v - rmn) * inv)) for v in vals])
        p = t - np.floor(t)
        Eq = qs[:, g * G:(g + 1) * G].mean(axis=0)
        sig = np.sqrt(p * (1 - p) / N)
        assert np.all(np.abs(Eq - t) <= 4 * sig + 2.0 ** -9 + 1e-12)
        # E[y] = x (paper's unbiasedness), y = mn + q scale; transform rounding <= 4 ulp(L)
        Ey = float(rmn) + Eq * float(rsc)
        tol = (4 * sig + 2.0 ** -9) * float(rsc) + 8 * np.spacing(np.float32(np.abs(vals).max() + 1))
        assert np.all(np.abs(Ey - vals) <= tol)
        var = qs[:, g * G:(g + 1) * G].var(axis=0)
        m = p * (1 - p) > 0.02
        assert np.all(np.abs(var[m] - (p * (1 - p))[m]) <= 0.25 * (p * (1 - p))[m])
        # B2 bound: Var[y] = scale^2 Var[q] <= 1/4 range^2 S(b) = scale^2 / 4 (+ MC noise)
        assert np.all(var <= 0.25 * (1 + 5 / np.sqrt(N)))
        assert L * float(rsc) <= float(np.max(vals) - np.min(vals)) * (1 + 1e-6)
    # B1: neighbours (i, i+1) share a Philox word; (i, i+8) share a counter position
    qc = qs - qs.mean(axis=0)
    sd = qs.std(axis=0)
    for lag in (1, 2, 8):
        for i in range(0, n - lag):
            if sd[i] > 0.1 and sd[i + lag] > 0.1:
                r = (qc[:, i] * qc[:, i + lag]).mean() / (sd[i] * sd[i + lag])
                assert abs(r) < 4.5 / np.sqrt(N), (lag, i, r)


def test_requantize_is_near_idempotent(orc):
    """B3 off the exact grid: re-quantizing a decoded tensor with a fresh seed
    reproduces its codes except where binary32 rounding moved a decoded value across a
    code by less than one step (|q' - q| <= 1, rare)."""
    rng = np.random.default_rng(9)
    for bits in LADDER:
        x = rng.standard_normal(256 * 40).astype(np.float32)
        p, mn, sc = orc.quantize_pack(x, orc.F32, 256, bits, 1)
        y = orc.unpack_dequantize(p, mn, sc, x.size, 256, bits, orc.F32).view(np.float32)
        q1 = orc.unpack(p, x.size, bits).astype(int)
        p2, _, _ = orc.quantize_pack(y, orc.F32, 256, bits, 2)
        q2 = orc.unpack(p2, x.size, bits).astype(int)
        assert np.abs(q2 - q1).max() <= 1
        assert np.mean(q2 != q1) < 2e-3


def test_tiny_and_subnormal_ranges(orc):
    """Degenerate groups: range 0 (t = 0, q = 0, y = mn), subnormal ranges (no inf/NaN,
    decode error <= range)."""
    rng = np.random.default_rng(4)
    for bits in LADDER:
        base = np.float32(rng.standard_normal())
        x = np.full(512, base, dtype=np.float32)
        x[256:] = (rng.integers(0, 4, 256) * 2.0 ** -149).astype(np.float32)
        p, mn, sc = orc.quantize_pack(x, orc.F32, 256, bits, 5)
        y = orc.unpack_dequantize(p, mn, sc, 512, 256, bits, orc.F32).view(np.float32)
        assert np.array_equal(y[:256], x[:256])
        assert np.all(np.isfinite(y))
        assert np.all(np.abs(y[256:] - x[256:]) <= 3 * 2.0 ** -149)


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_threshold_ties_closed_form(orc, bits):
    """T + u exactly on an integer N (q = N) and one fp32 step below / above it (q = N - 1 /
    N): the closed form of q = floor(T + (2k+1) 2^-9) at its discontinuities (include/gact.h;
    DESIGN.md R4, R5). Inputs from tests/tie_cases.py (mn = 0, inv = 1, so T = x exactly)."""
    import tie_cases
    seed = 0x7E5 + bits
    x, want = tie_cases.tie_groups(6, 256, bits, seed, orc.rand8, np.random.default_rng(bits))
    q, mn, sc = orc.quantize_codes(x, orc.F32, 256, bits, seed)
    assert np.all(mn == 0.0) and np.all(sc == 1.0)
    assert np.array_equal(q.astype(np.int64), want)
    # the three cases all occur, for every b
    ties = x[2:] != np.round(x[2:])
    assert ties.sum() > 100
