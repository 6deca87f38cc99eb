"""Pins of the oracle's packing (R6) and bit allocator (R9, R10).

Packing: hand-worked words (tests/golden/pack_examples.txt); NumPy's packbits (b=1),
the little-endian byte view (b=8) and nibble interleave (b=4) as independent library
layouts; round trips at ragged n; zero padding.

Allocator (eqn:ilp P:471-475, greedy P:534): SPEC.md examples (corrected where SPEC is
infeasible, tests/golden/spec_examples.txt); the exact Lagrangian pin — S is convex along
the ladder, so every greedy iterate is optimal for the bits it uses (Everett 1963): the
greedy value equals a brute-force minimum (itertools, independent of the oracle) at the
greedy's own bit count; monotonicity in B; dominance; scale invariance.
"""
import itertools
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _pack_examples():
    for line in open(os.path.join(GOLD, "pack_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        b, q, w = line.strip().split(";")
        yield int(b), [int(v) for v in q.split(",")], [int(v, 16) for v in w.split(",")]


def test_hand_worked_words(orc):
    n = 0
    for bits, q, words in _pack_examples():
        got = orc.pack(np.array(q, dtype=np.uint8), bits)
        assert got.tolist() == words
        assert orc.unpack(got, len(q), bits).tolist() == q
        n += 1
    assert n == 4


@pytest.mark.parametrize("n", [1, 7, 31, 32, 33, 255, 1000, 4097])
def test_library_layouts(orc, n):
    rng = np.random.default_rng(n)
    q1 = rng.integers(0, 2, n).astype(np.uint8)
    p1 = orc.pack(q1, 1)
    ref1 = np.packbits(q1, bitorder="little")
    assert np.array_equal(p1.view(np.uint8)[: ref1.size], ref1)
    assert not p1.view(np.uint8)[ref1.size:].any()
    q8 = rng.integers(0, 256, n).astype(np.uint8)
    p8 = orc.pack(q8, 8)
    assert np.array_equal(p8.view(np.uint8)[:n], q8) and not p8.view(np.uint8)[n:].any()
    q4 = rng.integers(0, 16, n).astype(np.uint8)
    p4 = orc.pack(q4, 4)
    qq = np.concatenate([q4, np.zeros(n % 2, np.uint8)])
    ref4 = qq[0::2] | (qq[1::2] << 4)
    assert np.array_equal(p4.view(np.uint8)[: ref4.size], ref4)


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_round_trip_and_padding(orc, bits):
    rng = np.random.default_rng(bits)
    for n in [0, 1, 5, 16, 17, 31, 100, 1023]:
        q = rng.integers(0, 1 << bits, n).astype(np.uint8)
        p = orc.pack(q, bits)
        assert p.size == (n * bits + 31) // 32
        assert np.array_equal(orc.unpack(p, n, bits), q)
        if n:
            used = n * bits - 32 * (p.size - 1)
            assert int(p[-1]) >> used == 0 if used < 32 else True


# ----------------------------------------------------------------------------- allocator
def test_S_values(orc):
    assert orc.S(2) == 1 / 9 and orc.S(4) == 1 / 225 and orc.S(1) == 1.0
    assert orc.S(8) == 1 / 255 ** 2 and orc.S(32) == 0.0
    assert orc.predicted_variance([9.0], [2]) == 1.0


@pytest.mark.parametrize("B,expect", [(100, [2, 8]), (80, [2, 2])])
def test_spec_two_slot_example(orc, B, expect):
    rc, bits = orc.allocate_bits([1.0, 100.0], [10, 10], [2, 8], B)
    assert rc == 0 and bits.tolist() == expect
    rc, bbits, _ = orc.allocate_bruteforce([1.0, 100.0], [10, 10], [2, 8], B)
    assert rc == 0 and bbits.tolist() == expect


def test_symmetric_uniform(orc):
    for ladder in ([1, 2, 4, 8], [2, 3, 4, 8]):
        rc, bits = orc.allocate_bits([3.0] * 6, [100] * 6, ladder, 4 * 600)
        assert rc == 0 and bits.tolist() == [4] * 6


def test_infeasible_and_invalid(orc):
    assert orc.allocate_bits([1.0, 1.0], [10, 10], [2, 4], 39)[0] == orc.EINFEASIBLE
    assert orc.allocate_bits([1.0, 1.0], [10, 10], [2, 4], 40)[0] == 0
    assert orc.allocate_bits([float("nan")], [1], [1, 2], 10)[0] == orc.EINVAL
    assert orc.allocate_bits([-1.0], [1], [1, 2], 10)[0] == orc.EINVAL
    assert orc.allocate_bits([1.0], [0], [1, 2], 10)[0] == orc.EINVAL
    assert orc.allocate_bits([1.0], [1], [2, 1], 10)[0] == orc.EINVAL


def test_pinned_infinite_sensitivity(orc):
    """c = +inf is lowered only after every finite tensor is at the bottom (SPEC S:348
    pins such a slot to 32 bits when the budget permits)."""
    rc, bits = orc.allocate_bits([1.0, np.inf, 2.0], [100, 10, 100], [2, 4, 8, 32], 4 * 210 + 28 * 10)
    assert rc == 0 and bits[1] == 32


def _brute(c, D, ladder, B):
    best, arg = None, None
    for s in itertools.product(ladder, repeat=len(c)):
        if sum(b * d for b, d in zip(s, D)) <= B:
            v = sum(ci * (0.0 if b == 32 else 1.0 / ((2 ** b - 1) ** 2)) for ci, b in zip(c, s))
            if best is None or v < best:
                best, arg = v, s
    return best, arg


def _instances(rng, count, ladder):
    for _ in range(count):
        L = int(rng.integers(1, 7))
        D = rng.choice([1, 2, 3, 5, 8, 13, 64, 100], size=L).astype(np.int64)
        c = 10.0 ** rng.uniform(-4, 4, size=L)
        lo, hi = ladder[0] * D.sum(), ladder[-1] * D.sum()
        B = int(rng.integers(lo, hi + 1))
        yield c, D, B


@pytest.mark.parametrize("ladder", [[1, 2, 4, 8], [1, 2, 4, 8, 32], [2, 3, 4, 8]])
def test_greedy_is_lagrangian_optimal(orc, ladder):
    rng = np.random.default_rng(len(ladder) * 31 + ladder[0])
    gaps = []
    for c, D, B in _instances(rng, 400, ladder):
        rc, bits = orc.allocate_bits(c, D, ladder, B)
        assert rc == 0
        used = int((bits.astype(np.int64) * D).sum())
        assert used <= B
        v = orc.predicted_variance(c, bits)
        vb, _ = _brute(list(c), list(D), ladder, used)
        assert v <= vb * (1 + 1e-12) + 1e-300
        # the oracle's brute force agrees with itertools at the nominal budget
        rcb, _, vb_nom = orc.allocate_bruteforce(c, D, ladder, B)
        assert rcb == 0 and abs(vb_nom - _brute(list(c), list(D), ladder, B)[0]) <= 1e-12 * vb_nom
        gaps.append(v / vb_nom if vb_nom > 0 else 1.0)
    # nominal-budget gap is a statistic, not a pin (SPEC S:579 is not robust)
    assert np.median(gaps) <= 1.0 + 1e-9


def test_monotone_dominance_scale(orc):
    rng = np.random.default_rng(77)
    ladder = [1, 2, 4, 8]
    for _ in range(100):
        L = int(rng.integers(2, 12))
        D = rng.integers(1, 1000, size=L)
        c = 10.0 ** rng.uniform(-3, 3, size=L)
        Bs = sorted(rng.integers(D.sum(), 8 * D.sum() + 1, size=5))
        vals = [orc.predicted_variance(c, orc.allocate_bits(c, D, ladder, int(B))[1]) for B in Bs]
        assert all(vals[i + 1] <= vals[i] for i in range(len(vals) - 1))
        B = int(Bs[2])
        b1 = orc.allocate_bits(c, D, ladder, B)[1]
        b2 = orc.allocate_bits(c * 2.0 ** 7, D, ladder, B)[1]
        assert np.array_equal(b1, b2)
    # dominance: equal D, c_i > c_j  =>  b_i >= b_j
    for _ in range(100):
        L = 8
        D = np.full(L, 50)
        c = 10.0 ** rng.uniform(-3, 3, size=L)
        bits = orc.allocate_bits(c, D, ladder, int(rng.integers(L * 50, 8 * L * 50)))[1]
        order = np.argsort(c)
        assert np.all(np.diff(bits[order]) >= 0)


# ------------------------------------------------------------------ Alg. 1 reduction
def test_sq_diff_sum_exact_small(orc):
    """||a - b||^2 against exact rational arithmetic (Fractions), all dtypes."""
    from fractions import Fraction
    import torch
    rng = np.random.default_rng(8)
    for tag in (0, 1, 2):
        for n in (0, 1, 7, 100, 1000):
            a = rng.standard_normal(n).astype(np.float32) * 3
            b = rng.standard_normal(n).astype(np.float32)
            if tag == 1:
                a = torch.from_numpy(a).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
                b = torch.from_numpy(b).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
                av = (a.astype(np.uint32) << 16).view(np.float32)
                bv = (b.astype(np.uint32) << 16).view(np.float32)
            elif tag == 2:
                a, b = a.astype(np.float16).view(np.uint16), b.astype(np.float16).view(np.uint16)
                av, bv = a.view(np.float16).astype(np.float32), b.view(np.float16).astype(np.float32)
            else:
                av, bv = a, b
            exact = sum((Fraction(float(x)) - Fraction(float(y))) ** 2 for x, y in zip(av, bv))
            got = orc.sq_diff_sum(a, b, tag)
            assert abs(Fraction(got) - exact) <= Fraction(exact) * Fraction(1, 1 << 52) + Fraction(0)
