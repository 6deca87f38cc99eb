"""Pins of the oracle's Philox4x32-10 lanes (R3) to things other than itself:
the published Random123 known-answer vectors and ATen's independent implementation."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat_rows():
    rows = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(t, 16) for t in line.split()]
        rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


def test_kat_vectors(orc):
    rows = _kat_rows()
    assert len(rows) == 3
    for ctr, key, expect in rows:
        got = orc.philox4x32_10(ctr, key)
        assert [int(v) for v in got] == expect


_ATEN_PROG = r"""
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
// Prints, for each (seed, subsequence, offset) on stdin, the first 4 outputs of
// at::philox_engine: the Philox4x32-10 block of counter (offset, subsequence), key seed.
int main() {
  unsigned long long seed, subseq, offset;
  while (std::scanf("%llu %llu %llu", &seed, &subseq, &offset) == 3) {
    at::philox_engine e(seed, subseq, offset);
    uint32_t a = e(), b = e(), c = e(), d = e();
    std::printf("%u %u %u %u\n", a, b, c, d);
  }
  return 0;
}
"""


@pytest.fixture(scope="module")
def aten_philox():
    import torch
    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    d = tempfile.mkdtemp()
    src, exe = os.path.join(d, "p.cpp"), os.path.join(d, "p")
    open(src, "w").write(_ATEN_PROG)
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", inc, src, "-o", exe],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cannot compile against ATen's PhiloxRNGEngine.h: " + r.stderr[-300:])
    return exe


def test_matches_aten_philox_engine(orc, aten_philox):
    rng = np.random.default_rng(11)
    cases = [(0, 0, 0), (2**64 - 1, 2**64 - 1, 2**64 - 1)]
    cases += [tuple(int(v) for v in rng.integers(0, 2**63, size=3, dtype=np.uint64)) for _ in range(300)]
    inp = "\n".join(f"{s} {q} {o}" for s, q, o in cases) + "\n"
    out = subprocess.run([aten_philox], input=inp, capture_output=True, text=True, check=True).stdout
    lines = out.strip().split("\n")
    assert len(lines) == len(cases)
    for (seed, subseq, offset), line in zip(cases, lines):
        ctr = [offset & 0xFFFFFFFF, offset >> 32, subseq & 0xFFFFFFFF, subseq >> 32]
        key = [seed & 0xFFFFFFFF, seed >> 32]
        assert [int(v) for v in orc.philox4x32_10(ctr, key)] == [int(t) for t in line.split()]


def test_lane16_layout(orc):
    """Element i takes 16-bit lane i&7 of block i>>3 (low half first) — checked against
    the block function, which the two tests above pin."""
    seed = 0x0123456789ABCDEF
    for i in [0, 1, 2, 7, 8, 15, 1000, 2**33 + 5]:
        blk = i >> 3
        r = orc.philox4x32_10([blk & 0xFFFFFFFF, blk >> 32, 0, 0], [seed & 0xFFFFFFFF, seed >> 32])
        j = i & 7
        w = int(r[j >> 1])
        expect = (w >> 16) if (j & 1) else (w & 0xFFFF)
        assert orc.lane16(seed, i) == expect


def test_lanes_uniform(orc):
    """16-bit lanes look uniform: mean of 8*4096 lanes / 2^16 within 4 sigma of 1/2, and
    every lane position within a block has the same mean (no position bias)."""
    seed = 99
    k = np.array([orc.lane16(seed, i) for i in range(8 * 4096)], dtype=np.float64) / 65536.0
    sigma = np.sqrt(1 / 12 / k.size)
    assert abs(k.mean() - 0.5) < 4 * sigma
    per_pos = k.reshape(-1, 8).mean(axis=0)
    assert np.all(np.abs(per_pos - 0.5) < 4 * np.sqrt(1 / 12 / 4096))
