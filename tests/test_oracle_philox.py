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


def _bytes_of_block(orc, seed, block):
    r = orc.philox4x32_10([block & 0xFFFFFFFF, block >> 32, 0, 0], [seed & 0xFFFFFFFF, seed >> 32])
    return [(int(r[w]) >> (8 * b)) & 0xFF for w in range(4) for b in range(4)]  # little-endian bytes


def test_rand8_layout(orc):
    """Element i takes byte 8 (i/256 mod 2) + (i mod 8) of block 32 (i/512) + (i/8 mod 32)
    (R3) -- checked against the block function, which the two tests above pin."""
    seed = 0x0123456789ABCDEF
    for i in [0, 1, 7, 8, 255, 256, 263, 511, 512, 1000, 4095, 2**33 + 5, 2**40 + 300]:
        blk = 32 * (i // 512) + (i // 8) % 32
        byte = 8 * ((i // 256) % 2) + i % 8
        assert orc.rand8(seed, i) == _bytes_of_block(orc, seed, blk)[byte], i


def test_rand8_is_a_bijection_onto_block_bytes():
    """Over any 512-element span the (block, byte) pairs are distinct and cover 32 blocks x 16
    bytes exactly: every random byte of the stream is used once (no two elements share one)."""
    pairs = set()
    base = 7 * 512
    for i in range(base, base + 512):
        pairs.add((32 * (i // 512) + (i // 8) % 32, 8 * ((i // 256) % 2) + i % 8))
    assert len(pairs) == 512
    assert {b for b, _ in pairs} == set(range(32 * 7, 32 * 8))
    assert {j for _, j in pairs} == set(range(16))


def test_rand8_uniform(orc):
    """The bytes look uniform: mean of 16 x 2048 bytes / 256 within 4 sigma of the lattice
    mean 255/512, every byte position within a block with the same mean (no position bias),
    and all 256 values occur with frequencies within 5 sigma of 1/256."""
    seed = 99
    k = np.array([orc.rand8(seed, i) for i in range(16 * 2048)], dtype=np.int64)
    u = k / 256.0
    sigma = np.sqrt((1 / 12) / u.size)
    assert abs(u.mean() - 255 / 512) < 4 * sigma
    pos = np.array([8 * ((i // 256) % 2) + i % 8 for i in range(k.size)])
    for j in range(16):
        assert abs(u[pos == j].mean() - 255 / 512) < 4 * np.sqrt((1 / 12) / (pos == j).sum())
    f = np.bincount(k, minlength=256) / k.size
    assert np.all(np.abs(f - 1 / 256) < 5 * np.sqrt((1 / 256) * (1 - 1 / 256) / k.size))
