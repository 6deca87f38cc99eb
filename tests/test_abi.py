"""The C-ABI library without a GPU: it loads, exports every symbol include/gact.h declares,
its host-only logic (sizes, status strings, argument validation, the bit allocator) is
right, and device calls fail loudly (GACT_ERR_CUDA) instead of falling back to the CPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import paper_2206_11357_b200 as gact

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gact.h")


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(gact.LIB_PATH):
        subprocess.run(["make", "-j8", "lib"], cwd=ROOT, check=True)
    return gact.lib()


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gact_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert len(names) >= 10
    out = subprocess.run(["nm", "-D", "--defined-only", gact.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gact_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert getattr(L, n) is not None


def test_exports_testing_entry_point(L):
    """include/gact_testing.h (test-only generator access) is exported too."""
    src = open(os.path.join(os.path.dirname(HEADER), "gact_testing.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = sorted(set(re.findall(r"\b(gact_[a-z_0-9]+)\s*\(", src)))
    assert names == ["gact_test_philox_blocks"]
    out = subprocess.run(["nm", "-D", "--defined-only", gact.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "gact_test_philox_blocks" in set(re.findall(r"\bT (gact_\w+)", out))
    assert L.gact_test_philox_blocks(0, 0, 1, 4, None, None) == 1  # GACT_ERR_INVALID_ARG, no launch
    out = ctypes.c_void_p(16)  # never dereferenced: rejected before any launch
    assert L.gact_test_philox_blocks(0, 0, 1, 5, out, None) == 1


def test_no_oracle_linkage():
    """The product library neither links nor references the oracle."""
    out = subprocess.run(["nm", "-D", gact.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "oracle" not in out
    ldd = subprocess.run(["ldd", gact.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in ldd


def test_sizes_and_strings(L):
    assert L.gact_version() >> 16 == 1
    assert gact.num_groups(4096, 256) == 16 and gact.num_groups(4097, 256) == 17
    assert gact.num_groups(0, 256) == 0 and L.gact_num_groups(-1, 256) == -1
    assert gact.packed_words(4096, 2) == 256 and gact.packed_words(5, 1) == 1
    assert gact.packed_words(33, 8) == 9 and L.gact_packed_words(5, 0) == -1
    for s, name in enumerate(["GACT_OK", "GACT_ERR_INVALID_ARG", "GACT_ERR_UNSUPPORTED_BITS",
                              "GACT_ERR_GROUP_SIZE", "GACT_ERR_ALIGNMENT", "GACT_ERR_INFEASIBLE",
                              "GACT_ERR_CUDA"]):
        assert L.gact_status_string(s).decode() == name


A = 0x10000  # a 16-byte-aligned fake device address: validation never dereferences


@pytest.mark.parametrize("args,expect", [
    (dict(bits=3), 2), (dict(bits=0), 2), (dict(bits=16), 2),
    (dict(G=100), 3), (dict(G=16), 3), (dict(G=8192), 3), (dict(G=48), 3), (dict(G=4128), 3),
    (dict(G=0), 3), (dict(G=-32), 3), (dict(G=33), 3),
    (dict(x=A + 8), 4), (dict(packed=A + 4), 4), (dict(mn=A + 2), 4),
    (dict(n=-1), 1), (dict(dtype=3), 1), (dict(x=0), 1),
])
def test_quantize_validation(L, args, expect):
    a = dict(x=A, dtype=1, n=1000, G=256, bits=2, packed=A, mn=A, sc=A)
    a.update(args)
    st = L.gact_quantize_pack(a["x"], a["dtype"], a["n"], a["G"], a["bits"], 1, a["packed"], a["mn"], a["sc"], None)
    assert st == expect


def test_dequantize_validation(L):
    assert L.gact_unpack_dequantize(A, A, A, 10, 256, 3, A, 0, None) == 2
    assert L.gact_unpack_dequantize(A, A, A, 10, 100, 2, A, 0, None) == 3
    assert L.gact_unpack_dequantize(A, A, A, 10, 256, 2, A + 4, 0, None) == 4
    assert L.gact_unpack_dequantize(A, A, A, 10, 256, 2, A, 7, None) == 1
    assert L.gact_group_stats(A, 0, 10, 256, 5, A, A, None) == 2


def test_empty_is_a_no_op(L):
    assert L.gact_quantize_pack(0, 0, 0, 256, 2, 1, 0, 0, 0, None) == 0
    assert L.gact_unpack_dequantize(0, 0, 0, 0, 256, 2, 0, 0, None) == 0
    assert L.gact_quantize_pack_batch(None, 0, 256, None) == 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_device_call_without_gpu_fails_loudly(L):
    st = L.gact_quantize_pack(A, 1, 4096, 256, 2, 1, A, A, A, None)
    assert st == 6  # GACT_ERR_CUDA, never a silent CPU fallback
    with pytest.raises(ValueError):
        gact.quantize_pack(torch.zeros(256, dtype=torch.bfloat16), 2, 1)


def test_staged_validation_and_no_gpu(L):
    """The staged (host-buffer) forms validate before touching CUDA; with valid arguments
    and no GPU they fail with GACT_ERR_CUDA (no CPU fallback)."""
    WS = 0x100000  # 256-byte aligned fake workspace
    MIN = gact.STAGED_MIN_WORKSPACE

    def call(fn, row, G=256, ws=WS, nbytes=MIN, count=1):
        return getattr(L, fn)(gact._desc_array([row]), count, G, ws, nbytes, None)
    ok = (A, A, A, A, 4096, 1, 4, 1)
    for fn in ("gact_quantize_pack_staged", "gact_unpack_dequantize_staged"):
        assert call(fn, ok, G=100) == 3
        assert call(fn, ok[:6] + (3, 1)) == 2
        assert call(fn, (A + 8,) + ok[1:]) == 4
        assert call(fn, ok[:1] + (A + 4,) + ok[2:]) == 4
        assert call(fn, ok[:4] + (-1,) + ok[5:]) == 1
        assert call(fn, ok, ws=0) == 1
        assert call(fn, ok, ws=WS + 16) == 1
        assert call(fn, ok, nbytes=MIN - 1) == 1
        assert call(fn, ok, count=-1) == 1
        # G = 4064 (= 32 x 127) stages in pieces of lcm(4064, 4096) = 520,192 elements: the
        # minimum workspace cannot hold one (~3 MB per slot in the worst case)
        assert call(fn, ok, G=4064) == 1
        if not torch.cuda.is_available():
            assert call(fn, ok) == 6
            assert call(fn, ok, G=96) == 6
            assert call(fn, ok, G=4064, nbytes=3 * (4 << 20)) == 6


# ---------------------------------------------------------------- host allocator parity
def test_allocator_matches_oracle(L, orc):
    rng = np.random.default_rng(3)
    for ladder in ([1, 2, 4, 8], [1, 2, 4, 8, 32], [2, 3, 4, 8], [4]):
        for _ in range(300):
            Lt = int(rng.integers(1, 40))
            D = rng.integers(1, 10**6, size=Lt).astype(np.int64)
            c = 10.0 ** rng.uniform(-6, 6, size=Lt)
            c[rng.random(Lt) < 0.1] = 0.0
            B = int(rng.integers(ladder[0] * D.sum(), ladder[-1] * D.sum() + 1))
            rc, ref = orc.allocate_bits(c, D, ladder, B)
            assert rc == 0
            got = gact.allocate_bits(c, D, B, ladder)
            assert np.array_equal(got, ref)


def test_allocator_ties_and_errors(L, orc):
    c = np.ones(50)
    D = np.full(50, 7, dtype=np.int64)
    for B in range(50 * 7, 8 * 50 * 7 + 1, 97):
        assert np.array_equal(gact.allocate_bits(c, D, B), orc.allocate_bits(c, D, [1, 2, 4, 8], B)[1])
    with pytest.raises(gact.GactError) as e:
        gact.allocate_bits([1.0, 1.0], [10, 10], 19)
    assert e.value.status == 5
    with pytest.raises(gact.GactError):
        gact.allocate_bits([float("nan")], [10], 100)
    with pytest.raises(gact.GactError):
        gact.allocate_bits([1.0], [10], 100, ladder=[2, 2])


def test_variance_factor_matches_the_oracle(L, orc):
    """gact_variance_factor is S(b) = (2^b - 1)^-2 of P:479-480 (S(32) = 0), equal to the
    oracle's S and to the SPEC values S(2) = 1/9, S(4) = 1/225; -1 for invalid bits."""
    for b in list(range(1, 17)) + [32]:
        assert L.gact_variance_factor(b) == orc.S(b)
    assert gact.variance_factor(2) == 1 / 9 and gact.variance_factor(4) == 1 / 225
    for b in (0, 17, 31, 33, -1):
        assert L.gact_variance_factor(b) == -1.0
        with pytest.raises(ValueError):
            gact.variance_factor(b)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks validation on a host without a GPU")
@pytest.mark.parametrize("G", [32, 96, 160, 224, 256, 800, 2080, 4064, 4096])
def test_every_multiple_of_32_is_a_valid_group_size(L, G):
    """include/gact.h: group_size may be any multiple of 32 in [32, 4096] (powers of two take
    the specialised kernels). Validation passes, so the call fails only at the launch
    (GACT_ERR_CUDA, no GPU here), never with GACT_ERR_GROUP_SIZE."""
    assert L.gact_quantize_pack(A, 1, 4096, G, 2, 1, A, A, A, None) == 6
    assert L.gact_unpack_dequantize(A, A, A, 4096, G, 2, A, 1, None) == 6
    assert L.gact_group_stats(A, 1, 4096, G, 2, A, A, None) == 6
