"""Python view of the CPU oracle (oracle/gact_oracle.c) via ctypes + NumPy.

TEST INFRASTRUCTURE ONLY. Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this module. The product package
(``paper_2206_11357_b200``) never imports it and must fail loudly without its CUDA library.

Every function mirrors one C function of gact_oracle.c; see that file for the paper
passages (P:n = /root/reference/PAPER.md line n) and DESIGN.md §3 for the readings.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

F32, BF16, F16 = 0, 1, 2
DTYPE_TAG = {np.dtype(np.float32): F32, np.dtype(np.float16): F16}
OK, EINVAL, EINFEASIBLE, EINVARIANT = 0, 1, 5, 99


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no fast-math, no FMA contraction)."""
    src = os.path.join(_HERE, "gact_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-B" if force else "-s", "oracle"], cwd=_ROOT, check=True)
    return _LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, u64, u32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32
        sig = {
            "oracle_philox4x32_10": (None, [P, P, P]),
            "oracle_rand8": (u32, [u64, u64]),
            "oracle_widen": (ctypes.c_float, [P, i32, i64]),
            "oracle_round_to_dtype": (u32, [ctypes.c_double, i32]),
            "oracle_group_stats": (i32, [P, i32, i64, i32, i32, i64, i64, P, P]),
            "oracle_quantize_codes": (i32, [P, i32, i64, i32, i32, u64, i64, i64, P, P, P]),
            "oracle_pack": (i32, [P, i64, i32, P]),
            "oracle_unpack": (i32, [P, i64, i32, P]),
            "oracle_quantize_pack": (i32, [P, i32, i64, i32, i32, u64, P, P, P]),
            "oracle_dequantize_f64": (i32, [P, P, P, i64, i32, i32, P]),
            "oracle_unpack_dequantize": (i32, [P, P, P, i64, i32, i32, P, i32]),
            "oracle_S": (ctypes.c_double, [i32]),
            "oracle_predicted_variance": (ctypes.c_double, [P, P, i32]),
            "oracle_allocate_bits": (i32, [P, P, i32, P, i32, u64, P]),
            "oracle_allocate_bruteforce": (i32, [P, P, i32, P, i32, u64, P, P]),
            "oracle_sq_diff_sum": (ctypes.c_double, [P, P, i32, i64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


class OracleError(RuntimeError):
    pass


def _check(rc: int, what: str) -> None:
    if rc != OK:
        raise OracleError(f"{what}: oracle returned {rc}")


def dtype_tag(x) -> int:
    """Tag of a host array. bfloat16 data is carried as a uint16 array of bit patterns
    together with tag=BF16 (NumPy has no bfloat16)."""
    return DTYPE_TAG[np.dtype(x.dtype)]


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def rand8(seed: int, i: int) -> int:
    """k_i in [0, 256): the random byte of element i (R3)."""
    return int(lib().oracle_rand8(seed, i))


def widen(x: np.ndarray, tag: int) -> np.ndarray:
    x = np.ascontiguousarray(x)
    f = lib().oracle_widen
    return np.array([f(_ptr(x), tag, i) for i in range(x.size)], dtype=np.float32)


def round_to_dtype(v: float, tag: int) -> int:
    return int(lib().oracle_round_to_dtype(float(v), tag))


def num_groups(n: int, G: int) -> int:
    return (n + G - 1) // G


def packed_words(n: int, bits: int) -> int:
    return (n * bits + 31) // 32


def group_stats(x: np.ndarray, tag: int, G: int, bits: int, g0: int = 0, g1: int | None = None):
    x = np.ascontiguousarray(x).reshape(-1)
    n = x.size
    g1 = num_groups(n, G) if g1 is None else g1
    mn = np.zeros(max(g1 - g0, 0), dtype=np.float32)
    sc = np.zeros_like(mn)
    _check(lib().oracle_group_stats(_ptr(x), tag, n, G, bits, g0, g1, _ptr(mn), _ptr(sc)),
           "group_stats")
    return mn, sc


def quantize_codes(x: np.ndarray, tag: int, G: int, bits: int, seed: int,
                   g0: int = 0, g1: int | None = None):
    """Codes q (uint8, one per element) of groups [g0, g1) plus their mn / scale."""
    x = np.ascontiguousarray(x).reshape(-1)
    n = x.size
    g1 = num_groups(n, G) if g1 is None else g1
    count = max(min(g1 * G, n) - g0 * G, 0)
    q = np.zeros(max(count, 1), dtype=np.uint8)
    mn = np.zeros(max(g1 - g0, 1), dtype=np.float32)
    sc = np.zeros_like(mn)
    _check(lib().oracle_quantize_codes(_ptr(x), tag, n, G, bits, seed, g0, g1, _ptr(q),
                                       _ptr(mn), _ptr(sc)), "quantize_codes")
    return q[:count], mn[:g1 - g0], sc[:g1 - g0]


def pack(q: np.ndarray, bits: int) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.uint8)
    out = np.zeros(max(packed_words(q.size, bits), 1), dtype=np.uint32)
    _check(lib().oracle_pack(_ptr(q), q.size, bits, _ptr(out)), "pack")
    return out[:packed_words(q.size, bits)]


def unpack(packed: np.ndarray, n: int, bits: int) -> np.ndarray:
    p = np.ascontiguousarray(packed, dtype=np.uint32)
    q = np.zeros(max(n, 1), dtype=np.uint8)
    _check(lib().oracle_unpack(_ptr(p), n, bits, _ptr(q)), "unpack")
    return q[:n]


def quantize_pack(x: np.ndarray, tag: int, G: int, bits: int, seed: int):
    """(packed uint32[ceil(n b/32)], group_min f32[ng], group_scale f32[ng])."""
    x = np.ascontiguousarray(x).reshape(-1)
    n = x.size
    ng = num_groups(n, G)
    packed = np.zeros(max(packed_words(n, bits), 1), dtype=np.uint32)
    mn = np.zeros(max(ng, 1), dtype=np.float32)
    sc = np.zeros_like(mn)
    _check(lib().oracle_quantize_pack(_ptr(x), tag, n, G, bits, seed, _ptr(packed), _ptr(mn),
                                      _ptr(sc)), "quantize_pack")
    return packed[:packed_words(n, bits)], mn[:ng], sc[:ng]


def dequantize_f64(packed, mn, sc, n: int, G: int, bits: int) -> np.ndarray:
    p = np.ascontiguousarray(packed, dtype=np.uint32)
    m = np.ascontiguousarray(mn, dtype=np.float32)
    s = np.ascontiguousarray(sc, dtype=np.float32)
    y = np.zeros(max(n, 1), dtype=np.float64)
    _check(lib().oracle_dequantize_f64(_ptr(p), _ptr(m), _ptr(s), n, G, bits, _ptr(y)),
           "dequantize_f64")
    return y[:n]


def unpack_dequantize(packed, mn, sc, n: int, G: int, bits: int, y_tag: int) -> np.ndarray:
    """Rounded output as raw bit patterns: uint32 for F32, uint16 for BF16 / F16."""
    p = np.ascontiguousarray(packed, dtype=np.uint32)
    m = np.ascontiguousarray(mn, dtype=np.float32)
    s = np.ascontiguousarray(sc, dtype=np.float32)
    y = np.zeros(max(n, 1), dtype=np.uint32 if y_tag == F32 else np.uint16)
    _check(lib().oracle_unpack_dequantize(_ptr(p), _ptr(m), _ptr(s), n, G, bits, _ptr(y), y_tag),
           "unpack_dequantize")
    return y[:n]


def S(b: int) -> float:
    return float(lib().oracle_S(b))


def predicted_variance(c, bits) -> float:
    c = np.ascontiguousarray(c, dtype=np.float64)
    b = np.ascontiguousarray(bits, dtype=np.int32)
    return float(lib().oracle_predicted_variance(_ptr(c), _ptr(b), c.size))


def allocate_bits(c, D, ladder, B: int):
    """Greedy. Returns (rc, bits)."""
    c = np.ascontiguousarray(c, dtype=np.float64)
    D = np.ascontiguousarray(D, dtype=np.int64)
    lad = np.ascontiguousarray(ladder, dtype=np.int32)
    out = np.zeros(max(c.size, 1), dtype=np.int32)
    rc = lib().oracle_allocate_bits(_ptr(c), _ptr(D), c.size, _ptr(lad), lad.size, B, _ptr(out))
    return rc, out[:c.size]


def allocate_bruteforce(c, D, ladder, B: int):
    """Exhaustive minimum of eqn:ilp. Returns (rc, bits, value)."""
    c = np.ascontiguousarray(c, dtype=np.float64)
    D = np.ascontiguousarray(D, dtype=np.int64)
    lad = np.ascontiguousarray(ladder, dtype=np.int32)
    out = np.zeros(max(c.size, 1), dtype=np.int32)
    val = np.zeros(1, dtype=np.float64)
    rc = lib().oracle_allocate_bruteforce(_ptr(c), _ptr(D), c.size, _ptr(lad), lad.size, B,
                                          _ptr(out), _ptr(val))
    return rc, out[:c.size], float(val[0])


def quantize_codes_span(x_span: np.ndarray, tag: int, n: int, G: int, bits: int, seed: int,
                        g0: int, g1: int):
    """Like quantize_codes for groups [g0, g1) of an n-element tensor, given only the host
    copy of those groups' elements (x_span = x[g0*G : min(g1*G, n)]). The oracle indexes the
    tensor by global element index; the base pointer is offset so that only the span is read."""
    x_span = np.ascontiguousarray(x_span).reshape(-1)
    n, G, bits, seed, g0, g1 = int(n), int(G), int(bits), int(seed), int(g0), int(g1)
    count = min(g1 * G, n) - g0 * G
    assert x_span.size == count and g1 > g0
    base = x_span.ctypes.data - g0 * G * x_span.itemsize
    q = np.zeros(count, dtype=np.uint8)
    mn = np.zeros(g1 - g0, dtype=np.float32)
    sc = np.zeros_like(mn)
    _check(lib().oracle_quantize_codes(base, tag, n, G, bits, seed, g0, g1, _ptr(q), _ptr(mn),
                                       _ptr(sc)), "quantize_codes_span")
    return q, mn, sc


def sq_diff_sum(a: np.ndarray, b: np.ndarray, tag: int) -> float:
    """||a - b||^2 (Alg. 1's ||g0 - g1||^2); bf16 arrays as uint16 patterns with tag=BF16."""
    a = np.ascontiguousarray(a).reshape(-1)
    b = np.ascontiguousarray(b).reshape(-1)
    assert a.size == b.size
    return float(lib().oracle_sq_diff_sum(_ptr(a), _ptr(b), tag, a.size))
