"""paper_2206_11357_b200 — B200-native GACT activation-compressor hot path.

Thin Python binding of the C ABI in include/gact.h (libgact.so, sm_100a CUDA kernels):
argument marshalling only. PyTorch supplies device memory (the caching allocator),
streams (the current stream is passed to every call) and process groups (dist.py).
Every step of the path runs in libgact's kernels; there is no CPU fallback: functions
raise if the library is missing or a tensor is not on a CUDA device.

Names follow the paper (arXiv 2206.11357): bits b, group size G, per-group min and scale,
sensitivity c_l, numel D_l, budget B (P:n = /root/reference/PAPER.md line n):
  quantize_pack        Q_b(h^(l))    App. Prop. 3
  unpack_dequantize    T^{-1}
  group_stats          min/max
  allocate_bits        eqn:ilp       P:471-475, greedy P:534
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

import numpy as np
import torch

__all__ = [
    "lib", "GactError", "F32", "BF16", "F16", "DEFAULT_GROUP", "LADDER",
    "num_groups", "packed_words", "group_stats", "quantize_pack", "unpack_dequantize",
    "quantize_pack_batch", "unpack_dequantize_batch", "allocate_bits", "CompressedTensor",
    "sq_diff_sum", "variance_factor", "BatchPlan", "quantize_pack_staged", "unpack_dequantize_staged",
    "staged_workspace",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GACT_LIB_PATH") or os.path.join(_HERE, "libgact.so")  # override: experiments only

F32, BF16, F16 = 0, 1, 2
DEFAULT_GROUP = 256
LADDER = (1, 2, 4, 8)
MAX_BATCH = 256
REDUCE_BLOCKS = 512  # GACT_REDUCE_BLOCKS
STAGED_SLOTS = 3  # GACT_STAGED_SLOTS
STAGED_MIN_WORKSPACE = 3 * 65536  # GACT_STAGED_MIN_WORKSPACE
STAGED_DEFAULT_WORKSPACE = 3 * (64 << 20)
_TORCH_TAG = {torch.float32: F32, torch.bfloat16: BF16, torch.float16: F16}
_TAG_TORCH = {v: k for k, v in _TORCH_TAG.items()}


class GactError(RuntimeError):
    """A libgact call returned a non-OK gact_status."""

    def __init__(self, fn: str, status: int):
        self.status = status
        name = lib().gact_status_string(status).decode()
        super().__init__(f"{fn}: {name} ({status})")


class _Desc(ctypes.Structure):
    """gact_tensor_desc (include/gact.h)."""
    _fields_ = [
        ("data", ctypes.c_void_p), ("packed", ctypes.c_void_p),
        ("group_min", ctypes.c_void_p), ("group_scale", ctypes.c_void_p),
        ("n", ctypes.c_int64), ("seed", ctypes.c_uint64),
        ("bits", ctypes.c_int32), ("dtype", ctypes.c_int32),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """The loaded libgact.so (raises if it has not been built: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        sig = {
            "gact_version": (i32, []),
            "gact_status_string": (ctypes.c_char_p, [i32]),
            "gact_num_groups": (i64, [i64, i32]),
            "gact_packed_words": (i64, [i64, i32]),
            "gact_group_stats": (i32, [P, i32, i64, i32, i32, P, P, P]),
            "gact_quantize_pack": (i32, [P, i32, i64, i32, i32, u64, P, P, P, P]),
            "gact_unpack_dequantize": (i32, [P, P, P, i64, i32, i32, P, i32, P]),
            "gact_quantize_pack_batch": (i32, [ctypes.POINTER(_Desc), i32, i32, P]),
            "gact_unpack_dequantize_batch": (i32, [ctypes.POINTER(_Desc), i32, i32, P]),
            "gact_allocate_bits": (i32, [P, P, i32, P, i32, u64, P]),
            "gact_variance_factor": (ctypes.c_double, [i32]),
            "gact_sq_diff_sum": (i32, [P, P, i32, i64, P, P, P]),
            "gact_quantize_pack_staged": (i32, [ctypes.POINTER(_Desc), i32, i32, P, u64, P]),
            "gact_unpack_dequantize_staged": (i32, [ctypes.POINTER(_Desc), i32, i32, P, u64, P]),
            "gact_test_philox_blocks": (i32, [u64, u64, i32, i32, P, P]),  # include/gact_testing.h
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(fn: str, status: int) -> None:
    if status != 0:
        raise GactError(fn, status)


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda:
            raise ValueError("libgact runs on CUDA tensors only (no CPU fallback)")


def _need(t: torch.Tensor, numel: int, dtype, device, what: str) -> None:
    """A caller-supplied buffer the kernels will read or write: it must be a contiguous CUDA
    tensor of `dtype` on `device` with at least `numel` elements (checked before any call,
    so a short or strided buffer raises instead of being written out of bounds)."""
    if not t.is_cuda or t.device != device:
        raise ValueError(f"{what}: must be on {device}, got {t.device}")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{what}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: must be contiguous")
    if t.numel() < numel:
        raise ValueError(f"{what}: {t.numel()} elements, needs >= {numel}")


def _aligned(x: torch.Tensor) -> torch.Tensor:
    """x contiguous and 16-byte aligned (the C ABI's requirement): a view whose storage offset
    breaks the alignment (x[1:], an odd split) is copied once."""
    x = x.contiguous()
    if x.data_ptr() % 16:
        x = x.clone()
    return x


def _codes_need(packed, group_min, group_scale, n, bits, group_size, device, what):
    _need(packed, max(packed_words(n, bits), 0), torch.int32, device, f"{what}: packed")
    ng = max(num_groups(n, group_size), 0)
    _need(group_min, ng, torch.float32, device, f"{what}: group_min")
    _need(group_scale, ng, torch.float32, device, f"{what}: group_scale")


def num_groups(n: int, group_size: int = DEFAULT_GROUP) -> int:
    return int(lib().gact_num_groups(n, group_size))


def packed_words(n: int, bits: int) -> int:
    return int(lib().gact_packed_words(n, bits))


class CompressedTensor:
    """Q_b(h^(l)): packed codes + per-group (min, scale), and how to undo it."""
    __slots__ = ("packed", "group_min", "group_scale", "shape", "dtype", "bits", "group_size", "seed")

    def __init__(self, packed, group_min, group_scale, shape, dtype, bits, group_size, seed):
        self.packed, self.group_min, self.group_scale = packed, group_min, group_scale
        self.shape, self.dtype, self.bits, self.group_size, self.seed = shape, dtype, bits, group_size, seed

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape)) if len(self.shape) else 1

    def nbytes(self) -> int:
        return (self.packed.numel() * 4 + self.group_min.numel() * 4 + self.group_scale.numel() * 4)

    def decompress(self, out: torch.Tensor | None = None, device=None) -> torch.Tensor:
        """Device-resident codes: gact_unpack_dequantize. Host-resident codes (a swapped-out
        context): gact_unpack_dequantize_staged into `out` or a new tensor on `device`."""
        if not self.packed.is_cuda:
            return unpack_dequantize_staged([self], None if out is None else [out], device=device)[0]
        return unpack_dequantize(self.packed, self.group_min, self.group_scale, self.numel,
                                 self.bits, self.group_size, self.dtype, out=out).view(self.shape)


def group_stats(x: torch.Tensor, bits: int, group_size: int = DEFAULT_GROUP):
    """Per-group (min, scale) of a CUDA tensor (flattened row-major)."""
    _require_cuda(x)
    x = _aligned(x)
    n = x.numel()
    ng = max(num_groups(n, group_size), 0)
    mn = torch.empty(ng, dtype=torch.float32, device=x.device)
    sc = torch.empty(ng, dtype=torch.float32, device=x.device)
    _check("gact_group_stats", lib().gact_group_stats(
        x.data_ptr(), _TORCH_TAG[x.dtype], n, group_size, bits, mn.data_ptr(), sc.data_ptr(), _stream(x)))
    return mn, sc


def quantize_pack(x: torch.Tensor, bits: int, seed: int, group_size: int = DEFAULT_GROUP,
                  out: tuple | None = None) -> CompressedTensor:
    """Compress one context tensor: fused group min/max + stochastic rounding + packing."""
    _require_cuda(x)
    xc = _aligned(x)
    n = xc.numel()
    if out is None:
        packed = torch.empty(max(packed_words(n, bits), 0), dtype=torch.int32, device=x.device)
        mn = torch.empty(max(num_groups(n, group_size), 0), dtype=torch.float32, device=x.device)
        sc = torch.empty_like(mn)
    else:
        packed, mn, sc = out
        _codes_need(packed, mn, sc, n, bits, group_size, x.device, "quantize_pack out")
    _check("gact_quantize_pack", lib().gact_quantize_pack(
        xc.data_ptr(), _TORCH_TAG[x.dtype], n, group_size, bits, seed & (2**64 - 1),
        packed.data_ptr(), mn.data_ptr(), sc.data_ptr(), _stream(xc)))
    return CompressedTensor(packed, mn, sc, tuple(x.shape), x.dtype, bits, group_size, seed)


def unpack_dequantize(packed: torch.Tensor, group_min: torch.Tensor, group_scale: torch.Tensor,
                      n: int, bits: int, group_size: int = DEFAULT_GROUP,
                      dtype: torch.dtype = torch.float32, out: torch.Tensor | None = None) -> torch.Tensor:
    """Decompress: y = RNE_dtype(fma(q, scale, mn)) for n elements."""
    _require_cuda(packed, group_min, group_scale)
    _codes_need(packed, group_min, group_scale, n, bits, group_size, packed.device, "unpack_dequantize")
    if out is None:
        y = torch.empty(n, dtype=dtype, device=packed.device)
    else:
        y = out
        _need(y, n, None, packed.device, "unpack_dequantize out")
        if y.dtype not in _TORCH_TAG:
            raise ValueError(f"unpack_dequantize out: unsupported dtype {y.dtype}")
    _check("gact_unpack_dequantize", lib().gact_unpack_dequantize(
        packed.data_ptr(), group_min.data_ptr(), group_scale.data_ptr(), n, group_size, bits,
        y.data_ptr(), _TORCH_TAG[y.dtype], _stream(packed)))
    return y


def _desc_array(rows) -> ctypes.Array:
    arr = (_Desc * max(len(rows), 1))()
    for i, r in enumerate(rows):
        arr[i] = _Desc(*r)
    return arr


def quantize_pack_batch(xs: Sequence[torch.Tensor], bits: Sequence[int], seeds: Sequence[int],
                        group_size: int = DEFAULT_GROUP, outs: Sequence[tuple] | None = None):
    """Compress a whole context h = (h^(l)) with per-tensor bits in one launch per
    (dtype, bits) class. Returns a list of CompressedTensor."""
    res, rows = [], []
    for i, (x, b, s) in enumerate(zip(xs, bits, seeds)):
        _require_cuda(x)
        if not x.is_contiguous():
            raise ValueError("quantize_pack_batch needs contiguous tensors")
        if x.device != xs[0].device:
            raise ValueError("quantize_pack_batch: all tensors on one device")
        n = x.numel()
        if outs is None:
            packed = torch.empty(max(packed_words(n, b), 0), dtype=torch.int32, device=x.device)
            mn = torch.empty(max(num_groups(n, group_size), 0), dtype=torch.float32, device=x.device)
            sc = torch.empty_like(mn)
        else:
            packed, mn, sc = outs[i]
            _codes_need(packed, mn, sc, n, b, group_size, x.device, f"quantize_pack_batch outs[{i}]")
        rows.append((x.data_ptr(), packed.data_ptr(), mn.data_ptr(), sc.data_ptr(), n,
                     s & (2**64 - 1), b, _TORCH_TAG[x.dtype]))
        res.append(CompressedTensor(packed, mn, sc, tuple(x.shape), x.dtype, b, group_size, s))
    if rows:
        _check("gact_quantize_pack_batch", lib().gact_quantize_pack_batch(
            _desc_array(rows), len(rows), group_size, _stream(xs[0])))
    return res


def unpack_dequantize_batch(cts: Sequence[CompressedTensor], outs: Sequence[torch.Tensor] | None = None):
    """Decompress a list of CompressedTensor (one launch per (dtype, bits) class)."""
    ys, rows = [], []
    gs = {c.group_size for c in cts}
    if len(gs) > 1:
        raise ValueError("one group size per batch")
    for i, c in enumerate(cts):
        _require_cuda(c.packed, c.group_min, c.group_scale)
        _codes_need(c.packed, c.group_min, c.group_scale, c.numel, c.bits, c.group_size, cts[0].packed.device,
                    f"unpack_dequantize_batch[{i}]")
        if outs is None:
            y = torch.empty(c.shape, dtype=c.dtype, device=c.packed.device)
        else:
            y = outs[i]
            _need(y, c.numel, None, cts[0].packed.device, f"unpack_dequantize_batch outs[{i}]")
        rows.append((y.data_ptr(), c.packed.data_ptr(), c.group_min.data_ptr(),
                     c.group_scale.data_ptr(), c.numel, 0, c.bits, _TORCH_TAG[y.dtype]))
        ys.append(y)
    if rows:
        _check("gact_unpack_dequantize_batch", lib().gact_unpack_dequantize_batch(
            _desc_array(rows), len(rows), gs.pop(), _stream(cts[0].packed)))
    return ys


_workspaces: dict = {}


def staged_workspace(device=None, nbytes: int = STAGED_DEFAULT_WORKSPACE) -> torch.Tensor:
    """The device workspace of the staged calls (cached per device; grows on demand)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    ws = _workspaces.get(dev)
    if ws is None or ws.numel() < nbytes:
        ws = _workspaces[dev] = torch.empty(max(nbytes, STAGED_MIN_WORKSPACE), dtype=torch.uint8, device=dev)
    return ws


def _staged_device(tensors, device):
    if device is not None:
        return torch.device(device)
    for t in tensors:
        if t.is_cuda:
            return t.device
    if not torch.cuda.is_available():
        raise ValueError("libgact runs on CUDA devices only (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _host_out(shape, dtype, like_host: bool, device):
    if like_host:
        return torch.empty(shape, dtype=dtype, pin_memory=True)
    return torch.empty(shape, dtype=dtype, device=device)


def quantize_pack_staged(xs: Sequence[torch.Tensor], bits: Sequence[int], seeds: Sequence[int],
                         group_size: int = DEFAULT_GROUP, outs: Sequence[tuple] | None = None,
                         device=None, workspace: torch.Tensor | None = None, out_host: bool = True):
    """Compress tensors that live in HOST memory (pinned for overlap) or on the device, with
    the compressed context written to host memory (default) or the device: the swap-out of
    "Parallel Swap and Prefetch" in one blocking libgact call
    (gact_quantize_pack_staged). Bit-identical to quantize_pack_batch."""
    dev = _staged_device(xs, device)
    ws = staged_workspace(dev) if workspace is None else workspace
    res, rows = [], []
    for i, (x, b, s) in enumerate(zip(xs, bits, seeds)):
        if not x.is_contiguous():
            raise ValueError("quantize_pack_staged needs contiguous tensors")
        n = x.numel()
        if outs is None:
            packed = _host_out(max(packed_words(n, b), 0), torch.int32, out_host, dev)
            mn = _host_out(max(num_groups(n, group_size), 0), torch.float32, out_host, dev)
            sc = _host_out(max(num_groups(n, group_size), 0), torch.float32, out_host, dev)
        else:
            packed, mn, sc = outs[i]
        rows.append((x.data_ptr(), packed.data_ptr(), mn.data_ptr(), sc.data_ptr(), n,
                     s & (2**64 - 1), b, _TORCH_TAG[x.dtype]))
        res.append(CompressedTensor(packed, mn, sc, tuple(x.shape), x.dtype, b, group_size, s))
    if rows:
        with torch.cuda.device(dev):
            _check("gact_quantize_pack_staged", lib().gact_quantize_pack_staged(
                _desc_array(rows), len(rows), group_size, ws.data_ptr(), ws.numel(),
                torch.cuda.current_stream(dev).cuda_stream))
    return res


def unpack_dequantize_staged(cts: Sequence[CompressedTensor], outs: Sequence[torch.Tensor] | None = None,
                             device=None, workspace: torch.Tensor | None = None, out_host: bool = False):
    """Decompress contexts whose codes live in HOST memory (or on the device) into device
    tensors (default; the swap-in + decompress of P:589-592) or host tensors, in one blocking
    libgact call (gact_unpack_dequantize_staged). Bit-identical to unpack_dequantize_batch."""
    gs = {c.group_size for c in cts}
    if len(gs) > 1:
        raise ValueError("one group size per batch")
    dev = _staged_device([c.packed for c in cts] + list(outs or []), device)
    ws = staged_workspace(dev) if workspace is None else workspace
    ys, rows = [], []
    for i, c in enumerate(cts):
        y = _host_out(c.shape, c.dtype, out_host, dev) if outs is None else outs[i]
        rows.append((y.data_ptr(), c.packed.data_ptr(), c.group_min.data_ptr(),
                     c.group_scale.data_ptr(), c.numel, 0, c.bits, _TORCH_TAG[y.dtype]))
        ys.append(y)
    if rows:
        with torch.cuda.device(dev):
            _check("gact_unpack_dequantize_staged", lib().gact_unpack_dequantize_staged(
                _desc_array(rows), len(rows), gs.pop(), ws.data_ptr(), ws.numel(),
                torch.cuda.current_stream(dev).cuda_stream))
    return ys


def allocate_bits(sensitivity, numel, budget_bits: int, ladder: Sequence[int] = LADDER) -> np.ndarray:
    """Greedy solution of eqn:ilp (host computation inside libgact)."""
    c = np.ascontiguousarray(sensitivity, dtype=np.float64)
    D = np.ascontiguousarray(numel, dtype=np.int64)
    lad = np.ascontiguousarray(ladder, dtype=np.int32)
    out = np.zeros(max(c.size, 1), dtype=np.int32)
    _check("gact_allocate_bits", lib().gact_allocate_bits(
        c.ctypes.data, D.ctypes.data, c.size, lad.ctypes.data, lad.size, int(budget_bits), out.ctypes.data))
    return out[:c.size]


def variance_factor(bits: int) -> float:
    """S(b) of P:479-480 (S(32) = 0): gact_variance_factor, the allocator's own definition."""
    v = float(lib().gact_variance_factor(int(bits)))
    if v < 0:
        raise ValueError(f"no variance factor for {bits} bits")
    return v


def sq_diff_sum(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """||a - b||^2 as a 1-element float64 CUDA tensor (deterministic reduction in libgact;
    the ||g0 - g1||^2 of Alg. 1)."""
    _require_cuda(a, b)
    if a.shape != b.shape or a.dtype != b.dtype:
        raise ValueError("sq_diff_sum needs two tensors of the same shape and dtype")
    a, b = a.contiguous(), b.contiguous()
    partials = torch.empty(REDUCE_BLOCKS, dtype=torch.float64, device=a.device)  # caller-owned workspace
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    _check("gact_sq_diff_sum", lib().gact_sq_diff_sum(
        a.data_ptr(), b.data_ptr(), _TORCH_TAG[a.dtype], a.numel(), partials.data_ptr(),
        out.data_ptr(), _stream(a)))
    return out


# numpy view of gact_tensor_desc (include/gact.h): 4 pointers, n, seed, bits, dtype = 56 bytes
_DESC_NP = np.dtype([("data", np.uint64), ("packed", np.uint64), ("group_min", np.uint64),
                     ("group_scale", np.uint64), ("n", np.int64), ("seed", np.uint64),
                     ("bits", np.int32), ("dtype", np.int32)])
assert _DESC_NP.itemsize == ctypes.sizeof(_Desc)


class BatchPlan:
    """A prepared batched call over fixed tensors and bits (the descriptor table is built once;
    a step only rewrites the seeds). `kind` is "quantize" (xs are inputs, outs the
    (packed, min, scale) triples) or "dequantize" (xs are outputs y, outs the triples read)."""

    def __init__(self, kind: str, xs, outs, bits, group_size: int = DEFAULT_GROUP):
        self.kind, self.group_size = kind, group_size
        self.refs = (list(xs), list(outs))  # keep the tensors alive
        self.table = np.zeros(len(xs), dtype=_DESC_NP)
        for i, (x, (p, mn, sc), b) in enumerate(zip(xs, outs, bits)):
            _require_cuda(x, p, mn, sc)
            _need(x, x.numel(), None, xs[0].device, f"BatchPlan xs[{i}]")
            _codes_need(p, mn, sc, x.numel(), int(b), group_size, xs[0].device, f"BatchPlan outs[{i}]")
            self.table[i] = (x.data_ptr(), p.data_ptr(), mn.data_ptr(), sc.data_ptr(), x.numel(), 0, int(b),
                             _TORCH_TAG[x.dtype])
        self.stream_of = xs[0] if len(xs) else None
        self.fn = lib().gact_quantize_pack_batch if kind == "quantize" else lib().gact_unpack_dequantize_batch

    def set_seeds(self, seeds) -> None:
        self.table["seed"] = np.asarray(seeds, dtype=np.uint64)

    def run(self) -> None:
        if not len(self.table):
            return
        ptr = ctypes.cast(self.table.ctypes.data, ctypes.POINTER(_Desc))
        _check(f"gact_{self.kind}_batch", self.fn(ptr, len(self.table), self.group_size, _stream(self.stream_of)))
