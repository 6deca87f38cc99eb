"""Data-parallel piece of the path: the per-tensor sensitivity vector is
the only cross-GPU data. Each rank estimates c^(r) on its own micro-batch; one small
all-reduce (NCCL over NVLink on B200s, gloo in the CPU tests) merges them,
c = (sum_r c^(r)) / world in fp64, so that every rank runs the same deterministic greedy
(gact_allocate_bits) and obtains the same bits b (one c_l per tensor).

torch.distributed is plumbing here; no compression data crosses ranks.
"""
from __future__ import annotations

import hashlib

import numpy as np
import torch
import torch.distributed as dist


def _active(force: bool = False) -> bool:
    if not (dist.is_available() and dist.is_initialized()):
        return False
    return force or dist.get_world_size() > 1


_side_streams: dict = {}


def _side_stream(device) -> torch.cuda.Stream:
    """The exchange's stream on `device`: highest priority, so that the all-reduce kernel is
    scheduled ahead of queued compression CTAs as soon as SMs free up."""
    side = _side_streams.get(device)
    if side is None:
        lo, hi = torch.cuda.Stream.priority_range()
        side = _side_streams[device] = torch.cuda.Stream(device, priority=min(lo, hi))
    return side


def merge_sensitivities(c_local, device=None, force: bool = False) -> np.ndarray:
    """All-reduce(SUM) / world of the local sensitivity vector (float64, L entries).

    With NCCL the exchange runs on a dedicated high-priority side stream, so that waiting for
    the merged vector (the allocator runs on the host) waits only for the exchange, not for the
    compute stream's queue. `force` runs the exchange in a one-rank group too (tests)."""
    c = np.ascontiguousarray(c_local, dtype=np.float64)
    if not _active(force):
        return c
    backend = dist.get_backend()
    if backend == "nccl" and device is not None:
        side = _side_stream(device)
        with torch.cuda.stream(side):
            t = torch.from_numpy(c).to(device, non_blocking=False)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            t /= dist.get_world_size()
            out = t.cpu().numpy()
        return out
    t = torch.from_numpy(c)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    t /= dist.get_world_size()
    return t.numpy()


def allocation_digest(bits) -> int:
    """63-bit digest of an allocation (for cross-rank agreement checks)."""
    h = hashlib.blake2b(np.ascontiguousarray(bits, dtype=np.int32).tobytes(), digest_size=8).digest()
    return int.from_bytes(h, "little") >> 1


def assert_same_allocation(bits, device=None) -> None:
    """Every rank holds the same bits: all-reduce MIN and MAX of the digest agree."""
    if not _active():
        return
    backend = dist.get_backend()
    dev = device if (backend == "nccl" and device is not None) else torch.device("cpu")
    d = allocation_digest(bits)
    lo = torch.tensor([d], dtype=torch.int64, device=dev)
    hi = lo.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    if int(lo.item()) != int(hi.item()):
        raise RuntimeError("ranks disagree on the bit allocation")
