"""GPU: the staged (host-buffer) forms gact_quantize_pack_staged / gact_unpack_dequantize_staged
(include/gact.h; the paper's "Parallel Swap and Prefetch").

They must be bit-identical to the batch forms on the same descriptors (and so to the oracle)
whatever mix of host (pinned or pageable) and device buffers is passed, and however the
tensors are cut into pieces: small workspaces force many pieces per tensor (Philox counters
continue across piece boundaries) and many chunks through the rotating slots.
"""
import numpy as np
import pytest
import torch

from test_gpu_parity import TAGS, host_bits, make_input, oracle_input, ulp_distance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gact():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2206_11357_b200 as g
    g.lib()
    return g


def _inputs(seed=0):
    """Ragged sizes, mixed dtypes and bits; one tensor of 2^20 + 4099 elements."""
    sizes = [1, 255, 4096, 4097, 70_001, (1 << 20) + 4099, 12_288, 3]
    dts = [torch.bfloat16, torch.float32, torch.float16, torch.bfloat16, torch.float32,
           torch.bfloat16, torch.float16, torch.float32]
    bits = [2, 4, 8, 1, 2, 4, 8, 1]
    xs = [make_input(n, dt, seed + i, kind="mixed") for i, (n, dt) in enumerate(zip(sizes, dts))]
    seeds = [0x1234 + 7919 * i for i in range(len(xs))]
    return xs, bits, seeds


def _same(ct_a, ct_b):
    for a, b in ((ct_a.packed, ct_b.packed), (ct_a.group_min, ct_b.group_min),
                 (ct_a.group_scale, ct_b.group_scale)):
        assert np.array_equal(host_bits(a), host_bits(b))


@pytest.mark.parametrize("G", [32, 256, 2048, 4096])
@pytest.mark.parametrize("ws_bytes", [3 * 65536, 3 * (1 << 20), 3 * (64 << 20)])
def test_staged_quantize_equals_batch(gact, G, ws_bytes):
    xs, bits, seeds = _inputs()
    ref = gact.quantize_pack_batch(xs, bits, seeds, G)
    hx = [x.cpu().pin_memory() for x in xs]
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    got = gact.quantize_pack_staged(hx, bits, seeds, G, workspace=ws)
    torch.cuda.synchronize()
    assert all(not c.packed.is_cuda for c in got)
    for a, b in zip(got, ref):
        _same(a, b)
    # decompress from host codes (swap-in) == device decompress
    ys = gact.unpack_dequantize_staged(got, workspace=ws)
    ys_ref = gact.unpack_dequantize_batch(ref)
    torch.cuda.synchronize()
    for y, yr in zip(ys, ys_ref):
        assert y.is_cuda and np.array_equal(host_bits(y), host_bits(yr))


def test_staged_against_oracle_across_pieces(gact, orc):
    """A tensor cut into many pieces by a minimum workspace, checked against the oracle."""
    n, G, b, seed = 300_000 + 37, 256, 4, 0xBEEF
    x = make_input(n, torch.bfloat16, 5)
    ws = torch.empty(gact.STAGED_MIN_WORKSPACE, dtype=torch.uint8, device="cuda")
    (ct,) = gact.quantize_pack_staged([x.cpu().pin_memory()], [b], [seed], G, workspace=ws)
    rp, rmn, rsc = orc.quantize_pack(oracle_input(x), TAGS[x.dtype], G, b, seed)
    assert np.array_equal(host_bits(ct.packed), rp)
    assert np.array_equal(host_bits(ct.group_min), rmn.view(np.uint32))
    assert np.array_equal(host_bits(ct.group_scale), rsc.view(np.uint32))
    (y,) = gact.unpack_dequantize_staged([ct], workspace=ws, out_host=True)
    assert not y.is_cuda
    ry = orc.unpack_dequantize(rp, rmn, rsc, n, G, b, TAGS[x.dtype])
    assert ulp_distance(host_bits(y), ry, 16).max() <= 1


@pytest.mark.parametrize("x_host,out_host", [(False, True), (True, False), (False, False)])
def test_staged_mixed_placement(gact, x_host, out_host):
    xs, bits, seeds = _inputs(11)
    ref = gact.quantize_pack_batch(xs, bits, seeds, 256)
    src = [x.cpu().pin_memory() for x in xs] if x_host else xs
    ws = torch.empty(3 * (1 << 20), dtype=torch.uint8, device="cuda")
    got = gact.quantize_pack_staged(src, bits, seeds, 256, workspace=ws, out_host=out_host)
    torch.cuda.synchronize()
    for a, b in zip(got, ref):
        assert a.packed.is_cuda == (not out_host)
        _same(a, b)


def test_staged_pageable_host_memory(gact):
    xs, bits, seeds = _inputs(23)
    ref = gact.quantize_pack_batch(xs, bits, seeds, 256)
    hx = [x.cpu() for x in xs]  # not page-locked
    outs = [(torch.empty_like(c.packed, device="cpu"), torch.empty_like(c.group_min, device="cpu"),
             torch.empty_like(c.group_scale, device="cpu")) for c in ref]
    ws = torch.empty(3 * (1 << 20), dtype=torch.uint8, device="cuda")
    got = gact.quantize_pack_staged(hx, bits, seeds, 256, outs=outs, workspace=ws)
    for a, b in zip(got, ref):
        _same(a, b)
    ys = gact.unpack_dequantize_staged(got, outs=[torch.empty(x.shape, dtype=x.dtype) for x in xs],
                                       workspace=ws)
    ys_ref = gact.unpack_dequantize_batch(ref)
    torch.cuda.synchronize()
    for y, yr in zip(ys, ys_ref):
        assert np.array_equal(host_bits(y), host_bits(yr))


def test_staged_orders_after_stream_work(gact):
    """Device inputs produced by earlier work on the stream are read after that work."""
    x = torch.empty(1 << 22, dtype=torch.bfloat16, device="cuda")
    torch.cuda._sleep(20_000_000)  # keep the stream busy so the fill below is still queued
    x.copy_(torch.linspace(-3, 3, x.numel(), device="cuda").to(torch.bfloat16))
    (ct,) = gact.quantize_pack_staged([x], [4], [9], 256)
    ref = gact.quantize_pack(x, 4, 9, 256)
    torch.cuda.synchronize()
    _same(ct, ref)


def test_staged_validation(gact):
    import ctypes
    L = gact.lib()
    x = torch.zeros(4096, dtype=torch.bfloat16).pin_memory()
    p = torch.zeros(1024, dtype=torch.int32).pin_memory()
    m = torch.zeros(16).pin_memory()
    row = (x.data_ptr(), p.data_ptr(), m.data_ptr(), m.data_ptr(), 4096, 1, 4, 1)
    ws = torch.empty(gact.STAGED_MIN_WORKSPACE, dtype=torch.uint8, device="cuda")
    arr = gact._desc_array([row])
    s = torch.cuda.current_stream().cuda_stream
    assert L.gact_quantize_pack_staged(arr, 1, 256, ws.data_ptr(), ws.numel() - 1, s) == 1
    assert L.gact_quantize_pack_staged(arr, 1, 256, ws.data_ptr() + 16, ws.numel() - 256, s) == 1
    assert L.gact_quantize_pack_staged(arr, 1, 100, ws.data_ptr(), ws.numel(), s) == 3
    bad = gact._desc_array([(x.data_ptr() + 2,) + row[1:]])
    assert L.gact_quantize_pack_staged(bad, 1, 256, ws.data_ptr(), ws.numel(), s) == 4
    assert L.gact_quantize_pack_staged(arr, 1, 256, ws.data_ptr(), ws.numel(), s) == 0
    assert L.gact_quantize_pack_staged(ctypes.cast(None, ctypes.POINTER(gact._Desc)), 0, 256,
                                       ws.data_ptr(), ws.numel(), s) == 0


@pytest.mark.parametrize("G", [96, 288, 1056, 2080, 4064])
@pytest.mark.parametrize("ws_bytes", [3 * (4 << 20), 3 * (64 << 20)])
def test_staged_generic_group_sizes(gact, orc, G, ws_bytes):
    """Group sizes that are not powers of two stage in pieces of lcm(G, 4096) elements (a
    piece never splits a group, and its Philox block offset stays off / 16): bit-identical to
    the batch forms, and the codes equal the oracle's."""
    xs, bits, seeds = _inputs(seed=G)
    ref = gact.quantize_pack_batch(xs, bits, seeds, G)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    got = gact.quantize_pack_staged([x.cpu().pin_memory() for x in xs], bits, seeds, G, workspace=ws)
    ys = gact.unpack_dequantize_staged(got, workspace=ws)
    ys_ref = gact.unpack_dequantize_batch(ref)
    torch.cuda.synchronize()
    for x, b, s, a, r, y, yr in zip(xs, bits, seeds, got, ref, ys, ys_ref):
        _same(a, r)
        assert torch.equal(y.view(-1).view(torch.uint8), yr.view(-1).view(torch.uint8))
        p, mn, sc = orc.quantize_pack(oracle_input(x), TAGS[x.dtype], G, b, s)
        assert np.array_equal(host_bits(a.packed), p)
        assert np.array_equal(host_bits(a.group_min), mn.view(np.uint32))
