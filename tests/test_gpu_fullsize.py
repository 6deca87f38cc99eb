"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(batched launches over the whole context, the bench's seeds and allocation): codes,
group min/scale and decoded values of SAMPLED groups of every tensor are compared with the
oracle (which computes those groups one by one from the host copy of their inputs), and
properties that hold at any size are checked on everything (codes within [0, 2^b - 1] via
the decoded range, decoded values inside [min, max] of their group).

configs[1]: 256 MiB bf16 at b = 1, 2, 4, 8; configs[2]: the ResNet-50 b256 context (105
tensors, 5.36 G elements, adaptive bits avg 4); configs[3]: one BERT-large layer (b avg 2);
configs[4] (per rank): GCN + Swin-T.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

TAGS = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}
G = 256


@pytest.fixture(scope="module")
def gact():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2206_11357_b200 as g
    g.lib()
    return g


def _bits_u32(t):
    return t.detach().contiguous().view(torch.int32).cpu().numpy().view(np.uint32).reshape(-1)


def _host_span(x, lo, hi):
    s = x.reshape(-1)[lo:hi].contiguous().cpu()
    if s.dtype == torch.float32:
        return s.numpy()
    return s.view(torch.int16).numpy().view(np.uint16)


def _ulp_distance(a, b, width):
    sign, mag = 1 << (width - 1), (1 << (width - 1)) - 1
    key = lambda v: np.where(v & sign, -(v & mag), v & mag)  # noqa: E731
    return np.abs(key(a) - key(b))


def _check_sampled(orc, x, ct, y, bits, seed, rng, nsamples=24):
    n = x.numel()
    ng = (n + G - 1) // G
    groups = sorted(set([0, ng - 1] + list(rng.integers(0, ng, size=nsamples))))
    packed = ct.packed
    for g in groups:
        lo, hi = g * G, min(n, (g + 1) * G)
        span = _host_span(x, lo, hi)
        q, mn, sc = orc.quantize_codes_span(span, TAGS[x.dtype], n, G, bits, seed, g, g + 1)
        assert _bits_u32(ct.group_min[g:g + 1])[0] == mn.view(np.uint32)[0]
        assert _bits_u32(ct.group_scale[g:g + 1])[0] == sc.view(np.uint32)[0]
        # the group's words (G*b/32 of them; a group starts on a word boundary)
        w0, w1 = lo * bits // 32, (hi * bits + 31) // 32
        words = _bits_u32(packed[w0:w1])
        got = orc.unpack(words, hi - lo, bits)
        assert np.array_equal(got, q), f"group {g}: {np.sum(got != q)} codes differ"
        # decoded values within 1 ulp of the oracle's
        ref = orc.unpack_dequantize(words, mn, sc, hi - lo, G, bits, TAGS[y.dtype])
        yv = y.reshape(-1)[lo:hi].contiguous().cpu()
        width = 32 if yv.dtype == torch.float32 else 16
        yb = yv.view(torch.int32 if width == 32 else torch.int16).numpy().astype(np.int64) & ((1 << width) - 1)
        assert _ulp_distance(yb, ref.astype(np.int64), width).max() <= 1


def _check_range_property(x, ct, y):
    """Every decoded value lies in [mn, mn + L*scale] of its group (any size)."""
    n = x.numel()
    ng = ct.group_min.numel()
    yf = y.reshape(-1).float()
    pad = ng * G - n
    if pad:
        yf = torch.cat([yf, yf[-1:].expand(pad)])
    yg = yf.view(ng, G)
    L = (1 << ct.bits) - 1
    lo = ct.group_min.view(ng, 1)
    hi = (ct.group_min + L * ct.group_scale).view(ng, 1)
    tol = 1e-2 * ct.group_scale.view(ng, 1) + 1e-30
    if y.dtype != torch.float32:
        tol = tol + (hi.abs() + lo.abs()) * 2 ** -7
    assert bool(((yg >= lo - tol) & (yg <= hi + tol)).all())


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_buf256_bits_sweep(gact, orc, bits):
    spec = synth.workload_specs("buf256")[0]
    x = synth.make_tensor(spec, synth.DATA_SEED, "cuda", torch.bfloat16)
    seed = synth.tensor_seed(2022, 0)
    ct = gact.quantize_pack(x, bits, seed, G)
    y = ct.decompress()
    torch.cuda.synchronize()
    _check_sampled(orc, x, ct, y, bits, seed, np.random.default_rng(bits))
    _check_range_property(x, ct, y)


def _run_workload(gact, orc, name, avg_bits, dtype=torch.bfloat16, rank=0):
    specs = synth.workload_specs(name)
    dev = torch.device("cuda")
    xs = [synth.make_tensor(s, synth.DATA_SEED + 1000 * rank + i, dev, dtype) for i, s in enumerate(specs)]
    D = np.array([s.numel for s in specs], dtype=np.int64)
    c = synth.sensitivities(specs, seed=7, rank=rank)
    bits = gact.allocate_bits(c, D, int(avg_bits * D.sum()))
    rc, ref_bits = orc.allocate_bits(c, D, [1, 2, 4, 8], int(avg_bits * D.sum()))
    assert rc == 0 and np.array_equal(bits, ref_bits)
    seeds = [synth.tensor_seed(2022, i, rank) for i in range(len(specs))]
    cts = gact.quantize_pack_batch(xs, bits.tolist(), seeds, G)
    ys = gact.unpack_dequantize_batch(cts)
    torch.cuda.synchronize()
    rng = np.random.default_rng(len(specs))
    for x, ct, y, b, s in zip(xs, cts, ys, bits, seeds):
        _check_sampled(orc, x, ct, y, int(b), s, rng, nsamples=4)
        _check_range_property(x, ct, y)
    return bits


def test_resnet50_context(gact, orc):
    bits = _run_workload(gact, orc, "resnet50", 4.0)
    assert len(bits) == 105 and bits[-1] == 8  # the loss head is the most sensitive


def test_bert_layer(gact, orc):
    _run_workload(gact, orc, "bert_layer", 2.0)


def test_gcn_swin_rank1(gact, orc):
    _run_workload(gact, orc, "gcn_swin", 2.0, rank=1)


def test_bert_layer_staged_host_buffers(gact, orc):
    """The host-buffer forms (the bench's e2e path) at full size: one BERT-large layer
    (2^30 elements, 2 GiB bf16) from pinned host memory through the default workspace,
    bit-identical to the device batch forms everywhere, and oracle-exact on sampled groups."""
    specs = synth.workload_specs("bert_layer")
    xs = [synth.make_tensor(s, synth.DATA_SEED + i, "cuda", torch.bfloat16) for i, s in enumerate(specs)]
    D = np.array([s.numel for s in specs], dtype=np.int64)
    bits = gact.allocate_bits(synth.sensitivities(specs, seed=7), D, int(2.0 * D.sum())).tolist()
    seeds = [synth.tensor_seed(2022, i) for i in range(len(specs))]
    ref = gact.quantize_pack_batch(xs, bits, seeds, G)
    hx = [x.cpu().pin_memory() for x in xs]
    got = gact.quantize_pack_staged(hx, bits, seeds, G)
    for a, b in zip(got, ref):
        assert not a.packed.is_cuda
        for ha, db in ((a.packed, b.packed), (a.group_min, b.group_min), (a.group_scale, b.group_scale)):
            assert torch.equal(ha.cuda().view(torch.int32), db.view(torch.int32))
    ys = gact.unpack_dequantize_staged(got)
    ys_ref = gact.unpack_dequantize_batch(ref)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    for x, ct, y, yr, b, s in zip(xs, got, ys, ys_ref, bits, seeds):
        assert torch.equal(y.view(torch.int16), yr.view(torch.int16))
        _check_sampled(orc, x, ct, y, int(b), s, rng, nsamples=3)


@pytest.mark.parametrize("G", [256, 4064])
def test_tensor_past_2_31_elements(gact, orc, G):
    """One tensor of 2^31 + 3 * 2^20 + 77 bf16 elements (4.3 GB): 64-bit element, word and
    group indices and Philox block counters past 2^31 / 2^32 elements, in the specialised and
    the generic kernels. Groups at the start, around element 2^31 and at the ragged end are
    compared with the oracle (codes, min, scale, decoded values)."""
    n = (1 << 31) + 3 * (1 << 20) + 77
    x = torch.randn(n, device="cuda", dtype=torch.bfloat16)
    seed = 0xB16B00B5
    ct = gact.quantize_pack(x, 4, seed, G)
    y = ct.decompress()
    torch.cuda.synchronize()
    ng = (n + G - 1) // G
    mid = (1 << 31) // G
    groups = sorted({0, 1, mid - 1, mid, mid + 1, ng - 2, ng - 1} | set(np.random.default_rng(G).integers(0, ng, 8)))
    for g in groups:
        lo, hi = g * G, min(n, (g + 1) * G)
        span = _host_span(x, lo, hi)
        q, mn, sc = orc.quantize_codes_span(span, TAGS[x.dtype], n, G, 4, seed, g, g + 1)
        assert _bits_u32(ct.group_min[g:g + 1])[0] == mn.view(np.uint32)[0], g
        assert _bits_u32(ct.group_scale[g:g + 1])[0] == sc.view(np.uint32)[0], g
        w0, w1 = lo * 4 // 32, (hi * 4 + 31) // 32
        words = _bits_u32(ct.packed[w0:w1])
        assert np.array_equal(orc.unpack(words, hi - lo, 4), q), g
        ref = orc.unpack_dequantize(words, mn, sc, hi - lo, G, 4, TAGS[y.dtype])
        yb = y.reshape(-1)[lo:hi].contiguous().cpu().view(torch.int16).numpy().astype(np.int64) & 0xFFFF
        assert _ulp_distance(yb, ref.astype(np.int64), 16).max() <= 1
    del x, y, ct
    torch.cuda.empty_cache()
