"""GPU parity on EVERY group at BASELINE.json's full sizes (the verdict's "whole-tensor,
every-group parity"): configs[1] (256 MiB bf16, b = 1, 2, 4, 8, single-tensor launches)
and one complete ResNet-50 b256 context (configs[2]: 105 tensors, 5.36 G elements, the
bench's batched launches, allocation and seeds). For every tensor the packed words, group
min and group scale are compared bit for bit with the oracle over the whole tensor, and
every decoded value is compared with the oracle's (<= 1 ulp, mismatches counted).

The oracle runs unchanged, partitioned over the host cores by group ranges (threads; ctypes
releases the GIL): quantize_codes_span computes a span's codes at their absolute element
indices, pack / unpack_dequantize work span-relative. Counts are written to
gpurun_out/everygroup_counts.json for DESIGN.md.
"""
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

TAGS = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}
G = 256
SPAN_GROUPS = 1 << 16  # 16 M elements per oracle work item
COUNTS = {}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gact():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2206_11357_b200 as g
    g.lib()
    return g


def _host_bits(t: torch.Tensor) -> np.ndarray:
    t = t.detach().contiguous().reshape(-1).cpu()
    if t.element_size() == 4:
        return t.view(torch.int32).numpy().view(np.uint32)
    return t.view(torch.int16).numpy().view(np.uint16)


def _ulp(a: np.ndarray, b: np.ndarray, width: int) -> np.ndarray:
    a = a.astype(np.int64)
    b = b.astype(np.int64)
    sign, mag = 1 << (width - 1), (1 << (width - 1)) - 1

    def key(v):
        return np.where(v & sign, -(v & mag), v & mag)
    return np.abs(key(a) - key(b))


def check_every_group(orc, x, ct, y, bits, seed, pool):
    """All groups of one tensor: returns (elements, code mismatches, y mismatches (<= 1 ulp))."""
    n = x.numel()
    tag = TAGS[x.dtype]
    xh = _host_bits(x)
    xh = xh.view(np.float32) if x.dtype == torch.float32 else xh
    words = _host_bits(ct.packed).view(np.uint32)
    mn_g = _host_bits(ct.group_min).view(np.uint32)
    sc_g = _host_bits(ct.group_scale).view(np.uint32)
    yh = _host_bits(y)
    width = 32 if y.dtype == torch.float32 else 16
    ng = (n + G - 1) // G
    wpg = G * bits // 32  # words per group (a group starts on a word boundary)

    def work(g0):
        g1 = min(ng, g0 + SPAN_GROUPS)
        lo, hi = g0 * G, min(n, g1 * G)
        q, mn, sc = orc.quantize_codes_span(xh[lo:hi], tag, n, G, bits, seed, g0, g1)
        ref_words = orc.pack(q, bits)
        got_words = words[g0 * wpg: g0 * wpg + ref_words.size]
        bad_codes = int(np.count_nonzero(got_words != ref_words))
        bad_stats = int(np.count_nonzero(mn_g[g0:g1] != mn.view(np.uint32)) +
                        np.count_nonzero(sc_g[g0:g1] != sc.view(np.uint32)))
        ref_y = orc.unpack_dequantize(ref_words, mn, sc, hi - lo, G, bits, TAGS[y.dtype])
        d = _ulp(yh[lo:hi], ref_y, width)
        return bad_codes, bad_stats, int(np.count_nonzero(d)), int(d.max(initial=0))

    res = list(pool.map(work, range(0, ng, SPAN_GROUPS)))
    bad_codes = sum(r[0] for r in res)
    bad_stats = sum(r[1] for r in res)
    y_mis = sum(r[2] for r in res)
    y_max = max(r[3] for r in res)
    assert bad_codes == 0, f"{bad_codes} packed words differ from the oracle"
    assert bad_stats == 0, f"{bad_stats} group min / scale values differ"
    assert y_max <= 1, f"decoded values up to {y_max} ulp from the oracle"
    return n, bad_codes, y_mis


def _record(key, n, bad, y_mis, dtype):
    c = COUNTS.setdefault(key, {"elements": 0, "code_word_mismatches": 0, "y_mismatches_1ulp": 0,
                                "y_dtype": str(dtype).replace("torch.", "")})
    c["elements"] += n
    c["code_word_mismatches"] += bad
    c["y_mismatches_1ulp"] += y_mis


@pytest.fixture(scope="module")
def pool():
    with ThreadPoolExecutor(max(1, os.cpu_count() or 1)) as ex:
        yield ex


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_buf256_every_group(gact, orc, pool, bits):
    spec = synth.workload_specs("buf256")[0]
    x = synth.make_tensor(spec, synth.DATA_SEED, "cuda", torch.bfloat16)
    seed = synth.tensor_seed(2022, 0)
    ct = gact.quantize_pack(x, bits, seed, G)
    y = ct.decompress()
    torch.cuda.synchronize()
    n, bad, y_mis = check_every_group(orc, x, ct, y, bits, seed, pool)
    _record(f"configs[1] buf256 b={bits}", n, bad, y_mis, y.dtype)


@pytest.mark.timeout(3600)
def test_resnet50_context_every_group(gact, orc, pool):
    """The whole bench context: tensors are generated, compressed in the bench's batched
    launches, decompressed, and checked one at a time against the oracle."""
    specs = synth.workload_specs("resnet50")
    D = np.array([s.numel for s in specs], dtype=np.int64)
    bits = gact.allocate_bits(synth.sensitivities(specs, seed=7), D, int(4.0 * D.sum()))
    seeds = [synth.tensor_seed(2022, i) for i in range(len(specs))]
    total = 0
    # batches of tensors (<= ~1.5 G elements resident at a time), each one batched launch
    batch, size = [], 0
    groups_of = []
    for i, s in enumerate(specs):
        batch.append(i)
        size += s.numel
        if size > 1_500_000_000 or i == len(specs) - 1:
            groups_of.append(batch)
            batch, size = [], 0
    for idx in groups_of:
        xs = [synth.make_tensor(specs[i], synth.DATA_SEED + i, "cuda", torch.bfloat16) for i in idx]
        cts = gact.quantize_pack_batch(xs, [int(bits[i]) for i in idx], [seeds[i] for i in idx], G)
        ys = gact.unpack_dequantize_batch(cts)
        torch.cuda.synchronize()
        for i, x, ct, y in zip(idx, xs, cts, ys):
            n, bad, y_mis = check_every_group(orc, x, ct, y, int(bits[i]), seeds[i], pool)
            _record("configs[2] resnet50 b256 context", n, bad, y_mis, y.dtype)
            total += n
        del xs, cts, ys
        torch.cuda.empty_cache()
    assert total == int(D.sum()) == 5_357_168_640


def test_write_counts():
    if not COUNTS:
        pytest.skip("no every-group test ran")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "everygroup_counts.json"), "w") as f:
        json.dump(COUNTS, f, indent=1)
    print(json.dumps(COUNTS))
