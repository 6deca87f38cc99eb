"""Randomised GPU parity (a fixed-seed fuzz over the whole argument space of include/gact.h):
random n (1 .. 300k), any group size (every multiple of 32 in [32, 4096]), dtype, bits, seed
and input recipe (normal with random scale, the edge groups, the mixed constant / exact-grid /
subnormal / signed-zero groups), single and batched calls, all against the oracle: codes and
group statistics bit-exact, decoded values within 1 ulp of the output dtype."""
import numpy as np
import pytest
import torch

import synth
from test_gpu_parity import (BITS, DTYPES, TAGS, check_dequantize, check_quantize, host_bits,
                             make_input, oracle_input, ulp_distance)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gact():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2206_11357_b200 as g
    g.lib()
    return g


def _case(rng):
    G = 32 * int(rng.integers(1, 129))
    if rng.random() < 0.5:  # half the cases on the specialised power-of-two kernels
        G = int(2 ** rng.integers(5, 13))
    n = int(rng.integers(1, 300_000)) if rng.random() < 0.8 else int(rng.integers(1, 2 * G + 9))
    dtype = DTYPES[int(rng.integers(0, 3))]
    bits = BITS[int(rng.integers(0, 4))]
    kind = ["normal", "edge2", "mixed"][int(rng.integers(0, 3))]
    seed = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
    return G, n, dtype, bits, kind, seed


@pytest.mark.parametrize("case", range(48))
def test_fuzz_single(gact, orc, case):
    rng = np.random.default_rng(9000 + case)
    G, n, dtype, bits, kind, seed = _case(rng)
    x = make_input(n, dtype, seed=case, kind=kind, group=G if kind == "edge2" else 256)
    ct, ref = check_quantize(gact, orc, x, G, bits, seed)
    ydt = DTYPES[int(rng.integers(0, 3))]
    check_dequantize(gact, orc, ct, ref, n, G, bits, ydt)


@pytest.mark.parametrize("case", range(8))
def test_fuzz_batched(gact, orc, case):
    """One group size per batch (the ABI's rule), everything else random per tensor."""
    rng = np.random.default_rng(7000 + case)
    G = _case(rng)[0]
    xs, bits, seeds = [], [], []
    for i in range(int(rng.integers(2, 60))):
        _, n, dtype, b, kind, seed = _case(rng)
        n = min(n, 120_000)
        xs.append(make_input(n, dtype, seed=100 * case + i, kind=kind, group=G if kind == "edge2" else 256))
        bits.append(b)
        seeds.append(seed)
    batch = gact.quantize_pack_batch(xs, bits, seeds, G)
    ys = gact.unpack_dequantize_batch(batch)
    torch.cuda.synchronize()
    for x, b, s, ct, y in zip(xs, bits, seeds, batch, ys):
        ref_p, ref_mn, ref_sc = orc.quantize_pack(oracle_input(x), TAGS[x.dtype], G, b, s)
        assert np.array_equal(host_bits(ct.packed), ref_p), (G, b, x.numel(), x.dtype)
        assert np.array_equal(host_bits(ct.group_min), ref_mn.view(np.uint32))
        assert np.array_equal(host_bits(ct.group_scale), ref_sc.view(np.uint32))
        ref_y = orc.unpack_dequantize(ref_p, ref_mn, ref_sc, x.numel(), G, b, TAGS[x.dtype])
        assert ulp_distance(host_bits(y), ref_y, 32 if x.dtype == torch.float32 else 16).max(initial=0) <= 1


def test_fuzz_seeds_are_independent_streams(gact):
    """Different seeds give different codes; equal seeds, equal codes (Alg. 1's replay)."""
    x = make_input(100_003, torch.bfloat16, seed=1)
    a = gact.quantize_pack(x, 4, synth.tensor_seed(5, 0))
    b = gact.quantize_pack(x, 4, synth.tensor_seed(5, 0))
    c = gact.quantize_pack(x, 4, synth.tensor_seed(5, 1))
    assert torch.equal(a.packed, b.packed)
    frac_diff = float((a.packed != c.packed).float().mean())
    assert frac_diff > 0.3
