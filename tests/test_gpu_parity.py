"""GPU parity: the CUDA path (through the C ABI, via the thin binding) against the CPU
oracle on the same seeded inputs.

Bar (BASELINE.json north_star): packed codes, group_min and group_scale BIT-EXACT;
dequantized values within 1 ulp of the output dtype (fp32 / bf16 / fp16); allocations
identical (tests/test_abi.py). Sizes span several tiles and a ragged tail; edge cases
cover empty / tiny / constant / subnormal / signed-zero / exact-grid groups, and every
group size 32..4096. Full-size workloads are checked on sampled groups in
tests/test_gpu_fullsize.py.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

TAGS = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}
DTYPES = [torch.float32, torch.bfloat16, torch.float16]
BITS = [1, 2, 4, 8]
GROUPS = [32, 64, 128, 256, 512, 1024, 2048, 4096]


@pytest.fixture(scope="module")
def gact():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2206_11357_b200 as g
    g.lib()
    return g


def host_bits(t: torch.Tensor) -> np.ndarray:
    """Raw bit patterns of a tensor as a host array (uint32 for fp32, uint16 otherwise)."""
    t = t.detach().contiguous().cpu()
    if t.dtype == torch.float32:
        return t.view(torch.int32).numpy().view(np.uint32).reshape(-1)
    if t.dtype in (torch.bfloat16, torch.float16):
        return t.view(torch.int16).numpy().view(np.uint16).reshape(-1)
    if t.dtype == torch.int32:
        return t.numpy().view(np.uint32).reshape(-1)
    raise TypeError(t.dtype)


def oracle_input(x: torch.Tensor) -> np.ndarray:
    b = host_bits(x)
    return b.view(np.float32) if x.dtype == torch.float32 else b


def ulp_distance(a: np.ndarray, b: np.ndarray, width: int) -> np.ndarray:
    """Distance in representable steps between two arrays of float bit patterns."""
    a = a.astype(np.int64)
    b = b.astype(np.int64)
    sign = 1 << (width - 1)
    mag = sign - 1

    def key(v):
        return np.where(v & sign, -(v & mag), v & mag)
    return np.abs(key(a) - key(b))


def check_quantize(gact, orc, x: torch.Tensor, G: int, bits: int, seed: int):
    ct = gact.quantize_pack(x, bits, seed, G)
    torch.cuda.synchronize()
    ref_p, ref_mn, ref_sc = orc.quantize_pack(oracle_input(x), TAGS[x.dtype], G, bits, seed)
    got_p = host_bits(ct.packed)
    assert got_p.size == ref_p.size
    bad = np.nonzero(got_p != ref_p)[0]
    assert bad.size == 0, f"{bad.size} packed words differ, first at word {bad[:5]}"
    assert np.array_equal(host_bits(ct.group_min), ref_mn.view(np.uint32))
    assert np.array_equal(host_bits(ct.group_scale), ref_sc.view(np.uint32))
    return ct, (ref_p, ref_mn, ref_sc)


def check_dequantize(gact, orc, ct, ref, n, G, bits, dtype):
    ref_p, ref_mn, ref_sc = ref
    y = gact.unpack_dequantize(ct.packed, ct.group_min, ct.group_scale, n, bits, G, dtype)
    torch.cuda.synchronize()
    ref_y = orc.unpack_dequantize(ref_p, ref_mn, ref_sc, n, G, bits, TAGS[dtype])
    d = ulp_distance(host_bits(y), ref_y, 32 if dtype == torch.float32 else 16)
    assert d.max(initial=0) <= 1, f"max ulp distance {d.max()}"
    c = DEQUANT_COUNTS.setdefault(str(dtype).replace("torch.", ""), [0, 0])
    c[0] += int((d != 0).sum())
    c[1] += int(d.size)
    return int((d != 0).sum())


DEQUANT_COUNTS = {}  # output dtype -> [values differing from the oracle (by 1 ulp), values checked]


def make_input(n, dtype, seed, kind="normal", group=256):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n) * 10.0 ** rng.uniform(-2, 2)
    if kind == "mixed" and n > 0:
        G = 256
        ng = (n + G - 1) // G
        for g in range(ng):
            sl = slice(g * G, min(n, (g + 1) * G))
            r = g % 6
            if r == 1:
                v[sl] = 3.25  # constant group
            elif r == 2:
                fits = dict(e_range=(-12, -2), m_range=64) if dtype == torch.float16 else {}
                v[sl] = synth.exact_grid_group(G, 2, rng, **fits)[: v[sl].size]
            elif r == 3:
                v[sl] = rng.integers(0, 5, v[sl].size) * 2.0 ** -149  # subnormal range
            elif r == 4:
                v[sl] = np.where(rng.random(v[sl].size) < 0.5, -0.0, 0.0)  # signed zeros only
            elif r == 5:  # the largest magnitudes the dtype holds without overflow
                big = 1e4 if dtype == torch.float16 else 1e30
                v[sl] = rng.standard_normal(v[sl].size) * big
    if kind == "edge2" and n > 0:
        return edge_groups(n, dtype, seed, group)
    t = torch.from_numpy(v.astype(np.float32)).to(dtype)
    return t.cuda()


def edge_groups(n, dtype, seed, G):
    """Groups (of G elements) that exercise the 2-byte paths at their edges, cycling through:
    subnormals only (bf16 k 2^-133, f16 k 2^-24; fp32 k 2^-149), subnormals with zeros of
    both signs, negative zeros only, values just below the largest finite (one sign per
    group, so that max - min stays finite), the smallest normals with subnormals, mixed signs
    of tiny magnitude, and a normal group. Values are exact in the dtype (bit patterns)."""
    rng = np.random.default_rng(seed)
    if dtype == torch.float32:
        sub, top, width = 2.0 ** -149, 3.0e38, 32
    elif dtype == torch.bfloat16:
        sub, top, width = 2.0 ** -133, 3.38e38, 16
    else:
        sub, top, width = 2.0 ** -24, 65504.0, 16
    nsub = 128 if dtype == torch.bfloat16 else (1024 if dtype == torch.float16 else 1 << 23)
    v = np.zeros(n, dtype=np.float64)
    ng = (n + G - 1) // G
    for g in range(ng):
        sl = slice(g * G, min(n, (g + 1) * G))
        m = v[sl].size
        r = g % 8
        if r == 0:
            v[sl] = rng.integers(0, nsub, m) * sub
        elif r == 1:
            v[sl] = rng.integers(-nsub + 1, nsub, m) * sub
            v[sl][rng.random(m) < 0.2] = -0.0
        elif r == 2:
            v[sl] = -0.0
        elif r == 3:
            v[sl] = top * (1 - rng.random(m) * 0.5)
        elif r == 4:
            v[sl] = -top * (1 - rng.random(m) * 0.5)
        elif r == 5:
            v[sl] = np.where(rng.random(m) < 0.5, rng.integers(0, nsub, m) * sub, 2.0 ** -126 if width == 32 or dtype == torch.bfloat16 else 2.0 ** -14)
        elif r == 6:
            v[sl] = rng.standard_normal(m) * sub * 3
        else:
            v[sl] = rng.standard_normal(m)
    if dtype == torch.float32:
        t = torch.from_numpy(v.astype(np.float32))
    elif dtype == torch.float16:
        t = torch.from_numpy(v.astype(np.float16))
    else:  # bf16: the subnormal / zero groups are exact; the others are rounded once to bf16
        t = torch.from_numpy(v.astype(np.float32)).to(torch.bfloat16)
    return t.cuda()


# ----------------------------------------------------------------------------- configs
def test_c1_config(gact, orc):
    """configs[0]: 4096 fp32, G=256, b=2, fixed seed (plus a constant and a grid group)."""
    x = torch.from_numpy(synth.c1_tensor(2, 256)).cuda()
    ct, ref = check_quantize(gact, orc, x, 256, 2, 0x5EED)
    assert check_dequantize(gact, orc, ct, ref, x.numel(), 256, 2, torch.float32) == 0
    # exact-grid group decodes bit-exactly (B3 on the grid)
    y = ct.decompress()
    assert torch.equal(y[5 * 256: 6 * 256], x[5 * 256: 6 * 256])
    assert torch.equal(y[3 * 256: 4 * 256], x[3 * 256: 4 * 256])


@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16", "f16"])
@pytest.mark.parametrize("bits", BITS)
@pytest.mark.parametrize("G", GROUPS)
def test_quantize_dequantize_parity(gact, orc, dtype, bits, G):
    TE = max(G, 256)
    # two of the largest CTA units (32768 elements: 8 warps x 16 chunks x 256 for 2-byte
    # inputs; the unguarded fast path of every kernel), then several tiles, a ragged tail and
    # a partial chunk (the guarded path)
    n = 2 * 32768 + 3 * TE + 8 * 5 + 3
    x = make_input(n, dtype, seed=G * 10 + bits)
    ct, ref = check_quantize(gact, orc, x, G, bits, seed=0xABCDEF0123456789 ^ (G * bits))
    for ydt in DTYPES:
        check_dequantize(gact, orc, ct, ref, n, G, bits, ydt)


GENERIC_GROUPS = [96, 160, 192, 224, 288, 320, 384, 480, 800, 1056, 2080, 4064]  # multiples of 32, not powers of two


@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16", "f16"])
@pytest.mark.parametrize("bits", BITS)
@pytest.mark.parametrize("G", GENERIC_GROUPS)
def test_generic_group_sizes(gact, orc, dtype, bits, G):
    """include/gact.h: any multiple of 32 in [32, 4096] is a group size. Those that are not
    powers of two (generic kernels: a warp per group; the dequantize group index by an exact
    reciprocal multiply) against the oracle: many groups, a short last group, a partial chunk,
    and the edge groups (subnormals, signed zeros, near-overflow)."""
    n = 37 * G + 3 * 8 + 5
    for kind in ("normal", "edge2"):
        x = make_input(n, dtype, seed=G * 13 + bits, kind=kind, group=G)
        ct, ref = check_quantize(gact, orc, x, G, bits, seed=0xC0DE0000 + G * 8 + bits)
        for ydt in DTYPES:
            check_dequantize(gact, orc, ct, ref, n, G, bits, ydt)
        mn, sc = gact.group_stats(x, bits, G)
        assert torch.equal(mn, ct.group_min) and torch.equal(sc, ct.group_scale)


@pytest.mark.parametrize("G", [96, 192, 352, 1056, 2080])
def test_generic_group_sizes_batched(gact, orc, G):
    """Batched launches with a generic G: 40 ragged tensors of mixed dtype and bits, each
    against the oracle (CTAs start at arbitrary tensors: binary-searched cursors). G = 96 /
    192: the super-tile kernel; 1056 / 2080: the register kernel (2-byte) and the two-pass
    kernel (fp32 at 2080)."""
    rng = np.random.default_rng(G)
    xs, bits, seeds = [], [], []
    for i in range(40):
        n = int(rng.integers(1, 30 * G))
        xs.append(make_input(n, DTYPES[i % 3], seed=2000 + i))
        bits.append(BITS[(i // 3) % 4])
        seeds.append(synth.tensor_seed(31, i))
    batch = gact.quantize_pack_batch(xs, bits, seeds, G)
    ys = gact.unpack_dequantize_batch(batch)
    torch.cuda.synchronize()
    for x, b, s, ct, y in zip(xs, bits, seeds, batch, ys):
        ref_p, ref_mn, ref_sc = orc.quantize_pack(oracle_input(x), TAGS[x.dtype], G, b, s)
        assert np.array_equal(host_bits(ct.packed), ref_p)
        assert np.array_equal(host_bits(ct.group_min), ref_mn.view(np.uint32))
        assert np.array_equal(host_bits(ct.group_scale), ref_sc.view(np.uint32))
        ref_y = orc.unpack_dequantize(ref_p, ref_mn, ref_sc, x.numel(), G, b, TAGS[x.dtype])
        assert ulp_distance(host_bits(y), ref_y, 32 if x.dtype == torch.float32 else 16).max(initial=0) <= 1


@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16", "f16"])
@pytest.mark.parametrize("bits", BITS)
@pytest.mark.parametrize("G", GROUPS)
def test_edge_groups_every_kernel(gact, orc, dtype, bits, G):
    """Subnormal, signed-zero and near-overflow groups through every kernel (all G, every b,
    every dtype), full units and a ragged tail: codes bit-exact, decoded values <= 1 ulp."""
    TE = max(G, 256)
    n = 2 * 32768 + 8 * TE + 77  # two of the largest CTA units (2-byte: 32768 elements), then a tail
    x = make_input(n, dtype, seed=G * 7 + bits, kind="edge2", group=G)
    hb = host_bits(x)
    if dtype != torch.float32:  # the inputs really are 2-byte subnormals / -0 / near-max
        assert np.any((hb & 0x7F80 if dtype == torch.bfloat16 else hb & 0x7C00) == 0)
        assert np.any(hb == 0x8000)
    ct, ref = check_quantize(gact, orc, x, G, bits, seed=0x5EED0000 + G + bits)
    for ydt in DTYPES:
        check_dequantize(gact, orc, ct, ref, n, G, bits, ydt)


@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16", "f16"])
@pytest.mark.parametrize("bits", BITS)
def test_edge_values(gact, orc, dtype, bits):
    """Constant groups, exact grids, subnormal ranges, signed zeros, 1e30 magnitudes."""
    n = 256 * 12 + 5
    x = make_input(n, dtype, seed=bits, kind="mixed")
    ct, ref = check_quantize(gact, orc, x, 256, bits, seed=bits * 1000003)
    assert check_dequantize(gact, orc, ct, ref, n, 256, bits, dtype) >= 0


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 31, 33, 255, 256, 257, 511, 1023, 1025])
@pytest.mark.parametrize("G", [32, 256, 2048])
def test_tiny_and_ragged_sizes(gact, orc, n, G):
    for bits in BITS:
        x = make_input(n, torch.bfloat16, seed=n + bits)
        ct, ref = check_quantize(gact, orc, x, G, bits, seed=n * 31 + bits)
        check_dequantize(gact, orc, ct, ref, n, G, bits, torch.float32)


def test_empty(gact):
    x = torch.empty(0, device="cuda", dtype=torch.bfloat16)
    ct = gact.quantize_pack(x, 2, 1)
    assert ct.packed.numel() == 0 and ct.group_min.numel() == 0
    y = ct.decompress()
    assert y.numel() == 0


def test_padding_words_are_zero(gact):
    """The unused high bits of the last packed word are zero (include/gact.h)."""
    for bits in BITS:
        for n in [1, 3, 5, 9, 17, 100]:
            x = make_input(n, torch.float32, seed=n)
            ct = gact.quantize_pack(x, bits, 7, 32)
            last = int(host_bits(ct.packed)[-1])
            used = n * bits - 32 * (ct.packed.numel() - 1)
            if used < 32:
                assert last >> used == 0


@pytest.mark.parametrize("G", [32, 256, 1024, 4096])
def test_group_stats_matches(gact, orc, G):
    for dtype in DTYPES:
        x = make_input(5 * max(G, 256) + 77, dtype, seed=G)
        for bits in BITS:
            mn, sc = gact.group_stats(x, bits, G)
            ct = gact.quantize_pack(x, bits, 3, G)
            rmn, rsc = orc.group_stats(oracle_input(x), TAGS[dtype], G, bits)
            assert np.array_equal(host_bits(mn), rmn.view(np.uint32))
            assert np.array_equal(host_bits(sc), rsc.view(np.uint32))
            assert torch.equal(mn, ct.group_min) and torch.equal(sc, ct.group_scale)


def test_determinism_and_streams(gact):
    x = make_input(1 << 20, torch.bfloat16, seed=5)
    a = gact.quantize_pack(x, 4, 99)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b = gact.quantize_pack(x, 4, 99)
    s.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(a.packed, b.packed) and torch.equal(a.group_scale, b.group_scale)
    c = gact.quantize_pack(x, 4, 100)
    assert not torch.equal(a.packed, c.packed)


@pytest.mark.parametrize("G", GROUPS)
def test_batch_equals_single(gact, G):
    """Batched launches (mixed dtypes and bits, > GACT_MAX_BATCH tensors) give results
    identical to one call per tensor."""
    rng = np.random.default_rng(G)
    xs, bits, seeds = [], [], []
    for i in range(300):
        n = int(rng.integers(1, 3000)) if i % 3 else int(rng.integers(1, 70000))
        dt = DTYPES[i % 3]
        xs.append(make_input(n, dt, seed=i))
        bits.append(BITS[int(rng.integers(0, 4))])
        seeds.append(synth.tensor_seed(11, i))
    batch = gact.quantize_pack_batch(xs, bits, seeds, G)
    ys = gact.unpack_dequantize_batch(batch)
    torch.cuda.synchronize()
    for x, b, s, ct, y in zip(xs, bits, seeds, batch, ys):
        single = gact.quantize_pack(x, b, s, G)
        assert torch.equal(ct.packed, single.packed)
        assert torch.equal(ct.group_min, single.group_min)
        assert torch.equal(ct.group_scale, single.group_scale)
        assert torch.equal(y.view(-1), single.decompress().view(-1))


@pytest.mark.parametrize("G", GROUPS + [96, 800])
def test_one_tensor_batch_vs_oracle(gact, orc, G):
    """A batch call holding one tensor of a (dtype, bits) class launches the single-tensor
    kernels (gact_host.cu, single_of): codes and decoded values against the oracle, at sizes
    whose last CTA unit is whole, partial by a few tiles, or partial inside its last tile."""
    te = max(G, 256)
    for k, n in enumerate([64 * te, 64 * te * 3 + 5 * te, 64 * te + 3 * te + 77, 1000]):
        dt = DTYPES[k % 3]
        b = BITS[k % 4]
        x = make_input(n, dt, seed=500 + k)
        s = synth.tensor_seed(41, k)
        ct = gact.quantize_pack_batch([x], [b], [s], G)[0]
        y = gact.unpack_dequantize_batch([ct])[0]
        torch.cuda.synchronize()
        ref_p, ref_mn, ref_sc = orc.quantize_pack(oracle_input(x), TAGS[dt], G, b, s)
        assert np.array_equal(host_bits(ct.packed), ref_p)
        assert np.array_equal(host_bits(ct.group_min), ref_mn.view(np.uint32))
        assert np.array_equal(host_bits(ct.group_scale), ref_sc.view(np.uint32))
        ref_y = orc.unpack_dequantize(ref_p, ref_mn, ref_sc, n, G, b, TAGS[dt])
        d = ulp_distance(host_bits(y), ref_y, 32 if dt == torch.float32 else 16)
        assert d.max(initial=0) <= 1


@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16", "f16"])
@pytest.mark.parametrize("G", [2048, 4096])
def test_batch_large_groups_vs_oracle(gact, orc, dtype, G):
    """Batched launches at G = 2048 / 4096 (the fp32 CTA-wide kernel, the 2-byte register
    and shared-memory-stage kernels) against the oracle, tensor by tensor. 40 ragged tensors
    per launch: every tensor ends in a partial group and is padded to 128 tiles, so guarded
    units interleave with full ones inside one CTA's sequence, and the launch has more units
    than its grid (CTAs wrap across tensor tails)."""
    rng = np.random.default_rng(G + TAGS[dtype])
    xs, bits, seeds = [], [], []
    for i in range(40):
        n = int(rng.integers(2 * G, 48 * G)) + int(rng.integers(1, G))
        xs.append(make_input(n, dtype, seed=1000 + i))
        bits.append(BITS[i % 4])
        seeds.append(synth.tensor_seed(29, i))
    batch = gact.quantize_pack_batch(xs, bits, seeds, G)
    ys = gact.unpack_dequantize_batch(batch)
    torch.cuda.synchronize()
    for x, b, s, ct, y in zip(xs, bits, seeds, batch, ys):
        ref_p, ref_mn, ref_sc = orc.quantize_pack(oracle_input(x), TAGS[dtype], G, b, s)
        assert np.array_equal(host_bits(ct.packed), ref_p)
        assert np.array_equal(host_bits(ct.group_min), ref_mn.view(np.uint32))
        assert np.array_equal(host_bits(ct.group_scale), ref_sc.view(np.uint32))
        ref_y = orc.unpack_dequantize(ref_p, ref_mn, ref_sc, x.numel(), G, b, TAGS[dtype])
        d = ulp_distance(host_bits(y), ref_y, 32 if dtype == torch.float32 else 16)
        assert d.max(initial=0) <= 1


def test_unbiased_on_gpu(gact, orc):
    """E[Q(x)] = x over 10^5 seeds of the C1 tensor: the GPU mean of
    the decoded values is within 4.5 sigma (+ the 2^-9 lattice bias, R4) of x, and the per-element
    variance never exceeds the paper's bound 1/4 range^2 S(b) = scale^2 / 4 (B2).
    Seeds are batched 256 per launch (one descriptor per seed, same input)."""
    G, bits, N, per = 256, 2, 100_000, 256
    xh = synth.c1_tensor(bits, G)
    x = torch.from_numpy(xh).cuda()
    n = x.numel()
    acc = torch.zeros(n, dtype=torch.float64, device="cuda")
    acc2 = torch.zeros_like(acc)
    done = 0
    while done < N:
        m = min(per, N - done)
        cts = gact.quantize_pack_batch([x] * m, [bits] * m, list(range(done, done + m)), G)
        ys = torch.stack(gact.unpack_dequantize_batch(cts)).double()
        acc += ys.sum(0)
        acc2 += (ys * ys).sum(0)
        done += m
    mean = (acc / N).cpu().numpy()
    var = (acc2 / N).cpu().numpy() - mean ** 2
    mn, sc = orc.group_stats(xh, 0, G, bits)
    scale = np.repeat(sc.astype(np.float64), G)[: n]
    lo = np.repeat(mn.astype(np.float64), G)[: n]
    t = np.where(scale > 0, (xh.astype(np.float64) - lo) / np.maximum(scale, 1e-300), 0.0)
    p = t - np.floor(t)
    sig = np.sqrt(np.maximum(p * (1 - p), 1e-12) / N) * scale
    tol = 4.5 * sig + (2.0 ** -9 + 1e-6) * scale + 4 * np.spacing(np.abs(xh)).astype(np.float64)
    assert np.all(np.abs(mean - xh) <= tol)
    assert np.all(var <= scale ** 2 / 4 * (1 + 6 / np.sqrt(N)) + 1e-30)


@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16", "f16"])
def test_sq_diff_sum(gact, orc, dtype):
    """||a - b||^2 (Alg. 1's reduction, NEXT-3) vs the oracle (long double, index order):
    relative difference <= n 2^-52 (summation order only); bit-reproducible run to run."""
    for n in [0, 1, 7, 8, 1000, 1 << 20, (1 << 22) + 13]:
        a = make_input(n, dtype, seed=n + 1)
        b = make_input(n, dtype, seed=n + 2)
        got = gact.sq_diff_sum(a, b)
        again = gact.sq_diff_sum(a, b)
        torch.cuda.synchronize()
        ref = orc.sq_diff_sum(oracle_input(a), oracle_input(b), TAGS[dtype])
        g = float(got.item())
        assert g == float(again.item())
        assert abs(g - ref) <= max(n, 1) * 2.0 ** -52 * abs(ref) + 1e-300


@pytest.mark.parametrize("bits", BITS)
def test_dequant_narrow_and_wide_paths_agree(gact, bits):
    """The 256-bit-store path (y 32-byte, packed 16-byte aligned) and the ABI's 16-byte path
    (taken for less-aligned buffers) write identical values."""
    for dtype in DTYPES:
        n = 256 * 40 + 77
        x = make_input(n, dtype, seed=bits)
        ct = gact.quantize_pack(x, bits, 5, 256)
        wide = ct.decompress().reshape(-1)
        es = torch.tensor([], dtype=dtype).element_size()
        pad = 16 // es                                   # 16-byte offset: not 32-byte aligned
        ybuf = torch.empty(n + pad, dtype=dtype, device="cuda")
        pbuf = torch.zeros(ct.packed.numel() + 2, dtype=torch.int32, device="cuda")
        pbuf[2:] = ct.packed                             # 8-byte offset: not 16-byte aligned
        narrow = gact.unpack_dequantize(pbuf[2:], ct.group_min, ct.group_scale, n, bits, 256, dtype,
                                        out=ybuf[pad:])
        torch.cuda.synchronize()
        assert torch.equal(narrow, wide)


@pytest.mark.parametrize("bits", BITS)
@pytest.mark.parametrize("G", [32, 256, 1024])
def test_threshold_ties(gact, orc, bits, G):
    """T + u exactly on an integer and one fp32 step either side (tests/tie_cases.py): the
    GPU's rounding shortcuts for the exact floor(T + u) (fma.rm for b = 8, fma.rn on the
    2^-16 grid for b <= 4; R5) agree with the oracle and the closed form, on the
    unguarded fast path (>= 2 CTA units) and a ragged tail."""
    import tie_cases
    seed = 0x5EED0000 + G * 16 + bits
    ng = max(2 * 32768 // G, 2) + 3
    xh, want = tie_cases.tie_groups(ng, G, bits, seed, orc.rand8, np.random.default_rng(G + bits))
    xh = xh[: xh.size - 5]  # ragged tail: the last group is short
    want = want[: xh.size]
    x = torch.from_numpy(xh).cuda()
    ct, ref = check_quantize(gact, orc, x, G, bits, seed)
    q = orc.unpack(host_bits(ct.packed), xh.size, bits).astype(np.int64)
    assert np.array_equal(q, want)


def test_concurrent_host_threads(gact):
    """The C ABI is stateless and thread-safe (include/gact.h): four host threads, each on its
    own stream, compress and decompress their tensors repeatedly (G = 2048 bf16 exercises the
    shared-memory kernel whose attribute is set once per device) and get exactly the results
    of a single-threaded call."""
    import threading
    cases = [(make_input(200_000 + 4099 * i, (torch.bfloat16, torch.float32)[i % 2], seed=40 + i),
              (1, 2, 4, 8)[i], 1000 + i, (2048, 256, 32, 4096)[i]) for i in range(4)]
    ref = []
    for x, b, s, G in cases:
        ct = gact.quantize_pack(x, b, s, G)
        ref.append((ct.packed.clone(), ct.group_min.clone(), ct.group_scale.clone(), ct.decompress().clone()))
    torch.cuda.synchronize()
    errors = []

    def work(k):
        try:
            x, b, s, G = cases[k]
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(20):
                    ct = gact.quantize_pack(x, b, s, G)
                    y = ct.decompress()
            st.synchronize()
            p, mn, sc, yr = ref[k]
            if not (torch.equal(ct.packed, p) and torch.equal(ct.group_min, mn)
                    and torch.equal(ct.group_scale, sc) and torch.equal(y, yr)):
                errors.append(f"thread {k}: results differ")
        except Exception as e:  # surfaced below
            errors.append(f"thread {k}: {e!r}")
    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("nblk", [4, 8])
@pytest.mark.parametrize("shared", [1, 0], ids=["shared_rounds", "plain"])
def test_philox_blocks_at_counter_boundaries(gact, orc, shared, nblk):
    """The device generator (include/gact_testing.h) at the counters where the batched
    kernels' shared-round Philox form (N = 4 fp32, N = 8 bf16/fp16 blocks per lane) switches
    to its fallback (lo32(blk) + 32 (N - 1) wrapping) and across the 2^32 carry into the
    counter's high word, against the oracle's Philox4x32-10."""
    L = gact.lib()
    out = torch.zeros(4 * nblk, dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(7)
    seeds = [0, 0x5EED, 0xFFFFFFFFFFFFFFFF, int(rng.integers(0, 2**63))]
    top = 2**32
    edge = 32 * (nblk - 1)
    blks = [0, 1, 31, 32, 96, 224, top - 300, top - edge - 2, top - edge - 1, top - edge, top - edge + 1,
            top - 97, top - 96, top - 95, top - 33, top - 32, top - 1, top, top + 5, 5 * top - edge,
            2**40 - edge - 1, 2**63 + 12345] + [int(v) for v in rng.integers(0, 2**62, 8)]
    for seed in seeds:
        for blk in blks:
            assert L.gact_test_philox_blocks(blk, seed, shared, nblk, out.data_ptr(), None) == 0
            torch.cuda.synchronize()
            got = out.cpu().numpy().view(np.uint32)
            for m in range(nblk):
                b = (blk + 32 * m) % 2**64
                ref = orc.philox4x32_10([b & 0xFFFFFFFF, b >> 32, 0, 0], [seed & 0xFFFFFFFF, seed >> 32])
                assert np.array_equal(got[4 * m: 4 * m + 4], ref), (hex(blk), m, hex(seed))


def test_binding_rejects_bad_buffers(gact):
    """Caller-supplied outputs are checked before any launch (size, dtype, device,
    contiguity): a short or strided buffer raises instead of being written out of bounds."""
    x = make_input(10000, torch.bfloat16, seed=1)
    ct = gact.quantize_pack(x, 4, 1)
    short = torch.empty(ct.packed.numel() - 1, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        gact.quantize_pack(x, 4, 1, out=(short, ct.group_min, ct.group_scale))
    with pytest.raises(ValueError):
        gact.quantize_pack(x, 4, 1, out=(ct.packed, ct.group_min.double(), ct.group_scale))
    with pytest.raises(ValueError):
        gact.unpack_dequantize(ct.packed, ct.group_min, ct.group_scale, 10000, 4,
                               out=torch.empty(9999, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(ValueError):
        gact.unpack_dequantize(ct.packed, ct.group_min, ct.group_scale, 10000, 4,
                               out=torch.empty(20000, dtype=torch.float32, device="cuda")[::2])
    with pytest.raises(ValueError):  # codes too short for n
        gact.unpack_dequantize(ct.packed[:-1], ct.group_min, ct.group_scale, 10000, 4)
    y = gact.unpack_dequantize(ct.packed, ct.group_min, ct.group_scale, 10000, 4, dtype=torch.bfloat16)
    assert torch.equal(y, ct.decompress())


def test_zz_report_dequant_mismatch_counts():
    """Runs last in this file: the dequantize mismatch counts of every check above, per output
    dtype (written to gpurun_out/dequant_counts.json and quoted in DESIGN.md)."""
    import json
    import os
    if not DEQUANT_COUNTS:
        pytest.skip("no dequantize check ran")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    os.makedirs(os.path.join(root, "gpurun_out"), exist_ok=True)
    with open(os.path.join(root, "gpurun_out", "dequant_counts.json"), "w") as f:
        json.dump(DEQUANT_COUNTS, f)
    print("dequantize mismatches (1 ulp) / values:", DEQUANT_COUNTS)


@pytest.mark.parametrize("G", [32, 96, 256, 1056, 2048, 4064, 4096])
def test_every_output_word_is_written(gact, orc, G):
    """Output buffers pre-filled with ones: after one call every packed word (including the
    zero padding of the last one) and every group statistic equals the oracle's, for every
    kernel family and a ragged n (no word may be left unwritten)."""
    for dtype in DTYPES:
        for bits in BITS:
            n = 3 * max(G, 256) + 8 * 7 + 3
            x = make_input(n, dtype, seed=G + bits)
            packed = torch.full((gact.packed_words(n, bits),), -1, dtype=torch.int32, device="cuda")
            mn = torch.full((gact.num_groups(n, G),), float("nan"), device="cuda")
            sc = torch.full_like(mn, float("nan"))
            gact.quantize_pack(x, bits, 77, G, out=(packed, mn, sc))
            torch.cuda.synchronize()
            ref_p, ref_mn, ref_sc = orc.quantize_pack(oracle_input(x), TAGS[dtype], G, bits, 77)
            assert np.array_equal(host_bits(packed), ref_p), (dtype, bits)
            assert np.array_equal(host_bits(mn), ref_mn.view(np.uint32))
            assert np.array_equal(host_bits(sc), ref_sc.view(np.uint32))
