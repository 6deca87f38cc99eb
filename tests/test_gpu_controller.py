"""The GACT controller on CUDA through libgact (NEXT-1 of SURVEY §8f): saved-tensor capture
(P:545), the filters and dedup, Alg. 1, the bit allocation
(P:534), and the properties the paper relies on:

* all-32 scheme == plain backward (lossless path);
* the AC gradient of a linear map is unbiased, E_Q[g(Q(h))] = g(h);
* Alg. 1's c_l agrees with the brute-force Var_Q[g] / S(b_l) per tensor (SPEC acceptance 5);
* adaptive bits give a gradient variance no larger than uniform bits at the same budget
  (Fig. 4(b); SPEC acceptance 7);
* the context shrinks >= 6x at 4 bits on fp32 (the abstract's "up to 8.1x", SPEC acc. 12).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctl():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2206_11357_b200 as g
    g.lib()
    from paper_2206_11357_b200 import controller
    return controller


def mlp(widths, act=torch.nn.Tanh, seed=0):
    torch.manual_seed(seed)
    layers = []
    for a, b in zip(widths[:-1], widths[1:]):
        layers += [torch.nn.Linear(a, b), act()]
    return torch.nn.Sequential(*layers[:-1]).cuda()


def fwdbwd(model, x, y):
    def f():
        torch.nn.functional.cross_entropy(model(x), y).backward()
    return f


def grads(model):
    return torch.cat([p.grad.reshape(-1) for p in model.parameters()])


def test_all_raw_equals_plain(ctl):
    m = mlp([64, 256, 256, 10])
    x, y = torch.randn(512, 64, device="cuda"), torch.randint(0, 10, (512,), device="cuda")
    fwdbwd(m, x, y)()
    ref = grads(m).clone()
    c = ctl.Controller(m, avg_bits=32, ladder=(32,), merge=False, adapt_interval=10**9)
    c.iteration = 1
    c.iterate(fwdbwd(m, x, y))
    assert torch.equal(grads(m), ref)
    assert c.stats.packed == 0


def test_linear_gradient_unbiased(ctl):
    """out = W2 h with h = W1 x; loss = <out, R>: grad W2 = R^T h is linear in the saved h,
    so its expectation over the compressor is exact (P:381 / eqn:first-order P:389-398)."""
    torch.manual_seed(3)
    lin1 = torch.nn.Linear(128, 256, bias=False).cuda()
    lin2 = torch.nn.Linear(256, 64, bias=False).cuda()
    m = torch.nn.Sequential(lin1, lin2)
    x = torch.randn(512, 128, device="cuda")
    R = torch.randn(512, 64, device="cuda")

    def f():
        (m(x) * R).sum().backward()
    f()
    exact = lin2.weight.grad.double().clone()
    c = ctl.Controller(m, avg_bits=2, ladder=(2,), merge=False, adapt_interval=10**9, seed=11)
    c.iteration = 1
    N = 400
    acc = torch.zeros_like(exact)
    acc2 = torch.zeros_like(exact)
    for _ in range(N):
        c.iterate(f)
        g = lin2.weight.grad.double()
        acc += g
        acc2 += g * g
    mean = acc / N
    sd = (acc2 / N - mean ** 2).clamp(min=0).sqrt()
    z = (mean - exact).abs() / (sd / np.sqrt(N) + 1e-12)
    assert c.stats.packed >= N
    assert float((z > 5).float().mean()) < 1e-3      # 5-sigma excursions essentially absent
    assert float(z.mean()) < 1.0                      # |N(0,1)| has mean 0.8
    assert not torch.equal(g, exact)                  # compression did perturb each draw


def _bruteforce_c(ctl, m, f, L, b, draws=48):
    """Var_Q[g] / S(b) per slot: compress every slot at b with FIXED seeds, except slot l whose
    seed varies over `draws` draws (the quantity Alg. 1 estimates)."""
    c = ctl.Controller(m, merge=False, adapt_interval=10**9)
    c._bits_override = lambda s: b
    out = []
    for l in range(L):
        gs = []
        for d in range(draws):
            c._seed_of = (lambda s, l=l, d=d: 1000 + s if s != l else 10**6 + d)
            gs.append(c._run(f))
        G = torch.stack(gs).double()
        out.append(float(G.var(dim=0, unbiased=True).sum()) / (1.0 / (2 ** b - 1) ** 2))
    return np.array(out)


def test_alg1_matches_bruteforce(ctl):
    m = mlp([32, 256, 256, 256, 8], seed=5)
    x, y = torch.randn(1024, 32, device="cuda"), torch.randint(0, 8, (1024,), device="cuda")
    f = fwdbwd(m, x, y)
    c = ctl.Controller(m, merge=False, adapt_interval=10**9, est_bits=4, seed=2)
    est = c.estimate_sensitivity(f, repeats=12)
    L = len(c.numel)
    assert L >= 4
    bf = _bruteforce_c(ctl, m, f, L, 4)
    r = np.corrcoef(np.log(est), np.log(bf))[0, 1]
    assert r > 0.9, (est, bf)
    assert np.all(np.abs(est / bf - 1) < 0.5), (est, bf)


def test_adaptive_no_worse_than_uniform(ctl):
    """Fig. 4(b) analog: with a sensitive head, the greedy scheme at an average of 4 bits
    has no larger gradient variance than uniform 4 bits (same budget)."""
    m = mlp([32, 512, 512, 512, 16], seed=9)
    x, y = torch.randn(2048, 32, device="cuda"), torch.randint(0, 16, (2048,), device="cuda")
    f = fwdbwd(m, x, y)
    ad = ctl.Controller(m, avg_bits=4, ladder=(1, 2, 4, 8), merge=False, adapt_interval=10**9, seed=4)
    bits = ad.adapt(f, repeats=4)
    D = np.array(ad.numel)
    assert (np.array(bits) * D).sum() <= 4 * D.sum()

    def variance(scheme, draws=32):
        c = ctl.Controller(m, merge=False, adapt_interval=10**9)
        c._bits_override = lambda s: scheme[s]
        gs = []
        for d in range(draws):
            c._seed_of = (lambda s, d=d: 7919 * d + s)
            gs.append(c._run(f))
        return float(torch.stack(gs).double().var(dim=0).sum())
    v_ad = variance(bits)
    v_un = variance([4] * len(bits))
    assert v_ad <= v_un * 1.05, (bits, v_ad, v_un)


def test_dedup_and_ratio(ctl):
    """Q/K/V share their input: one compression per iteration; the compressed
    context at 4 bits is >= 6x smaller than fp32 (abstract: up to 8.1x)."""
    torch.manual_seed(0)
    d = 256
    q, k, v, o = (torch.nn.Linear(d, d).cuda() for _ in range(4))
    params = torch.nn.ModuleList([q, k, v, o])
    x = torch.randn(1024, d, device="cuda")

    def f():
        h = torch.tanh(q.weight[:1].sum() * 0 + x)   # h depends on parameters -> requires grad
        a = torch.tanh(q(h)) * torch.sigmoid(k(h)) + torch.relu(v(h))
        o(a).pow(2).mean().backward()
    c = ctl.Controller(params, avg_bits=4, ladder=(4,), merge=False, adapt_interval=10**9)
    c.iteration = 1
    c.iterate(f)
    assert c.stats.dedup_hits >= 2
    assert c.compression_ratio() >= 6.0


def _linear_closed_form(orc, h, R, bits, G=256):
    """Alg. 1's c for out = h W^T with loss <out, R> (one compressed context tensor h,
    grad W = R^T h, linear in h): E||g0 - g1||^2 = 2 sum_{i,j} Var_Q[(R^T Q(h))_{ij}] with
    Var_Q[Q(h)_{bj}] = p (1 - p) scale^2 per element (independent elements, B1/B2 P:477-480),
    p = frac(T), T = (h - mn) / scale from the oracle's group statistics (p agrees with the
    generator's exact probability to 2^-9, R4). Returns (c, sigma of one Alg. 1 estimate): the
    estimate's variance 2 sum_j tr(C_j^2) / (2 S)^2 with C_j = R^T diag(2 v_.j) R."""
    hh = h.detach().cpu().numpy().astype(np.float32)
    mn, sc = orc.group_stats(hh.reshape(-1), orc.F32, G, bits)
    mn = np.repeat(mn.astype(np.float64), G)[: hh.size].reshape(hh.shape)
    sc = np.repeat(sc.astype(np.float64), G)[: hh.size].reshape(hh.shape)
    T = np.where(sc > 0, (hh.astype(np.float64) - mn) / np.where(sc > 0, sc, 1), 0.0)
    p = T - np.floor(T)
    v = p * (1 - p) * sc * sc                         # [B, K]
    Rn = R.detach().cpu().numpy().astype(np.float64)  # [B, O]
    S = orc.S(bits)
    c = float(((Rn * Rn).sum(1)[:, None] * v).sum()) / S
    var_sq = 0.0
    for j in range(v.shape[1]):
        C = Rn.T @ (2 * v[:, j:j + 1] * Rn)           # covariance of (g0 - g1)_{., j}
        var_sq += 2 * float(np.sum(C * C))
    return c, np.sqrt(var_sq) / (2 * S)


@pytest.mark.parametrize("est_bits", [2, 4, 8])
def test_alg1_closed_form_linear(ctl, orc, est_bits):
    """Alg. 1 pinned to a closed form: for a linear layer the controller's c
    (averaged over 24 independent seed draws) equals the exact compression variance of the
    weight gradient / S(b) within 5 standard deviations of the estimator."""
    torch.manual_seed(11)
    lin = torch.nn.Linear(512, 16, bias=False).cuda()
    h = torch.randn(256, 512, device="cuda").mul_(torch.rand(256, 1, device="cuda") * 3).requires_grad_(True)
    R = torch.randn(256, 16, device="cuda")

    def f():
        (lin(h) * R).sum().backward()
    c = ctl.Controller(lin, merge=False, adapt_interval=10**9, est_bits=est_bits, seed=7, min_numel=1)
    reps = 24
    est = c.estimate_sensitivity(f, repeats=reps)
    assert len(c.numel) == 1 and c.numel[0] == h.numel()   # the one context tensor: h
    exact, sigma = _linear_closed_form(orc, h, R, est_bits)
    assert abs(est[0] - exact) <= 5 * sigma / np.sqrt(reps), (est[0], exact, sigma)
    assert sigma / np.sqrt(reps) < 0.02 * exact              # the pin is tight (< 2% per sigma)


def test_alert_calibrated_linear(ctl, orc):
    """When compression is the only gradient noise (fixed batch, fixed weights), the running
    gradient variance estimate Var[g_hat] and the predicted V(b) = sum_l c_l S(b_l) agree
    (ratio ~ 1), so the default threshold (1/2) fires."""
    torch.manual_seed(12)
    lin = torch.nn.Linear(512, 16, bias=False).cuda()
    h = torch.randn(256, 512, device="cuda").requires_grad_(True)
    R = torch.randn(256, 16, device="cuda")

    def f():
        (lin(h) * R).sum().backward()
    c = ctl.Controller(lin, avg_bits=2, ladder=(2,), merge=False, adapt_interval=10**9, seed=3, min_numel=1)
    with pytest.warns(RuntimeWarning):
        for _ in range(60):
            c.iterate(f)
    ratios = [V / var for (_, V, var) in c.stats.variance_log[20:]]
    assert 0.7 < float(np.median(ratios)) < 1.4, ratios
    exact, _ = _linear_closed_form(orc, h, R, 2)
    assert abs(c.predicted_variance() / (exact * orc.S(2)) - 1) < 0.25


def test_failure_alert(ctl):
    """P:536-537 at the default threshold: a 1-bit budget with a tiny batch warns (compression
    dominates the gradient noise)."""
    m = mlp([16, 256, 256, 4], seed=1)
    x, y = torch.randn(64, 16, device="cuda"), torch.randint(0, 4, (64,), device="cuda")
    c = ctl.Controller(m, avg_bits=1, ladder=(1,), merge=False, adapt_interval=10**9)
    assert c.alert_ratio == 0.5
    with pytest.warns(RuntimeWarning):
        for _ in range(16):
            c.iterate(fwdbwd(m, x, y))
    assert c.stats.alerts


def test_no_alert_at_8_bits_training(ctl):
    """...and stays silent at 8 bits on the convergence task (fresh minibatches, SGD steps),
    where compression noise is a small part of the gradient noise."""
    import warnings
    g = torch.Generator(device="cuda").manual_seed(0)
    centers = torch.randn(16, 64, device="cuda", generator=g) * 1.5
    m = mlp([64, 512, 512, 16], act=torch.nn.ReLU, seed=1)
    opt = torch.optim.SGD(m.parameters(), lr=0.05, momentum=0.9)
    c = ctl.Controller(m, avg_bits=8, ladder=(8,), merge=False, adapt_interval=50, seed=3)
    with warnings.catch_warnings():
        warnings.simplefilter("error", RuntimeWarning)
        for it in range(120):
            y = torch.randint(0, 16, (512,), device="cuda", generator=g)
            x = centers[y] + torch.randn(512, 64, device="cuda", generator=g)
            c.iterate(fwdbwd(m, x, y))
            opt.step()
    assert not c.stats.alerts
    ratios = [V / var for (_, V, var) in c.stats.variance_log[10:] if var > 0]
    assert max(ratios) < c.alert_ratio and float(np.median(ratios)) < 0.1, ratios


def test_swap_prefetch_same_gradients_less_memory(ctl):
    """with swap, the compressed context is parked in pinned host memory during
    forward and prefetched on a side stream in backward: identical gradients (same seeds),
    less device memory held at the end of forward."""
    m = mlp([256, 2048, 2048, 2048, 16], seed=3)
    x, y = torch.randn(4096, 256, device="cuda"), torch.randint(0, 16, (4096,), device="cuda")
    peak = {}
    ctrls = {}

    def f_for(tag):
        def f():
            torch.cuda.synchronize()
            start = torch.cuda.memory_allocated()
            loss = torch.nn.functional.cross_entropy(m(x), y)
            ctrls[tag].flush()                     # swap-outs done: device copies released
            torch.cuda.synchronize()
            peak[tag] = torch.cuda.memory_allocated() - start   # context held by forward
            loss.backward()
        return f
    out = {}
    for swap in (False, True):
        c = ctl.Controller(m, avg_bits=4, ladder=(4,), merge=False, adapt_interval=10**9, seed=5, swap=swap)
        ctrls[swap] = c
        c.iteration = 1
        c.iterate(f_for(swap))
        torch.cuda.synchronize()
        out[swap] = grads(m).cpu()  # keep device memory comparable between the two runs
    assert torch.equal(out[False], out[True])
    assert peak[True] < 0.5 * peak[False]


def test_checkpoint_segments_cb1(ctl):
    """CB1: inside torch.utils.checkpoint segments only the segment inputs are
    saved in forward; the controller compresses them, and the activations re-saved during
    the backward recomputation go through the same hooks. All-32: bit-identical gradients to
    the plain checkpointed model; 4 bits: a finite, close gradient."""
    from torch.utils.checkpoint import checkpoint
    torch.manual_seed(0)
    blocks = torch.nn.ModuleList([torch.nn.Sequential(torch.nn.Linear(256, 256), torch.nn.Tanh()) for _ in range(4)]).cuda()
    head = torch.nn.Linear(256, 8).cuda()
    model = torch.nn.ModuleList([blocks, head])
    x, y = torch.randn(1024, 256, device="cuda", requires_grad=True), torch.randint(0, 8, (1024,), device="cuda")

    def f():
        h = x
        for b in blocks:
            # reentrant checkpointing: the recomputation runs inside backward under the
            # controller's saved-tensor hooks (the non-reentrant form keeps its recomputed
            # activations in its own storage, out of the hooks' reach)
            h = checkpoint(b, h, use_reentrant=True)
        torch.nn.functional.cross_entropy(head(h), y).backward()
    for p in model.parameters():
        p.grad = None
    f()
    ref = torch.cat([p.grad.reshape(-1) for p in model.parameters()]).clone()
    raw = ctl.Controller(model, avg_bits=32, ladder=(32,), merge=False, adapt_interval=10**9)
    raw.iteration = 1
    raw.iterate(f)
    assert torch.equal(torch.cat([p.grad.reshape(-1) for p in model.parameters()]), ref)
    c = ctl.Controller(model, avg_bits=4, ladder=(4,), merge=False, adapt_interval=10**9)
    c.iteration = 1
    c.iterate(f)
    g = torch.cat([p.grad.reshape(-1) for p in model.parameters()])
    assert c.stats.packed > 0 and torch.isfinite(g).all()
    assert float((g - ref).norm() / ref.norm()) < 0.2


class _RecordingBackend:
    """The libgact backend, recording each compression (input copy, bits, seed, result)."""

    def __init__(self, group_size=256):
        from paper_2206_11357_b200.controller import LibgactBackend
        self.inner = LibgactBackend(group_size)
        self.calls = []
        self.phase = "forward"

    def compress(self, t, bits, seed):
        ct = self.inner.compress(t, bits, seed)
        self.calls.append((self.phase, t.detach().clone(), bits, seed, ct))
        return ct

    def decompress(self, h):
        return self.inner.decompress(h)

    def nbytes(self, h):
        return self.inner.nbytes(h)

    def sq_diff(self, a, b):
        return self.inner.sq_diff(a, b)


def test_checkpoint_cb1_codes_match_oracle(ctl, orc):
    """CB1 against the oracle: every tensor the controller compresses under
    checkpoint segments -- the segment inputs saved in forward and the activations re-saved
    while backward recomputes the segments -- is compressed with the slot's bits and seed,
    and its codes, group min and scale equal the oracle's for that input, bits and seed."""
    from torch.utils.checkpoint import checkpoint
    torch.manual_seed(0)
    blocks = torch.nn.ModuleList([torch.nn.Sequential(torch.nn.Linear(256, 256), torch.nn.Tanh())
                                  for _ in range(3)]).cuda()
    head = torch.nn.Linear(256, 8).cuda()
    model = torch.nn.ModuleList([blocks, head])
    x, y = torch.randn(512, 256, device="cuda", requires_grad=True), torch.randint(0, 8, (512,), device="cuda")
    rec = _RecordingBackend()

    def f():
        rec.phase = "forward"
        h = x
        for b in blocks:
            h = checkpoint(b, h, use_reentrant=True)
        loss = torch.nn.functional.cross_entropy(head(h), y)
        rec.phase = "backward"
        loss.backward()
    c = ctl.Controller(model, avg_bits=4, ladder=(2, 4, 8), merge=False, adapt_interval=10**9, backend=rec,
                       min_numel=1)
    c.bits = [2, 4, 8] * 8
    c.iteration = 1
    c.iterate(f)
    phases = [ph for ph, *_ in rec.calls]
    assert phases.count("forward") >= 1 and phases.count("backward") >= 1, phases
    torch.cuda.synchronize()
    c.iteration -= 1  # the seeds of the iteration just run
    for slot, (ph, t, bits, seed, ct) in enumerate(rec.calls):
        assert bits == c.bits[slot] and seed == c._slot_seed(slot)
        xh = t.contiguous().cpu().numpy().reshape(-1)
        p, mn, sc = orc.quantize_pack(xh, orc.F32, 256, bits, seed)
        assert np.array_equal(ct.packed.cpu().numpy().view(np.uint32), p), (slot, ph)
        assert np.array_equal(ct.group_min.cpu().numpy(), mn)
        assert np.array_equal(ct.group_scale.cpu().numpy(), sc)


def test_training_converges_like_fp32(ctl):
    """§6.2 analog (SPEC acceptance 8): an MLP trained with the compressed context (adaptive
    bits, average 4 and 2) reaches the accuracy of uncompressed training on a synthetic
    Gaussian-mixture task (same initialisation, data order and steps)."""
    def run(avg_bits):
        g = torch.Generator(device="cuda").manual_seed(0)
        centers = torch.randn(16, 64, device="cuda", generator=g) * 1.5
        def batch():
            y = torch.randint(0, 16, (512,), device="cuda", generator=g)
            return centers[y] + torch.randn(512, 64, device="cuda", generator=g), y
        m = mlp([64, 512, 512, 16], act=torch.nn.ReLU, seed=1)
        # lr 0.02: at 0.05 a 1-bit allocation diverges in 2 of 4 controller seeds with the 16-bit
        # generator of round 1 and with the 8-bit one alike (tools/dbg_train.py); at 0.02 and 0.01
        # every seed (3-8) converges to accuracy 1.0
        opt = torch.optim.SGD(m.parameters(), lr=0.02, momentum=0.9)
        c = None if avg_bits is None else ctl.Controller(m, avg_bits=avg_bits, ladder=(1, 2, 4, 8), merge=False,
                                                         adapt_interval=100, seed=3)
        for it in range(300):
            x, y = batch()
            f = fwdbwd(m, x, y)
            if c is None:
                opt.zero_grad()
                f()
            else:
                c.iterate(f)
            opt.step()
        x, y = batch()
        with torch.no_grad():
            return float((m(x).argmax(1) == y).float().mean())
    acc32, acc4, acc2 = run(None), run(4), run(2)
    assert acc32 > 0.9
    assert acc4 >= acc32 - 0.015, (acc32, acc4)
    assert acc2 >= acc32 - 0.03, (acc32, acc2)


def test_resnet18_context(ctl):
    """A torchvision ResNet-18 (conv, BN, in-place ReLU, max-pool with int64 indices kept raw)
    under the controller. Gradients stay aligned with the uncompressed ones and the error
    shrinks with the bits (ReLU backward masks with the SAVED result, a nonlinear use of the
    context: values within one step of 0 may decode to 0, so the error is not zero-mean)."""
    torchvision = pytest.importorskip("torchvision")
    torch.manual_seed(0)
    m = torchvision.models.resnet18(num_classes=10).cuda().train()
    x = torch.randn(32, 3, 64, 64, device="cuda")
    y = torch.randint(0, 10, (32,), device="cuda")
    f = fwdbwd(m, x, y)
    m.zero_grad()
    f()
    ref = grads(m).clone()
    err, cos = {}, {}
    for b in (4, 8):
        c = ctl.Controller(m, avg_bits=b, ladder=(b,), merge=False, adapt_interval=10**9)
        c.iteration = 1
        c.iterate(f)
        g = grads(m)
        err[b] = float((g - ref).norm() / ref.norm())
        cos[b] = float(torch.nn.functional.cosine_similarity(g, ref, dim=0))
        assert c.stats.packed > 20 and c.stats.raw > 0
        assert c.compression_ratio() > (32 / (b + 0.25)) * 0.9
    assert err[8] < err[4] and cos[8] > 0.97 and cos[4] > 0.5, (err, cos)


def test_alg1_fixes_dropout_noise(ctl):
    """Alg. 1 fixes every source of randomness except Q^(l): with dropout in the
    model, two passes with the same compressor seeds give bit-identical gradients, so
    ||g0 - g1||^2 holds compression noise only, and the estimate is reproducible."""
    torch.manual_seed(3)
    m = torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Dropout(0.5),
                            torch.nn.Linear(256, 10)).cuda()
    x, y = torch.randn(256, 64, device="cuda"), torch.randint(0, 10, (256,), device="cuda")
    c = ctl.Controller(m, avg_bits=4, merge=False, adapt_interval=10**9)
    f = fwdbwd(m, x, y)
    c1 = c.estimate_sensitivity(f)
    c2 = c.estimate_sensitivity(f)
    assert np.array_equal(c1, c2)
    rng = c._rng_snapshot()
    c._seed_of = lambda s: 1000 + s
    g0 = c._run(f, rng)
    g0b = c._run(f, rng)
    c._seed_of = None
    assert torch.equal(g0, g0b)


def test_controller_offset_views(ctl):
    """Saved tensors that are views with a storage offset breaking 16-byte alignment (x[1:])
    are compressed (the binding copies them once) instead of failing with ALIGNMENT."""
    import paper_2206_11357_b200 as gact
    base = torch.randn(4097, 64, device="cuda")
    v = base[1:]  # offset 64 floats: aligned; a 1-element offset is not
    w = base.view(-1)[1:1 + 4096 * 63]
    for t in (v, w):
        ct = gact.quantize_pack(t, 4, 5)
        ref = gact.quantize_pack(t.clone(), 4, 5)
        assert torch.equal(ct.packed, ref.packed) and torch.equal(ct.group_min, ref.group_min)
    torch.manual_seed(0)
    lin = torch.nn.Linear(63, 10).cuda()
    xb = torch.randn(300 * 63 + 1, device="cuda", requires_grad=True)

    def f():
        lin(xb[1:].view(300, 63)).square().sum().backward()
    c = ctl.Controller(lin, avg_bits=4, merge=False, adapt_interval=10**9, min_numel=1)
    c.iteration = 1
    c.iterate(f)
    assert c.stats.packed >= 1 and torch.isfinite(lin.weight.grad).all()
