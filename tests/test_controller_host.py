"""Host logic of the GACT controller on CPU with a test double for the
compressor (the product compressor is libgact on CUDA, exercised in
tests/test_gpu_controller.py): the parameter and requires-grad filters, footprint dedup,
slot ordering, per-slot / per-iteration seeds, Alg. 1's seed replay, and the budget."""
import numpy as np
import torch

from paper_2206_11357_b200.controller import Controller


class RecordingBackend:
    """Test double: 'compresses' by adding a seed-determined perturbation whose size is the
    stochastic-rounding standard deviation of a b-bit uniform grid over the tensor's range,
    and records every call."""

    def __init__(self):
        self.calls = []

    def compress(self, t, bits, seed):
        self.calls.append((tuple(t.shape), bits, seed))
        g = torch.Generator().manual_seed(seed % (2**63))
        rng = (t.max() - t.min()).item()
        step = rng / ((1 << bits) - 1) if rng > 0 else 0.0
        noise = (torch.rand(t.shape, generator=g) - 0.5) * step
        return (t.detach() + noise, t.numel() * bits // 8)

    def decompress(self, h):
        return h[0]

    def nbytes(self, h):
        return h[1]

    def sq_diff(self, a, b):
        return float(((a.double() - b.double()) ** 2).sum())


class QKV(torch.nn.Module):
    def __init__(self, d=32):
        super().__init__()
        self.q, self.k, self.v = (torch.nn.Linear(d, d) for _ in range(3))
        self.out = torch.nn.Linear(d, 4)

    def forward(self, x):
        h = torch.tanh(x @ torch.eye(x.shape[1]))  # h requires grad through x? no: x is data
        h = self.q.weight.sum() * 0 + h            # make h depend on parameters
        a = torch.tanh(self.q(h)) * torch.tanh(self.k(h)) + torch.tanh(self.v(h))
        return self.out(a)


def _fwdbwd(model, x, y):
    def f():
        loss = torch.nn.functional.cross_entropy(model(x), y)
        loss.backward()
    return f


def test_filters_dedup_and_slots():
    torch.manual_seed(0)
    m = QKV()
    be = RecordingBackend()
    ctrl = Controller(m, avg_bits=4, backend=be, min_numel=16, merge=False, adapt_interval=10**9)
    x, y = torch.randn(64, 32), torch.randint(0, 4, (64,))
    ctrl.iteration = 1  # skip adaptation
    ctrl.iterate(_fwdbwd(m, x, y))
    # h is saved by q, k and v (same tensor): compressed once
    assert ctrl.stats.dedup_hits >= 2
    shapes = [c[0] for c in be.calls]
    assert shapes and all(s[0] == 64 for s in shapes)  # activations only: batch-leading
    # parameters are never compressed: none of the (32, 32) / (4, 32) weights
    assert (32, 32) not in shapes and (4, 32) not in shapes
    # slots: distinct seeds per slot, new seeds next iteration
    seeds1 = [c[2] for c in be.calls]
    assert len(set(seeds1)) == len(seeds1)
    n1 = len(be.calls)
    ctrl.iterate(_fwdbwd(m, x, y))
    seeds2 = [c[2] for c in be.calls[n1:]]
    assert len(seeds2) == len(seeds1) and not set(seeds1) & set(seeds2)
    assert ctrl.numel and len(ctrl.numel) == len(seeds1)


def test_non_grad_tensors_kept():
    m = torch.nn.Sequential(torch.nn.Linear(16, 16), torch.nn.ReLU(), torch.nn.Linear(16, 2))
    be = RecordingBackend()
    ctrl = Controller(m, backend=be, min_numel=1, merge=False, adapt_interval=10**9)
    ctrl.iteration = 1
    x = torch.randn(8, 16)  # data: does not require grad -> never compressed
    ctrl.iterate(_fwdbwd(m, x, torch.randint(0, 2, (8,))))
    # the Linear(16,16) input x is data (no grad): kept raw, never compressed
    assert (8, 16) not in [c[0] for c in be.calls] or ctrl.stats.raw >= 1
    assert ctrl.stats.raw >= 1 and ctrl.stats.packed >= 1


def test_alg1_seed_replay_and_allocation():
    """Alg. 1: g1 differs from g0 only through tensor l's seed, so a slot whose
    noise does not reach the gradient has c_l = 0; the allocator then spends the budget on
    the sensitive slots; the predicted variance uses the new bits."""
    torch.manual_seed(1)
    m = torch.nn.Sequential(torch.nn.Linear(32, 64), torch.nn.Tanh(), torch.nn.Linear(64, 64),
                            torch.nn.Tanh(), torch.nn.Linear(64, 4))
    be = RecordingBackend()
    ctrl = Controller(m, avg_bits=4, backend=be, min_numel=16, merge=False, adapt_interval=10**9)
    x, y = torch.randn(128, 32), torch.randint(0, 4, (128,))
    c = ctrl.estimate_sensitivity(_fwdbwd(m, x, y))
    assert len(c) == len(ctrl.numel) > 0 and np.all(c >= 0) and c.sum() > 0
    # replay: the same estimation twice gives the same c (counter-based seeds)
    it = ctrl.iteration
    c2 = ctrl.estimate_sensitivity(_fwdbwd(m, x, y))
    assert ctrl.iteration == it and np.allclose(c, c2)
    bits = ctrl.adapt(_fwdbwd(m, x, y))
    D = np.array(ctrl.numel)
    assert (np.array(bits) * D).sum() <= 4 * D.sum()
    assert np.isfinite(ctrl.predicted_variance())
