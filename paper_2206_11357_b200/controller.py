"""The GACT controller (§5): activation-compressed training on top of
the libgact C ABI.

  ctrl = Controller(model, avg_bits=4)           # P:571 "initialize the GACT controller"
  def fwdbwdprop():                              # P:571-573 "instruct GACT how to perform
      loss = loss_fn(model(x), y)                #  forward and backward propagation"
      loss.backward()
  ctrl.iterate(fwdbwdprop)                       # one training iteration (compressed context)
  optimizer.step()

* Capture: PyTorch saved-tensor hooks; pack_hook compresses every saved
  context tensor, unpack_hook decompresses it in backward.
* Filter: parameters (recorded data pointers) and tensors that do not require
  gradients are kept as they are.
* Dedup: a tensor saved by several ops (e.g. Q/K/V inputs) is compressed once per
  iteration; the footprint is (data pointer, storage offset, shape, strides, version) plus a
  weak reference to the first saver's tensor, so that a new tensor that reuses a freed
  tensor's memory is never mistaken for it.
* Bits (eqn:ilp P:471-475, greedy P:534): every `adapt_interval` iterations Alg. 1
   estimates c_l for each context slot l from two gradient evaluations whose
  compressor seeds differ only for tensor l, c_l = 1/2 ||g0 - g1||^2 / S(b_l); the
  sensitivities are merged across data-parallel ranks (dist.merge_sensitivities) and the
  greedy allocator of libgact assigns b_l under the budget avg_bits * sum_l D_l, with the
  ladder {1, 2, 4, 8, 32} (32 = keep uncompressed).
* Swap / prefetch (optional `swap=True`): compressed tensors are copied to pinned
  host memory on a swap-out stream right after compression (their device memory is released
  once the copy is done); in backward, decompressing slot l first issues the host-to-device
  copy of slot l - 1 (the next one backward needs) on a swap-in stream, and CUDA events
  order the streams.
* Failure alert: the predicted compression variance V = sum_l c_l S(b_l) is
  compared with the running variance of the gradient; a warning is raised when V is more
  than alert_ratio (default 1/2) of it, i.e. when compression dominates the gradient noise.

Slots are identified by the order in which distinct context tensors are first saved in an
iteration (a static graph saves the same tensors in the same order every iteration).
All compression arithmetic runs in libgact's kernels; this module only routes tensors.
"""
from __future__ import annotations

import math
import warnings
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import dist as gdist
from . import variance_factor

SUPPORTED = (torch.float32, torch.bfloat16, torch.float16)
LADDER = (1, 2, 4, 8, 32)
RAW = 32


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & (2**64 - 1)
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    return x ^ (x >> 31)


class LibgactBackend:
    """Compression through libgact (the product path; CUDA tensors only)."""

    def __init__(self, group_size: int = 256):
        from . import quantize_pack  # noqa: F401  (loads libgact: fails loudly if missing)
        self.group_size = group_size

    def compress(self, t: torch.Tensor, bits: int, seed: int):
        from . import quantize_pack
        return quantize_pack(t, bits, seed, self.group_size)

    def decompress(self, handle) -> torch.Tensor:
        return handle.decompress()

    def nbytes(self, handle) -> int:
        return handle.nbytes()

    def sq_diff(self, a: torch.Tensor, b: torch.Tensor) -> float:
        from . import sq_diff_sum
        return float(sq_diff_sum(a, b).item())


class SwappedTensor:
    """A compressed tensor parked in pinned host memory."""
    __slots__ = ("host", "meta", "done", "dev", "ready")

    def __init__(self, ct, swap_out: torch.cuda.Stream, pending: list):
        cur = torch.cuda.current_stream(ct.packed.device)
        swap_out.wait_stream(cur)                      # the codes are written
        self.meta = (ct.shape, ct.dtype, ct.bits, ct.group_size, ct.seed, ct.packed.device)
        dev = (ct.packed, ct.group_min, ct.group_scale)
        with torch.cuda.stream(swap_out):
            self.host = tuple(torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in dev)
            for h, d in zip(self.host, dev):
                h.copy_(d, non_blocking=True)
            self.done = torch.cuda.Event()
            self.done.record(swap_out)
        pending.append((self.done, dev))               # device copies live until the D2H is done
        self.dev = None
        self.ready = None

    def prefetch(self, swap_in: torch.cuda.Stream):
        if self.dev is not None:
            return
        swap_in.wait_event(self.done)
        with torch.cuda.stream(swap_in):
            self.dev = tuple(h.to(self.meta[5], non_blocking=True) for h in self.host)
            self.ready = torch.cuda.Event()
            self.ready.record(swap_in)

    def decompress(self, swap_in: torch.cuda.Stream) -> torch.Tensor:
        from . import CompressedTensor
        self.prefetch(swap_in)
        cur = torch.cuda.current_stream(self.meta[5])
        cur.wait_event(self.ready)
        for t in self.dev:
            t.record_stream(cur)
        shape, dtype, bits, G, seed, _ = self.meta
        return CompressedTensor(*self.dev, shape, dtype, bits, G, seed).decompress()


@dataclass
class Stats:
    packed: int = 0          # context tensors compressed
    raw: int = 0             # context tensors kept (filtered or at 32 bits)
    dedup_hits: int = 0      # repeated saves of an already-compressed tensor
    bytes_raw: int = 0       # bytes the compressed tensors would have taken
    bytes_compressed: int = 0
    alerts: list = field(default_factory=list)
    variance_log: list = field(default_factory=list)  # (iteration, V(b), Var[g_hat]) per iteration


class Controller:
    def __init__(self, model: torch.nn.Module, avg_bits: float = 4.0, group_size: int = 256,
                 ladder=LADDER, adapt_interval: int = 100, est_bits: int = 4, seed: int = 0,
                 min_numel: int = 256, alert_ratio: float = 0.5, backend=None, merge=True,
                 swap: bool = False):
        self.model = model
        self.avg_bits = float(avg_bits)
        self.ladder = tuple(int(b) for b in ladder)
        self.adapt_interval = int(adapt_interval)
        self.est_bits = int(est_bits)
        self.seed = int(seed)
        self.min_numel = int(min_numel)
        self.alert_ratio = float(alert_ratio)
        self.merge = merge
        self.backend = backend if backend is not None else LibgactBackend(group_size)
        self.param_ptrs = {p.data_ptr() for p in model.parameters()}
        self.bits: list[int] = []        # b_l per slot (empty until the first adaptation)
        self.numel: list[int] = []       # D_l per slot
        self.sensitivity: np.ndarray | None = None
        self.iteration = 0
        self.stats = Stats()
        self._seen: dict = {}
        self._slot = 0
        self._seed_of = None             # slot -> seed override (Alg. 1)
        self._bits_override = None       # slot -> bits override (Alg. 1 estimation scheme)
        self._grad_mean = None
        self._grad_sq = None
        self._grad_count = 0
        self._grad_w2 = 1.0
        self.swap = swap
        self._swapped: dict = {}         # slot -> SwappedTensor (this iteration)
        self._pending: list = []         # (event, device tensors) of swap-outs in flight
        if swap:
            self._swap_out = torch.cuda.Stream()
            self._swap_in = torch.cuda.Stream()

    # ---------------------------------------------------------------- capture hooks
    def _footprint(self, t: torch.Tensor):
        return (t.data_ptr(), t.storage_offset(), tuple(t.shape), tuple(t.stride()), t._version)

    def _slot_bits(self, slot: int) -> int:
        if self._bits_override is not None:
            return self._bits_override(slot)
        if slot < len(self.bits):
            return self.bits[slot]
        # before the first adaptation: the uniform scheme at the budget
        below = [b for b in self.ladder if b != RAW and b <= self.avg_bits]
        return max(below) if below else min(self.ladder)

    def _slot_seed(self, slot: int) -> int:
        if self._seed_of is not None:
            return self._seed_of(slot)
        return _splitmix64(_splitmix64(self.seed * 1_000_003 + self.iteration) ^ slot)

    def pack_hook(self, t: torch.Tensor):
        if (t.dtype not in SUPPORTED or not t.requires_grad or t.numel() < self.min_numel
                or t.data_ptr() in self.param_ptrs):
            self.stats.raw += 1
            return ("raw", t)
        fp = self._footprint(t)
        hit = self._seen.get(fp)
        if hit is not None and hit[0]() is not None:
            # same footprint AND the first saver's tensor still alive: the very same tensor
            # (a freed tensor's memory may be reused by a new one with the same footprint)
            self.stats.dedup_hits += 1
            return hit[1]
        slot = self._slot
        self._slot += 1
        if slot >= len(self.numel):
            self.numel.append(t.numel())
        b = self._slot_bits(slot)
        if b == RAW:
            h = ("raw", t)
            self.stats.raw += 1
        else:
            ct = self.backend.compress(t, b, self._slot_seed(slot))
            if self.swap:
                self._release_swapped()
                st = SwappedTensor(ct, self._swap_out, self._pending)
                self._swapped[slot] = st
                h = ("s", st, t.shape, t.dtype, slot)
            else:
                h = ("q", ct, t.shape, t.dtype)
            self.stats.packed += 1
            self.stats.bytes_raw += t.numel() * t.element_size()
            self.stats.bytes_compressed += self.backend.nbytes(ct)
        self._seen[fp] = (weakref.ref(t), h)
        return h

    def _release_swapped(self, wait: bool = False):
        """Drop the device copies of compressed tensors whose swap-out copy has finished."""
        keep = []
        for ev, dev in self._pending:
            if wait:
                ev.synchronize()
            elif not ev.query():
                keep.append((ev, dev))
        self._pending = keep

    def flush(self):
        """Wait for every swap-out and release the device copies (swap mode)."""
        self._release_swapped(wait=True)

    def unpack_hook(self, h):
        if h[0] == "raw":
            return h[1]
        if h[0] == "s":
            prev = self._swapped.get(h[4] - 1)        # backward visits slots in reverse
            if prev is not None:
                prev.prefetch(self._swap_in)
            return h[1].decompress(self._swap_in).view(h[2])
        return self.backend.decompress(h[1]).view(h[2])

    def hooks(self):
        """Context manager installing the pack / unpack hooks ("install hooks")."""
        self._seen = {}
        self._slot = 0
        self._swapped = {}
        return torch.autograd.graph.saved_tensors_hooks(self.pack_hook, self.unpack_hook)

    # ---------------------------------------------------------------- gradients
    def _params(self):
        return [p for p in self.model.parameters() if p.requires_grad]

    def _run(self, fwdbwdprop, rng=None) -> torch.Tensor:
        """One fwd+bwd under compression; returns the flattened fp32 gradient. `rng` (a
        snapshot from _rng_snapshot) is restored first, so that every pass of Alg. 1 draws
        the same dropout masks / stochastic-layer noise."""
        if rng is not None:
            self._rng_restore(rng)
        for p in self._params():
            p.grad = None
        with self.hooks():
            fwdbwdprop()
        self._seen = {}
        grads = [p.grad.reshape(-1).float() for p in self._params() if p.grad is not None]
        return torch.cat(grads) if grads else torch.zeros(0)

    @staticmethod
    def _rng_snapshot():
        cuda = torch.cuda.get_rng_state_all() if torch.cuda.is_available() else None
        return torch.get_rng_state(), cuda

    @staticmethod
    def _rng_restore(snap):
        cpu, cuda = snap
        torch.set_rng_state(cpu)
        if cuda is not None:
            torch.cuda.set_rng_state_all(cuda)

    # ---------------------------------------------------------------- Alg. 1
    def estimate_sensitivity(self, fwdbwdprop, repeats: int = 1) -> np.ndarray:
        """Alg. 1: c_l = 1/2 ||g0 - g1||^2 / S(b_l), where g0 seeds every Q^(l)
        with r_l and g1 re-seeds only Q^(l) with r_{L+1}. The estimation scheme compresses
        every slot at est_bits (Alg. 1 accepts any scheme b; under the linearisation c_l does
        not depend on b). Averaged over `repeats` seed draws."""
        saved_params = [p.grad for p in self._params()]
        # Alg. 1 fixes every source of randomness except Q^(l): all passes start
        # from one snapshot of the torch generators (dropout masks identical in g0 and g1).
        rng = self._rng_snapshot()
        L = len(self.numel)
        if L == 0:  # discover the slots with one pass
            self._bits_override = lambda s: self.est_bits
            self._run(fwdbwdprop, rng)
            self._bits_override = None
            L = len(self.numel)
        c = np.zeros(L)
        b_est = self.est_bits
        s_est = variance_factor(b_est)
        self._bits_override = lambda s: b_est
        try:
            for rep in range(repeats):
                base = _splitmix64(self.seed ^ 0xA5A5A5A5 ^ (self.iteration << 20) ^ rep)
                r = [_splitmix64(base + l + 1) for l in range(L + 1)]        # r_1 .. r_{L+1}
                self._seed_of = lambda s: r[s] if s < L else r[L]
                g0 = self._run(fwdbwdprop, rng)
                for l in range(L):
                    self._seed_of = (lambda s, l=l: r[L] if s == l else (r[s] if s < L else r[L]))
                    g1 = self._run(fwdbwdprop, rng)
                    c[l] += 0.5 * self.backend.sq_diff(g0, g1) / s_est
        finally:
            self._seed_of = None
            self._bits_override = None
            self._rng_restore(rng)
            for p, g in zip(self._params(), saved_params):
                p.grad = g
        return c / repeats

    def adapt(self, fwdbwdprop, repeats: int = 1) -> list[int]:
        """Refresh c (Alg. 1), merge it across ranks, and re-solve eqn:ilp."""
        from . import allocate_bits
        c = self.estimate_sensitivity(fwdbwdprop, repeats)
        if self.merge:
            c = gdist.merge_sensitivities(c, self.model_device())
        self.sensitivity = c
        D = np.asarray(self.numel, dtype=np.int64)
        B = int(self.avg_bits * D.sum())
        self.bits = [int(b) for b in allocate_bits(c, D, B, self.ladder)]
        if self.merge:
            gdist.assert_same_allocation(self.bits, self.model_device())
        return self.bits

    def model_device(self):
        for p in self.model.parameters():
            return p.device
        return torch.device("cpu")

    def predicted_variance(self) -> float:
        """V(b) <= sum_l c_l S(b_l) (eqn:var-decomposition)."""
        if self.sensitivity is None or not self.bits:
            return float("nan")
        return float(sum(c * variance_factor(b) for c, b in zip(self.sensitivity, self.bits)))

    # ---------------------------------------------------------------- training iteration
    def iterate(self, fwdbwdprop):
        """One iteration (Fig. 2 "Line 19"): adapt every adapt_interval iterations, then run
        fwdbwdprop with the compressed context; the parameters' .grad hold the AC gradient."""
        if self.iteration % self.adapt_interval == 0:
            self.adapt(fwdbwdprop)
        for p in self._params():
            p.grad = None
        with self.hooks():
            fwdbwdprop()
        self._seen = {}
        self._track_variance()
        self.iteration += 1

    def gradient_variance(self) -> float:
        """Var[g_hat] summed over coordinates, from the running (exponentially weighted) mean
        and second moment of the AC gradient over iterations ("maintaining a running
        mean of the gradient"), with the weights' bias correction: for weights w_t summing to
        1, E[sum_t w_t g_t^2 - (sum_t w_t g_t)^2] = (1 - sum_t w_t^2) Var[g]."""
        if self._grad_mean is None or self._grad_count < 2:
            return float("nan")
        raw = float((self._grad_sq - self._grad_mean ** 2).clamp_(min=0).sum().item())
        return raw / max(1e-12, 1.0 - self._grad_w2)

    def _track_variance(self, momentum: float = 0.9):
        """Running mean / second moment of the gradient; alert when the predicted compression
        variance V(b) = sum_l c_l S(b_l) is a large share of the gradient variance Var[g_hat]
        (P:536-537). Var[g_hat] includes the compression noise itself, so V / Var[g_hat] <= 1
        when c is accurate, and the default threshold alert_ratio = 0.5 reads "compression is
        the larger part of the gradient noise". No alert before 1 / (1 - momentum) tracked
        iterations (the running estimate needs that many samples)."""
        grads = [p.grad.reshape(-1).float() for p in self._params() if p.grad is not None]
        if not grads:
            return
        g = torch.cat(grads)
        a = 1.0 - momentum
        if self._grad_mean is None:
            self._grad_mean, self._grad_sq = g.clone(), (g * g)
            self._grad_count, self._grad_w2 = 1, 1.0
            return
        self._grad_mean.mul_(momentum).add_(g, alpha=a)
        self._grad_sq.mul_(momentum).add_(g * g, alpha=a)
        self._grad_count += 1
        self._grad_w2 = momentum * momentum * self._grad_w2 + a * a
        var = self.gradient_variance()
        V = self.predicted_variance()
        self.stats.variance_log.append((self.iteration, V, var))
        if self._grad_count < round(1.0 / a):
            return
        if var > 0 and not math.isnan(V) and V / var > self.alert_ratio:
            msg = (f"GACT: predicted compression variance {V:.3g} is more than {self.alert_ratio} x the "
                   f"gradient variance {var:.3g}; raise the bit budget")
            self.stats.alerts.append((self.iteration, V, var))
            warnings.warn(msg, RuntimeWarning, stacklevel=3)

    def compression_ratio(self) -> float:
        return self.stats.bytes_raw / max(1, self.stats.bytes_compressed)
