"""Seeded synthetic inputs shared by the tests, the bench and the oracle runs.

This module holds NO arithmetic of the method (no min/max, quantization, packing, Philox
or allocation). It only draws input tensors and sensitivity vectors, with the shapes of
the paper's workloads and the value distributions stated there:

  C1  one fp32 tensor of 4096 elements, N(0,1), with one constant group and one group on
      an exact b-bit grid (BASELINE.json configs[0]).
  C2  one 256 MiB bf16 buffer (2^27 elements), N(0,1) (configs[1]).
  C3  ResNet-50 batch 256 @224 context: 105 tensors (synth/shapes.json, enumerated by
      tools/enumerate_shapes.py with GACT's filters P:579-584) (configs[2]).
  C4  BERT-large seq 512 batch 64: 12 context tensors per layer (configs[3]).
  C5  GCN on an ogbn-arxiv-shaped graph (N = 169,343, hidden 256, 3 layers) and Swin-T
      batch 128: 154 tensors (configs[4]).

Distributions by the op that produced the tensor: BN inputs (conv outputs) per-channel
N(mu_c, sigma_c), mu_c ~ N(0, 0.5), sigma_c ~ LogU(0.1, 2); ReLU / max-pool outputs
max(0, N(0,1)); softmax rows of N(0, 2^2) logits; dropout(softmax) zeroes 10% and rescales
by 1/0.9; LayerNorm inputs Student-t(4) with 2 of every 1024 channels scaled by 20; the
loss head log_softmax of N(0, 2^2) logits; everything else N(0,1).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
DATA_SEED = 1234

BERT_HEADS, BERT_SEQ, BERT_HIDDEN, BERT_FFN = 16, 512, 1024, 4096
GCN_NODES, GCN_HIDDEN, GCN_CLASSES = 169_343, 256, 40


@dataclass(frozen=True)
class TensorSpec:
    name: str
    shape: tuple
    kind: str  # distribution tag, see module docstring

    @property
    def numel(self) -> int:
        return int(math.prod(self.shape))


def _shapes():
    with open(os.path.join(_HERE, "shapes.json")) as f:
        return json.load(f)


_KIND_BY_OP = {
    "ConvolutionBackward0": "bn_input",
    "ReluBackward0": "relu",
    "MaxPool2DWithIndicesBackward0": "relu",
    "ViewBackward0": "normal",
    "LogSoftmaxBackward0": "log_softmax",
    "SoftmaxBackward0": "softmax",
    "AddBackward0": "ln_input",
    "NativeLayerNormBackward0": "normal",
}


def resnet50_specs(batch: int = 256):
    """C3: the 105 context tensors of ResNet-50 (App. A.1 of SURVEY.md)."""
    out = []
    for i, e in enumerate(_shapes()["resnet50"]):
        shape = (e["shape"][0] * batch,) + tuple(e["shape"][1:])
        kind = _KIND_BY_OP.get(e["op"], "normal")
        if e["op"] == "ViewBackward0":
            kind = "relu"  # the flattened average-pool output is non-negative
        out.append(TensorSpec(f"resnet50.{i}.{e['op']}", shape, kind))
    return out


def swin_t_specs(batch: int = 128):
    """C5 (second half): the 154 context tensors of Swin-T."""
    out = []
    for i, e in enumerate(_shapes()["swin_t"]):
        shape = (e["shape"][0] * batch,) + tuple(e["shape"][1:])
        out.append(TensorSpec(f"swin_t.{i}.{e['op']}", shape, _KIND_BY_OP.get(e["op"], "normal")))
    return out


def bert_layer_specs(batch: int = 64, layers: int = 1):
    """C4: per layer, the 12 context tensors of a BERT-large encoder layer (App. A.2)."""
    B, S, H, NH, F = batch, BERT_SEQ, BERT_HIDDEN, BERT_HEADS, BERT_FFN
    per_layer = [
        ("x", (B, S, H), "ln_input"), ("q", (B, NH, S, H // NH), "normal"),
        ("k_t", (B, NH, H // NH, S), "normal"), ("v", (B, NH, S, H // NH), "normal"),
        ("attn_softmax", (B, NH, S, S), "softmax"), ("attn_dropout", (B, NH, S, S), "softmax_dropout"),
        ("context", (B, S, H), "normal"), ("ln1_in", (B, S, H), "ln_input"),
        ("ln1_out", (B, S, H), "normal"), ("gelu_in", (B, S, F), "normal"),
        ("gelu_out", (B, S, F), "relu"), ("ln2_in", (B, S, H), "ln_input"),
    ]
    return [TensorSpec(f"bert.l{l}.{n}", s, k) for l in range(layers) for (n, s, k) in per_layer]


def gcn_specs():
    """C5 (first half): 3-layer GCN, hidden 256, ogbn-arxiv-shaped node count."""
    N, Hd = GCN_NODES, GCN_HIDDEN
    out = []
    for l in range(2):
        out += [TensorSpec(f"gcn.l{l}.bn_in", (N, Hd), "bn_input"),
                TensorSpec(f"gcn.l{l}.relu_out", (N, Hd), "relu"),
                TensorSpec(f"gcn.l{l}.dropout_out", (N, Hd), "dropout_relu")]
    out.append(TensorSpec("gcn.out.log_softmax", (N, GCN_CLASSES), "log_softmax"))
    return out


def workload_specs(name: str):
    if name == "resnet50":
        return resnet50_specs(256)
    if name == "bert_layer":
        return bert_layer_specs(64, 1)
    if name == "bert24":
        return bert_layer_specs(64, 24)
    if name == "gcn":
        return gcn_specs()
    if name == "swin_t":
        return swin_t_specs(128)
    if name == "gcn_swin":
        return gcn_specs() + swin_t_specs(128)
    if name == "buf256":
        return [TensorSpec("buffer.256MiB", (1 << 27,), "normal")]
    raise KeyError(name)


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def make_tensor(spec: TensorSpec, seed: int, device="cpu", dtype=torch.float32) -> torch.Tensor:
    """Draw one tensor of `spec` with torch's generator on `device` (seeded)."""
    g = _gen(device, seed)
    shape = spec.shape
    kw = dict(device=device, dtype=torch.float32, generator=g)
    k = spec.kind
    if k == "normal":
        x = torch.randn(shape, **kw)
    elif k == "relu":
        x = torch.randn(shape, **kw).clamp_(min=0)
    elif k == "dropout_relu":
        x = torch.randn(shape, **kw).clamp_(min=0)
        keep = torch.rand(shape, **kw) >= 0.5
        x = x * keep * 2.0
    elif k == "bn_input":
        C = shape[1]
        cshape = (1, C) + (1,) * (len(shape) - 2)
        mu = torch.randn(cshape, **kw) * 0.5
        sigma = torch.exp(torch.empty(cshape, device=device).uniform_(math.log(0.1), math.log(2.0), generator=g))
        x = torch.randn(shape, **kw) * sigma + mu
    elif k in ("softmax", "softmax_dropout", "log_softmax"):
        logits = torch.randn(shape, **kw) * 2.0
        x = torch.log_softmax(logits, dim=-1) if k == "log_softmax" else torch.softmax(logits, dim=-1)
        if k == "softmax_dropout":
            keep = torch.rand(shape, **kw) >= 0.1
            x = x * keep / 0.9
    elif k == "ln_input":
        # Student-t(4) = N / sqrt(chi2_4 / 4); chi2_4 = -2 log(U1 U2)
        z = torch.randn(shape, **kw)
        u = torch.rand((2,) + tuple(shape), **kw).clamp_(min=1e-12)
        chi2 = -2.0 * torch.log(u[0] * u[1])
        x = z / torch.sqrt(chi2 / 4.0)
        H = shape[-1]
        outl = torch.zeros(H, device=device)
        outl[torch.randperm(H, generator=g, device=device)[: max(1, 2 * H // 1024)]] = 1.0
        x = x * (1.0 + 19.0 * outl)
    else:
        raise KeyError(k)
    return x.to(dtype)


def make_sample(spec: TensorSpec, seed: int, limit: int, dtype=torch.float32) -> torch.Tensor:
    """The first `limit` elements (flattened) of a tensor drawn like `spec` but with the
    leading (batch) dimension cut to what `limit` needs: a bounded CPU sample."""
    per_row = max(1, spec.numel // spec.shape[0])
    rows = min(spec.shape[0], -(-limit // per_row))
    small = TensorSpec(spec.name, (rows,) + tuple(spec.shape[1:]), spec.kind)
    return make_tensor(small, seed, "cpu", dtype).reshape(-1)[:limit]


def c1_tensor(bits: int = 2, G: int = 256, n: int = 4096, seed: int = DATA_SEED) -> np.ndarray:
    """C1: n fp32 values N(0,1); group 3 constant; group 5 on an exact b-bit grid
    (x = m0 + k 2^e with k in [0, 2^b - 1] and both ends present)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n).astype(np.float32)
    if n >= 4 * G:
        x[3 * G: 4 * G] = np.float32(0.75)
    if n >= 6 * G:
        x[5 * G: 6 * G] = exact_grid_group(G, bits, rng)
    return x


def exact_grid_group(G: int, bits: int, rng: np.random.Generator, e: int | None = None,
                     e_range=(-20, 10), m_range: int = 1 << 12) -> np.ndarray:
    """G values m0 + k 2^e, k uniform in [0, 2^b - 1] with 0 and 2^b - 1 present, m0 a
    multiple of 2^e (|m0| < m_range 2^e) small enough that every value is exact in binary32."""
    Lk = (1 << bits) - 1
    if e is None:
        e = int(rng.integers(*e_range))
    k = rng.integers(0, Lk + 1, size=G)
    k[rng.integers(0, G)] = 0
    j = int(rng.integers(0, G))
    while k[j] == 0 and G > 1:
        j = (j + 1) % G
    k[j] = Lk
    m0 = int(rng.integers(-m_range, m_range)) * 2.0 ** e
    return (m0 + k.astype(np.float64) * 2.0 ** e).astype(np.float32)


def sensitivities(specs, seed: int = 7, rank: int = 0, noise: float = 0.1) -> np.ndarray:
    """Synthetic per-tensor sensitivities c_l >= 0 (the allocator's input).
    c_l = D_l * 10^U(-3, 3), with the loss head (last tensor: the most sensitive)
    x1e6; rank r multiplies by (1 + noise N(0,1)) clipped at 0.1, as if each rank had
    estimated c on its own micro-batch."""
    rng = np.random.default_rng(seed)
    D = np.array([s.numel for s in specs], dtype=np.float64)
    c = D * 10.0 ** rng.uniform(-3, 3, size=len(specs))
    c[-1] *= 1e6
    if rank:
        r = np.random.default_rng(seed * 1000 + rank)
        c = c * np.clip(1.0 + noise * r.standard_normal(len(specs)), 0.1, None)
    return c


def tensor_seed(run_seed: int, tensor_id: int, rank: int = 0) -> int:
    """A distinct 64-bit Philox key per (run, tensor, rank): splitmix64 of the triple."""
    z = (run_seed * 0x9E3779B97F4A7C15 + tensor_id * 0xBF58476D1CE4E5B9 + rank * 0x94D049BB133111EB + 1) & (2**64 - 1)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    return z ^ (z >> 31)
