"""Enumerate the saved-activation (context) tensors of the paper's CNN / transformer
workloads at batch 1 and write synth/shapes.json (the workload tables of DESIGN.md §6).

GACT captures context tensors with PyTorch's saved-tensor pack_hook, skips
parameters (data-pointer set) and tensors that do not require grad, and dedups
repeated saves of the same tensor. This script applies exactly those filters
on CPU (train mode, forward + loss) and records each distinct tensor's shape and the op
that saved it, in first-save order. The leading dimension of every recorded shape scales
linearly with the batch (checked at batch 1 and 2). Run: python tools/enumerate_shapes.py
"""
import json
import os

import torch
import torchvision
from torch.autograd.graph import saved_tensors_hooks


def enumerate_context(model, inp, target):
    params = {p.data_ptr() for p in model.parameters()}
    seen, order = set(), []

    def pack(t):
        if t.dtype.is_floating_point and t.requires_grad and t.data_ptr() not in params:
            key = (t.data_ptr(), tuple(t.shape), t.storage_offset())
            if key not in seen:
                seen.add(key)
                fn = t.grad_fn.name() if t.grad_fn is not None else "leaf"
                order.append({"shape": list(t.shape), "op": fn})
        return t

    with saved_tensors_hooks(pack, lambda t: t):
        out = model(inp)
        loss = torch.nn.functional.cross_entropy(out, target)
    del loss
    return order


def main():
    torch.manual_seed(0)
    res = {}
    for name, ctor in [("resnet50", torchvision.models.resnet50), ("swin_t", torchvision.models.swin_t)]:
        m = ctor().train()
        t1 = enumerate_context(m, torch.randn(1, 3, 224, 224), torch.zeros(1, dtype=torch.long))
        t2 = enumerate_context(m, torch.randn(2, 3, 224, 224), torch.zeros(2, dtype=torch.long))
        assert len(t1) == len(t2)
        for a, b in zip(t1, t2):
            assert b["shape"][0] == 2 * a["shape"][0] and b["shape"][1:] == a["shape"][1:], (a, b)
        res[name] = t1
        print(name, len(t1), sum(torch.Size(e["shape"]).numel() for e in t1))
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "synth", "shapes.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=0)


if __name__ == "__main__":
    main()
