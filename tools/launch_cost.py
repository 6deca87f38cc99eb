"""Host enqueue cost and device time of small launches: single calls (QBatch<1>) against batched
calls of 1 / 16 / 256 tiny tensors (QBatch<256> parameter block), and the configs[1]-style
step (one 2^27-element bf16 tensor through BatchPlan). python tools/launch_cost.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_11357_b200 as gact  # noqa: E402

dev = torch.device("cuda")
R = 200


def host_and_device(fn, reps=R):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    th = (time.perf_counter() - t) / reps * 1e6
    torch.cuda.synchronize()
    return th, e0.elapsed_time(e1) / reps * 1e3


for m in (1, 16, 256):
    xs = [torch.randn(4096, device=dev).to(torch.bfloat16) for _ in range(m)]
    outs = [(torch.empty(gact.packed_words(4096, 2), dtype=torch.int32, device=dev),
             torch.empty(16, device=dev), torch.empty(16, device=dev)) for _ in range(m)]
    plan = gact.BatchPlan("quantize", xs, outs, [2] * m, 256)
    plan.set_seeds(np.arange(m, dtype=np.uint64))
    th, td = host_and_device(plan.run)
    print(f"BatchPlan quantize, {m} tensors of 4096: host {th:.1f} us/launch, device {td:.1f} us/launch")
x = torch.randn(4096, device=dev).to(torch.bfloat16)
ct = gact.quantize_pack(x, 2, 1)
th, td = host_and_device(lambda: gact.quantize_pack(x, 2, 1, out=(ct.packed, ct.group_min, ct.group_scale)))
print(f"quantize_pack single 4096: host {th:.1f} us/launch, device {td:.1f} us/launch")

n = 1 << 27
for b in (1, 2):
    x = torch.randn(n, device=dev).to(torch.bfloat16)
    outs = [(torch.empty(gact.packed_words(n, b), dtype=torch.int32, device=dev),
             torch.empty(n // 256, device=dev), torch.empty(n // 256, device=dev))]
    q = gact.BatchPlan("quantize", [x], outs, [b], 256)
    y = torch.empty_like(x)
    d = gact.BatchPlan("dequantize", [y], outs, [b], 256)
    th, td = host_and_device(q.run, 50)
    print(f"2^27 bf16 b={b} BatchPlan quantize back to back: host {th:.1f} us, device {td:.1f} us")
    ct = gact.quantize_pack(x, b, 1)
    th, td = host_and_device(lambda: gact.quantize_pack(x, b, 1, out=(ct.packed, ct.group_min, ct.group_scale)), 50)
    print(f"2^27 bf16 b={b} quantize_pack back to back: host {th:.1f} us, device {td:.1f} us")
    th, td = host_and_device(d.run, 50)
    print(f"2^27 bf16 b={b} BatchPlan dequantize back to back: host {th:.1f} us, device {td:.1f} us")
