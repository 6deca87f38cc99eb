"""Where the configs[1] quantize phase loses time against back-to-back launches: one 2^27
bf16 tensor, b = 1, BatchPlan quantize + dequantize per step with events around each phase
(as bench.py), host work between steps varied. python tools/phase_gap.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_11357_b200 as gact  # noqa: E402

n, b = 1 << 27, 1
x = torch.randn(n, device="cuda").to(torch.bfloat16)
outs = [(torch.empty(gact.packed_words(n, b), dtype=torch.int32, device="cuda"),
         torch.empty(n // 256, device="cuda"), torch.empty(n // 256, device="cuda"))]
q = gact.BatchPlan("quantize", [x], outs, [b], 256)
y = torch.empty_like(x)
d = gact.BatchPlan("dequantize", [y], outs, [b], 256)
for host_us in (0, 30, 80):
    for mode in ("q+d", "q only"):
        evs = []
        for it in range(60):
            if host_us:
                t = time.perf_counter()
                while (time.perf_counter() - t) * 1e6 < host_us:
                    pass
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            q.set_seeds(np.array([it], dtype=np.uint64))
            q.run()
            e[1].record()
            if mode == "q+d":
                d.run()
            e[2].record()
            evs.append(e)
        torch.cuda.synchronize()
        qs = [a.elapsed_time(bq) * 1e3 for a, bq, _ in evs[10:]]
        ds = [bq.elapsed_time(c) * 1e3 for _, bq, c in evs[10:]]
        print(f"host {host_us:3d} us, {mode:6s}: quantize phase {np.mean(qs):6.1f} us (min {np.min(qs):6.1f}), "
              f"dequantize phase {np.mean(ds):6.1f} us")
