"""Quantize / dequantize kernel times on one 2^28-element tensor per (dtype, bits), one process.
GACT_LIB_PATH selects a variant library. python tools/qtime.py [--dtypes bf16,f32] [--bits 1,2,4,8]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11357_b200 as gact  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--dtypes", default="bf16")
p.add_argument("--bits", default="1,2,4,8")
p.add_argument("--n", type=int, default=1 << 28)
p.add_argument("--G", type=int, default=256)
p.add_argument("--reps", type=int, default=20)
p.add_argument("--tag", default=os.environ.get("GACT_LIB_PATH", "default"))
a = p.parse_args()
peak = 6551.4
out = []
for dn in a.dtypes.split(","):
    dt = {"bf16": torch.bfloat16, "f32": torch.float32, "f16": torch.float16}[dn]
    x = torch.randn(a.n, device="cuda", dtype=torch.float32).to(dt)
    for b in [int(v) for v in a.bits.split(",")]:
        ct = gact.quantize_pack(x, b, 1, a.G)
        y = ct.decompress()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        n = a.n
        qb = n * x.element_size() + 4 * ((n * b + 31) // 32) + 8 * ((n + a.G - 1) // a.G)
        torch.cuda.synchronize()
        ev[0].record()
        for r in range(a.reps):
            gact.quantize_pack(x, b, 7 + r, a.G, out=(ct.packed, ct.group_min, ct.group_scale))
        ev[1].record()
        torch.cuda.synchronize()
        tq = ev[0].elapsed_time(ev[1]) / a.reps * 1e3
        out.append(f"{dn} b{b}: q {tq:.1f}us {qb / tq / 1e3:.0f}GB/s ({qb / tq / 1e3 / peak:.3f})")
print(f"[{a.tag}] G={a.G} " + " | ".join(out))
