"""Launch each hot kernel a few times on one large tensor, for ncu captures.
python tools/prof_kernels.py [--bits 4] [--dtype bf16] [--n 134217728] [--reps 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2206_11357_b200 as gact  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--bits", type=int, default=4)
p.add_argument("--dtype", default="bf16")
p.add_argument("--n", type=int, default=1 << 28)
p.add_argument("--G", type=int, default=256)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--ref", action="store_true", help="also time torch fill_/copy_ (write / copy bandwidth)")
a = p.parse_args()
dt = {"bf16": torch.bfloat16, "f32": torch.float32, "f16": torch.float16}[a.dtype]
x = torch.randn(a.n, device="cuda", dtype=torch.float32).to(dt)
out = None
st = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(a.reps):
    ct = gact.quantize_pack(x, a.bits, 100 + r, a.G)
    y = ct.decompress()
torch.cuda.synchronize()
# timing (outside ncu this prints real numbers)
n, b = a.n, a.bits
s_in = x.element_size()
qb = n * s_in + 4 * ((n * b + 31) // 32) + 8 * ((n + a.G - 1) // a.G)
st[0].record()
for r in range(10):
    gact.quantize_pack(x, a.bits, 7, a.G, out=(ct.packed, ct.group_min, ct.group_scale))
st[1].record()
torch.cuda.synchronize()
tq = st[0].elapsed_time(st[1]) / 10
st[0].record()
for r in range(10):
    gact.unpack_dequantize(ct.packed, ct.group_min, ct.group_scale, n, b, a.G, dt, out=y)
st[1].record()
torch.cuda.synchronize()
td = st[0].elapsed_time(st[1]) / 10
print(f"n={n} {a.dtype} b={b} G={a.G}: quantize {tq*1e3:.1f} us {qb/tq/1e6:.0f} GB/s | dequant {td*1e3:.1f} us {qb/td/1e6:.0f} GB/s")

if a.ref:
    buf = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    src = torch.empty_like(buf)
    for name, fn, nbytes in [("fill_ (write)", lambda: buf.fill_(3), buf.numel()),
                             ("copy_ (read+write)", lambda: buf.copy_(src), 2 * buf.numel())]:
        fn()
        st[0].record()
        for r in range(10):
            fn()
        st[1].record()
        torch.cuda.synchronize()
        t = st[0].elapsed_time(st[1]) / 10
        print(f"torch {name}: {t*1e3:.1f} us {nbytes/t/1e6:.0f} GB/s")
