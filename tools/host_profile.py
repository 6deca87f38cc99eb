"""Host-side cost of one bench.py step on the 256 MiB config (where the GPU work per step is
~110 us): time each part of the step with perf_counter, GPU work running asynchronously."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2206_11357_b200 as gact
from paper_2206_11357_b200 import dist as gdist
import synth
dev = torch.device("cuda", 0)
specs = synth.workload_specs("buf256")
xs = [synth.make_tensor(s, synth.DATA_SEED + i, dev, torch.bfloat16) for i, s in enumerate(specs)]
D = np.array([s.numel for s in specs], dtype=np.int64)
B = int(1 * D.sum())
c_local = synth.sensitivities(specs, seed=7)
G = 256
bits = gact.allocate_bits(c_local, D, B)
outs = [(torch.empty(gact.packed_words(int(n), 8), dtype=torch.int32, device=dev), torch.empty(gact.num_groups(int(n), G), device=dev), torch.empty(gact.num_groups(int(n), G), device=dev)) for n in D]
ys = [torch.empty_like(x) for x in xs]
outs_b = [(o[0][: gact.packed_words(int(n), int(b))], o[1], o[2]) for o, n, b in zip(outs, D, bits)]
qplan = gact.BatchPlan("quantize", xs, outs_b, bits, G); dplan = gact.BatchPlan("dequantize", ys, outs_b, bits, G)
seeds = np.array([synth.tensor_seed(2022, i) for i in range(len(specs))], dtype=np.uint64)
stream = torch.cuda.current_stream(dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
acc = np.zeros(8)
N = 200
for it in range(N + 10):
    t = [time.perf_counter()]
    c = gdist.merge_sensitivities(c_local, dev); t.append(time.perf_counter())
    b = gact.allocate_bits(c, D, B); t.append(time.perf_counter())
    key = b.tobytes(); qplan.set_seeds(seeds + np.uint64(it)); t.append(time.perf_counter())
    ev[0].record(stream); t.append(time.perf_counter())
    qplan.run(); t.append(time.perf_counter())
    ev[1].record(stream); t.append(time.perf_counter())
    dplan.run(); t.append(time.perf_counter())
    ev[2].record(stream); t.append(time.perf_counter())
    if it >= 10: acc += np.diff(t)
torch.cuda.synchronize()
names = ["merge", "allocate", "seeds", "ev0", "qrun", "ev1", "drun", "ev2"]
print("host us per step:", {n: round(v / N * 1e6, 1) for n, v in zip(names, acc)}, "total", round(acc.sum() / N * 1e6, 1))
