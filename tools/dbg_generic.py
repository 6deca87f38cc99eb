import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_2206_11357_b200 as gact, oracle as orc, synth
from test_gpu_parity import make_input, host_bits, oracle_input, TAGS, DTYPES, BITS
G = int(sys.argv[1]) if len(sys.argv) > 1 else 96
rng = np.random.default_rng(G)
xs, bits, seeds = [], [], []
for i in range(40):
    n = int(rng.integers(1, 30 * G))
    xs.append(make_input(n, DTYPES[i % 3], seed=2000 + i))
    bits.append(BITS[(i // 3) % 4])
    seeds.append(synth.tensor_seed(31, i))
batch = gact.quantize_pack_batch(xs, bits, seeds, G)
torch.cuda.synchronize()
for i, (x, b, s, ct) in enumerate(zip(xs, bits, seeds, batch)):
    ref_p, ref_mn, ref_sc = orc.quantize_pack(oracle_input(x), TAGS[x.dtype], G, b, s)
    got = host_bits(ct.packed)
    bad = np.nonzero(got != ref_p)[0]
    single = gact.quantize_pack(x, b, s, G)
    sb = np.nonzero(host_bits(single.packed) != ref_p)[0]
    mnbad = np.count_nonzero(host_bits(ct.group_min) != ref_mn.view(np.uint32))
    if bad.size or mnbad or sb.size:
        print(i, "n", x.numel(), "b", b, x.dtype, "words", got.size, "bad words", bad[:5], bad.size, "mn bad", mnbad, "single bad", sb.size,
              hex(int(got[bad[0]])) if bad.size else "", hex(int(ref_p[bad[0]])) if bad.size else "")
print("done")
