"""Per-opcode warp instructions and stall samples of one kernel from an ncu --set full report
(source page, SASS view): python tools/ncu_opcodes.py gpurun_out/bench_q_r01c.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 24
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
agg = defaultdict(lambda: [0, 0])
tot = [0, 0]
for r in rows[2:]:
    toks = r[1].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    for k, i in enumerate((iS, iE)):
        v = int(r[i] or 0)
        agg[op][k] += v
        tot[k] += v
print(f"kernel: {rows[0][1]}")
print(f"{'opcode':12s} {'warp instr':>12s} {'share':>6s} {'stall samples':>14s} {'share':>6s}")
for op, (s, e) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{op:12s} {e:12d} {100 * e / tot[1]:5.1f}% {s:14d} {100 * s / tot[0]:5.1f}%")
print(f"{'total':12s} {tot[1]:12d}        {tot[0]:14d}")
