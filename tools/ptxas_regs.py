"""Registers and spills per kernel from an nvcc -Xptxas -v log: python tools/ptxas_regs.py LOG [regex]"""
import re
import sys

cur, rows = None, {}
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        rows.setdefault(cur, {})["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
for k, v in rows.items():
    if pat is None or pat.search(k):
        short = re.sub(r"_ZN4gact\w*?(quantize|dequantize|philox)", r"\1", k)[:90]
        print(f"{v.get('regs', '?'):>4} regs {v.get('spill', 0):>5} B spill  {short}")
