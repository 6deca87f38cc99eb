"""Turn an ncu launch list (tools/gpu_check.sh: gpu__time_duration + dram bytes per launch of
the bench command) into profiles/traffic.json and a per-kernel summary table.

python tools/make_traffic.py gpurun_out/launches.csv resnet50 [profiles/launches_r01.md]

traffic (bench.py's roofline.traffic) = DRAM bytes (read + write) of ONE step's launches of
the dominant kernel class (all quantize_pack launches of a step), the same unit as the
algorithmic bytes bench.py divides by the phase time."""
import csv
import json
import os
import sys
from collections import defaultdict

path, workload = sys.argv[1], sys.argv[2]
out_md = sys.argv[3] if len(sys.argv) > 3 else None
rows = list(csv.reader(open(path)))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i]
ix = {k: h.index(k) for k in ["ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"]}
launch = defaultdict(dict)
for r in rows[i + 1:]:
    if len(r) < len(h):
        continue
    L = launch[int(r[ix["ID"]])]
    L["name"] = r[ix["Kernel Name"]]
    unit = r[ix["Metric Unit"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(unit, 1)
    L[r[ix["Metric Name"]]] = v * scale
ids = sorted(launch)
# one step = the first run of quantize launches followed by the dequantize launches
cls = lambda n: "quantize_pack" if "quantize_" in n and "dequantize" not in n else ("unpack_dequantize" if "dequantize" in n else "other")
per_class = defaultdict(list)
for k in ids:
    per_class[cls(launch[k]["name"])].append(launch[k])
steps = max(1, sum(1 for k in range(len(ids)) if k == 0 or (cls(launch[ids[k]]["name"]) == "quantize_pack" and cls(launch[ids[k - 1]]["name"]) != "quantize_pack")))
res = {}
for c, Ls in per_class.items():
    if c == "other":
        continue
    tb = sum(L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0) for L in Ls)
    tt = sum(L.get("gpu__time_duration.sum", 0) for L in Ls)
    res[c] = {"traffic_bytes_per_step": int(tb / steps), "ncu_time_s_per_step": tt / steps,
              "launches_per_step": len(Ls) // steps}
tpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
allres = json.load(open(tpath)) if os.path.exists(tpath) else {}
allres[workload] = {k: v["traffic_bytes_per_step"] for k, v in res.items()}
allres.setdefault("_note", "DRAM bytes (read+write) per bench step of each kernel class, from ncu launch lists (tools/make_traffic.py)")
json.dump(allres, open(tpath, "w"), indent=1)
lines = ["| id | kernel | time (us) | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|"]
for k in ids:
    L = launch[k]
    lines.append(f"| {k} | {L['name'][:70]} | {L.get('gpu__time_duration.sum', 0)*1e6:.1f} | "
                 f"{L.get('dram__bytes_read.sum', 0)/1e6:.1f} | {L.get('dram__bytes_write.sum', 0)/1e6:.1f} |")
tot = sum(L.get('gpu__time_duration.sum', 0) for L in launch.values())
share = {c: sum(L.get('gpu__time_duration.sum', 0) for L in Ls) / tot for c, Ls in per_class.items()}
lines.append("")
lines.append("Share of kernel time (cold-cache, serialised): " + ", ".join(f"{c} {v*100:.1f}%" for c, v in share.items()))
lines.append(f"Per step: " + json.dumps(res))
text = "\n".join(lines)
print(text)
if out_md:
    open(out_md, "w").write(f"# ncu launch list — bench.py --workload {workload}\n\n" + text + "\n")
