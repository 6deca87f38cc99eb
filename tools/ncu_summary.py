"""Summarise an ncu report: time, DRAM bytes, pipe utilisation, issue, stall samples.
python tools/ncu_summary.py gpurun_out/prof_q_r01c.ncu-rep [more.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (GHz)"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed.sum.pct_of_peak_sustained_elapsed", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        lines = [f"kernel: {d.get('Kernel Name', '?')[:110]}"]
        for k, name in KEYS:
            v = d.get(k)
            if v in (None, ""):
                continue
            u = units[hdr.index(k)]
            x = float(v.replace(",", ""))
            if "MB" in name:
                x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0, "GB": 1e3}.get(u, 1.0)
            if name.startswith("duration"):
                x = x * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)
            if name.startswith("SM clock"):
                x = x * {"hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0, "Hz": 1e-9, "GHz": 1.0}.get(u, 1.0)
            lines.append(f"  {name:24s} {x:,.3f}")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k] or 0)
                  for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        lines.append("  stall samples: " + ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in top))
        res.append("\n".join(lines))
    return "\n".join(res)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(summary(p))
