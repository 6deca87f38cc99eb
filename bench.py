#!/usr/bin/env python
"""bench.py — throughput of the GACT compressor hot path on B200 (one JSON line).

A STEP is one pass of the whole hot path (rows a1-a7) over one batch of
synthetic context tensors already resident in HBM:
  a7  per-rank sensitivities c^(r) -> NCCL all-reduce (N > 1) -> / N -> host
  a6  greedy bit allocation under the budget B = avg_bits * sum D_l (eqn:ilp)
  a1-a3  fused group-stats + stochastic-rounding quantize + pack of every tensor
  a4-a5  fused unpack + dequantize of every tensor back to its dtype
Metric (BASELINE.json): algorithmic GB/s = (bytes quantize must move + bytes dequantize
must move) / step time; whole-job value = sum over ranks / max-over-ranks time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload resnet50|bert_layer|...]
  python bench.py --impl reference ...   # the CPU oracle on a bounded sample (rank 0 only)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOAD_BITS = {"resnet50": 4.0, "bert_layer": 2.0, "bert24": 2.0, "gcn_swin": 2.0, "gcn": 2.0,
                 "swin_t": 2.0, "buf256": 2.0}
WORKLOAD_CONFIG = {
    "resnet50": "ResNet-50 batch 256 @224px saved-activation set, adaptive bits (avg 4) [configs[2]]",
    "bert_layer": "BERT-large seq 512 batch 64, one layer (12 tensors), avg 2 bits [configs[3]]",
    "bert24": "BERT-large seq 512 batch 64, 24 layers, avg 2 bits [configs[3]]",
    "gcn_swin": "GCN ogbn-arxiv-shaped + Swin-T batch 128 per rank, avg 2 bits [configs[4]]",
    "buf256": "256 MiB bf16 buffer, b = avg_bits_budget (default 2) [configs[1]]",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="resnet50", choices=sorted(WORKLOAD_BITS))
    p.add_argument("--group-size", type=int, default=256)
    p.add_argument("--dtype", default="bf16", choices=["bf16", "f32", "f16"])
    p.add_argument("--avg-bits", type=float, default=None)
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--dry-run", action="store_true",
                   help="host path only (launch, process group, a7 merge, a6 allocation); no kernels, no value")
    return p.parse_args()


def self_launch(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: start N ranks on this node the way
    the driver does (torch.distributed.run, 127.0.0.1) and return their exit status. Rank 0's
    JSON line passes through on stdout."""
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ, MASTER_ADDR="127.0.0.1"))


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def algorithmic_bytes(n, bits, G, s_in, s_out):
    """Bytes the method must move: quantize reads x once and writes codes + 8 B/group;
    dequantize reads codes + 8 B/group and writes y once."""
    codes = 4 * ((n * bits + 31) // 32)
    side = 8 * ((n + G - 1) // G)
    return n * s_in + codes + side, codes + side + n * s_out


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (NVML every 1 ms in a
    thread started before the region, plus one synchronous sample taken after the region's
    work is enqueued and before the host waits for it, so that regions shorter than the poll
    interval -- the 256 MiB configs[1] steps -- are sampled too)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}
    PERIOD_S = 0.001

    def __init__(self, index: int):
        self.index, self.rows, self.stop = index, [], threading.Event()
        self.active = threading.Event()
        self.max_mhz = None
        self._read = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def read():
                return (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
            self._read = read

            def poll():
                while not self.stop.is_set():
                    if self.active.is_set():
                        self.rows.append(read())
                    time.sleep(self.PERIOD_S)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def sample_now(self):
        """One synchronous sample (call while the timed work is still executing)."""
        if self._read is not None and self.active.is_set():
            try:
                self.rows.append(self._read())
            except Exception:
                pass

    def start(self):
        self.active.set()

    def end(self):
        self.active.clear()

    def __exit__(self, *a):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for _, rs in self.rows for bit, name in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml, 1 ms + one sample after enqueue, timed region only"}


def pin_to_gpu_cpus(index: int):
    """Bind this rank to the host cores nearest its GPU (NVML's CPU affinity of the device),
    so that its host work and its pinned host buffers (the e2e leg) stay on the GPU's NUMA
    node when N ranks share a node. Returns the number of cores, or None if unavailable."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count() or 1))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        pass
    return None


# ------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2206_11357_b200 as gact
    from paper_2206_11357_b200 import dist as gdist

    rank, world, local = dist_env()
    backend = os.environ.get("GACT_DIST_BACKEND", "nccl")  # gloo: functional test of the N > 1
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    if backend == "nccl" and world > torch.cuda.device_count():
        raise SystemExit(f"bench.py: {world} ranks over NCCL need {world} GPUs, "
                         f"this node has {torch.cuda.device_count()}")
    local = local % max(1, torch.cuda.device_count())  # several ranks per GPU only in gloo tests
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numa = pin_to_gpu_cpus(local) if world > 1 else None  # NUMA-pinned ranks
    if world > 1:                                           # path with several ranks on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    gact.lib()
    dtype = {"bf16": torch.bfloat16, "f32": torch.float32, "f16": torch.float16}[args.dtype]
    s_in = torch.tensor([], dtype=dtype).element_size()
    G = args.group_size
    avg_bits = args.avg_bits if args.avg_bits is not None else WORKLOAD_BITS[args.workload]

    specs = synth.workload_specs(args.workload)
    xs = [synth.make_tensor(s, synth.DATA_SEED + 1000 * rank + i, dev, dtype) for i, s in enumerate(specs)]
    D = np.array([s.numel for s in specs], dtype=np.int64)
    B = int(avg_bits * D.sum())
    c_local = synth.sensitivities(specs, seed=7, rank=rank)
    seeds_base = [synth.tensor_seed(2022, i, rank) for i in range(len(specs))]
    seeds_np = np.array(seeds_base, dtype=np.uint64)
    # outputs sized for the widest code so that any allocation fits
    outs = [(torch.empty(gact.packed_words(int(n), 8), dtype=torch.int32, device=dev),
             torch.empty(gact.num_groups(int(n), G), dtype=torch.float32, device=dev),
             torch.empty(gact.num_groups(int(n), G), dtype=torch.float32, device=dev)) for n in D]
    ys = [torch.empty_like(x) for x in xs]
    stream = torch.cuda.current_stream(dev)

    plans = {}

    host_t = {"allreduce_s": 0.0, "alloc_s": 0.0, "n": 0}

    def step(it, ev=None):
        t_a = time.perf_counter()
        c = gdist.merge_sensitivities(c_local, dev)                      # a7 (returns host c)
        t_b = time.perf_counter()
        bits = gact.allocate_bits(c, D, B)                               # a6
        t_c = time.perf_counter()
        if ev:
            host_t["allreduce_s"] += t_b - t_a
            host_t["alloc_s"] += t_c - t_b
            host_t["n"] += 1
        key = bits.tobytes()
        if os.environ.get("GACT_NO_PLAN"):
            if ev:
                ev[0].record(stream)
            cts = gact.quantize_pack_batch(xs, bits.tolist(), [(s + it) & (2**64 - 1) for s in seeds_base], G, outs=[
                (o[0][: gact.packed_words(int(n), int(b))], o[1], o[2]) for o, n, b in zip(outs, D, bits)])
            if ev:
                ev[1].record(stream)
            gact.unpack_dequantize_batch(cts, outs=ys)
            if ev:
                ev[2].record(stream)
            return bits
        if key not in plans:                                             # descriptor tables per scheme
            outs_b = [(o[0][: gact.packed_words(int(n), int(b))], o[1], o[2]) for o, n, b in zip(outs, D, bits)]
            plans.clear()
            plans[key] = (gact.BatchPlan("quantize", xs, outs_b, bits, G),
                          gact.BatchPlan("dequantize", ys, outs_b, bits, G))
        qplan, dplan = plans[key]
        qplan.set_seeds(seeds_np + np.uint64(it))                        # fresh rounding noise per step
        if ev:
            ev[0].record(stream)
        qplan.run()                                                      # a1-a3
        if ev:
            ev[1].record(stream)
        dplan.run()                                                      # a4-a5
        if ev:
            ev[2].record(stream)
        return bits

    for it in range(args.warmup):
        bits = step(it)
    torch.cuda.synchronize()
    qb = db = 0
    for n, b in zip(D, bits):
        q, d = algorithmic_bytes(int(n), int(b), G, s_in, s_in)
        qb += q
        db += d
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if not os.environ.get("GACT_NO_CLOCKS"):
            clk.start()
        t0.record(stream)
        for it in range(args.steps):
            bits = step(args.warmup + it, ev[it])
        t1.record(stream)
        clk.sample_now()  # the enqueued steps are still running
        torch.cuda.synchronize()
        clk.end()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    q_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    d_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)
    red_dev = dev if backend == "nccl" else torch.device("cpu")
    ms_t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)   # max over ranks of the device-timed region
        gdist.assert_same_allocation(bits, dev)
    ms_max = float(ms_t.item())
    step_bytes = qb + db
    value = world * step_bytes * args.steps / (ms_max * 1e-3) / 1e9

    # launches inside the timed region: one per (dtype, bits) class per <= 256 tensors, x2
    classes = {}
    for b in bits:
        classes[int(b)] = classes.get(int(b), 0) + 1
    launches_per_step = 2 * sum((cnt + gact.MAX_BATCH - 1) // gact.MAX_BATCH for cnt in classes.values())

    peak, peak_src = measured_peak()
    q_gbs, d_gbs = qb / (q_ms * 1e-3) / 1e9, db / (d_ms * 1e-3) / 1e9
    dom = "quantize_pack" if q_ms >= d_ms else "unpack_dequantize"
    achieved = q_gbs if dom == "quantize_pack" else d_gbs
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.workload, {}).get(dom)
        except Exception:
            traffic = None

    e2e = None
    if not args.no_e2e:
        try:
            # host buffers on the GPU's NUMA node: the e2e leg runs bound to its cores (at N = 1
            # too; restored afterwards, so the CPU baseline below still sees every core)
            saved = os.sched_getaffinity(0)
            e2e_cores = pin_to_gpu_cpus(local)
            try:
                e2e = run_e2e(args, gact, xs, D, B, c_local, seeds_base, G, s_in, dev, world)
            finally:
                os.sched_setaffinity(0, saved)
            e2e["cpu_affinity_cores"] = e2e_cores
        except (RuntimeError, MemoryError) as exc:  # e.g. pinned host memory exhausted
            e2e = {"value": None, "unit": "GB/s", "error": str(exc)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(xs, specs, G, args.cpu_seconds, avg_bits, dtype)

    out = {
        "metric": "quantize+pack / dequant GB/s per B200 (% of HBM peak); activation compression",
        "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded; shapes of the paper's workloads, DESIGN.md §6)",
        "config": {
            "workload": WORKLOAD_CONFIG.get(args.workload, args.workload), "tensors": len(specs),
            "input_dtype": args.dtype, "arithmetic": "binary32 (codes, stats, dequantize); binary64 allocator",
            "elements_per_rank": int(D.sum()), "group_size": G, "avg_bits_budget": avg_bits,
            "bits_histogram": {str(k): v for k, v in sorted(classes.items())},
            "bytes_per_step_per_rank": int(step_bytes),
            "l2": "inputs %.1f GB per rank > 126 MB L2: no flush needed" % (D.sum() * s_in / 1e9),
            "parallelism": f"dp{world} (per-rank compression + NCCL all-reduce of c)",
            "rank_cpu_affinity": numa,
        },
        "phases": {"allreduce_us": round(host_t["allreduce_s"] / max(1, host_t["n"]) * 1e6, 1),
                   "allocate_us": round(host_t["alloc_s"] / max(1, host_t["n"]) * 1e6, 1),
                   "quantize_ms": round(q_ms, 4), "dequantize_ms": round(d_ms, 4),
                   "quantize_gbs": round(q_gbs, 1), "dequantize_gbs": round(d_gbs, 1),
                   "quantize_frac": round(q_gbs / peak, 4), "dequantize_frac": round(d_gbs / peak, 4)},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic},
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, gact, xs, D, B, c_local, seeds_base, G, s_in, dev, world):
    """The same step through the public C ABI with HOST buffers: the staged calls
    (gact_quantize_pack_staged / gact_unpack_dequantize_staged, the paper's parallel swap,
    P:589-592) read every input from pinned host memory and write the compressed context
    back to pinned host memory (H2D x, D2H codes + group stats), then decompress it from host
    memory into device tensors (H2D codes + group stats); copies overlap the kernels inside
    libgact (internal swap-in / swap-out streams and events)."""
    import torch
    from paper_2206_11357_b200 import dist as gdist
    hx = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in xs]
    for h, x in zip(hx, xs):
        h.copy_(x)
    ys = [torch.empty_like(x) for x in xs]
    ws = torch.empty(3 * (128 << 20), dtype=torch.uint8, device=dev)
    host_out = {}
    stream = torch.cuda.current_stream(dev)

    def step(it):
        c = gdist.merge_sensitivities(c_local, dev)
        bits = gact.allocate_bits(c, D, B)
        key = tuple(int(b) for b in bits)
        if key not in host_out:  # pinned output buffers per allocation (reused across steps)
            host_out.clear()
            host_out[key] = [(torch.empty(max(gact.packed_words(int(n), int(b)), 0), dtype=torch.int32, pin_memory=True),
                              torch.empty(gact.num_groups(int(n), G), pin_memory=True),
                              torch.empty(gact.num_groups(int(n), G), pin_memory=True))
                             for n, b in zip(D, bits)]
        cts = gact.quantize_pack_staged(hx, bits.tolist(), [(s + it) & (2**64 - 1) for s in seeds_base], G,
                                        outs=host_out[key], workspace=ws)
        gact.unpack_dequantize_staged(cts, outs=ys, workspace=ws)
        ctx = sum(ct.nbytes() for ct in cts)
        return bits, ctx

    step(0)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    ctx = 0
    for it in range(args.e2e_steps):
        bits, ctx = step(it + 1)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    red_dev = dev if world == 1 or torch.distributed.get_backend() == "nccl" else torch.device("cpu")
    ms_t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    qb = db = 0
    for n, b in zip(D, bits):
        q, d = algorithmic_bytes(int(n), int(b), G, s_in, s_in)
        qb += q
        db += d
    val = world * (qb + db) * args.e2e_steps / (float(ms_t.item()) * 1e-3) / 1e9
    h2d = sum(h.numel() * h.element_size() for h in hx) + ctx
    del hx, ys, host_out, ws
    return {"value": round(val, 2), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(ctx), "steps": args.e2e_steps, "api": "gact_*_staged",
            "ms_per_step": round(float(ms_t.item()) / args.e2e_steps, 3)}


# ------------------------------------------------------------------- CPU oracle legs
def _host_input(x):
    import torch
    t = x.detach().contiguous().cpu()
    if t.dtype == torch.float32:
        return t.numpy(), 0
    return t.view(torch.int16).numpy().view(np.uint16), (1 if t.dtype == torch.bfloat16 else 2)


def oracle_sample_pass(samples, G, bits_of, budget_s):
    """Quantize+pack and unpack+dequantize with the CPU oracle over host samples until the
    time budget is spent; returns (algorithmic bytes, seconds, elements)."""
    import oracle
    done_bytes, elems, t_start = 0, 0, time.perf_counter()
    i = 0
    while True:
        for idx, (h, tag, s_in) in enumerate(samples):
            b = bits_of(idx)
            p, mn, sc = oracle.quantize_pack(h, tag, G, b, 1234 + i)
            oracle.unpack_dequantize(p, mn, sc, h.size, G, b, tag)
            q, d = algorithmic_bytes(h.size, b, G, s_in, s_in)
            done_bytes += q + d
            elems += h.size
            if time.perf_counter() - t_start >= budget_s:
                return done_bytes, time.perf_counter() - t_start, elems
        i += 1


def cpu_baseline(xs, specs, G, budget_s, avg_bits, dtype):
    """The oracle, as it stands (single-threaded C), on a bounded sample of the same
    workload: the first 64 groups of every tensor, cycled until ~budget_s seconds."""
    samples = []
    for x in xs:
        h, tag = _host_input(x.reshape(-1)[: 64 * G])
        samples.append((h, tag, x.element_size()))
    bits = int(round(avg_bits))
    nbytes, secs, elems = oracle_sample_pass(samples, G, lambda i: bits, budget_s)
    return {"value": round(nbytes / secs / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"first {64 * G} elements of each of the {len(xs)} tensors at b={bits}, "
                      f"cycled for {secs:.1f} s ({elems} elements quantized+dequantized)",
            "cpu": _cpu_model(), "all_cores": oracle_all_cores(samples, G, bits, budget_s / 2)}


def oracle_all_cores(samples, G, bits, budget_s):
    """The same oracle and sample with the tensors partitioned over every host core (one
    thread each: ctypes releases the GIL during the C calls)."""
    from concurrent.futures import ThreadPoolExecutor
    n = max(1, min(os.cpu_count() or 1, len(samples)))
    parts = [samples[i::n] for i in range(n)]
    with ThreadPoolExecutor(n) as ex:
        res = list(ex.map(lambda part: oracle_sample_pass(part, G, lambda i: bits, budget_s), parts))
    nbytes = sum(r[0] for r in res)
    secs = max(r[1] for r in res)
    return {"value": round(nbytes / secs / 1e9, 4), "unit": "GB/s", "cores": n,
            "sample": f"the same sample, tensors partitioned over {n} threads, {secs:.1f} s"}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cores available)"
    except OSError:
        pass
    return None


def run_reference(args):
    """--impl reference: the CPU oracle as it stands on the host cores, rank 0 only; each
    step is a bounded sample of this workload (the first 32 groups of every tensor)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import torch
    dtype = {"bf16": torch.bfloat16, "f32": torch.float32, "f16": torch.float16}[args.dtype]
    G = args.group_size
    avg_bits = args.avg_bits if args.avg_bits is not None else WORKLOAD_BITS[args.workload]
    specs = synth.workload_specs(args.workload)
    samples = []
    for i, s in enumerate(specs):
        h, tag = _host_input(synth.make_sample(s, synth.DATA_SEED + i, 32 * G, dtype))
        samples.append((h, tag, torch.tensor([], dtype=dtype).element_size()))
    bits = int(round(avg_bits))

    def one_step():
        tot = 0
        for h, tag, s_in in samples:
            import oracle
            p, mn, sc = oracle.quantize_pack(h, tag, G, bits, 7)
            oracle.unpack_dequantize(p, mn, sc, h.size, G, bits, tag)
            q, d = algorithmic_bytes(h.size, bits, G, s_in, s_in)
            tot += q + d
        return tot

    for _ in range(args.warmup):
        one_step()
    t = time.perf_counter()
    nbytes = sum(one_step() for _ in range(args.steps))
    secs = time.perf_counter() - t
    val = nbytes / secs / 1e9
    sample = f"first {32 * G} elements of each of the {len(specs)} tensors, b={bits}, per step"
    print(json.dumps({
        "impl": "reference", "metric": "quantize+pack / dequant GB/s per B200 (% of HBM peak); activation compression",
        "value": round(val, 4), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded)",
        "config": {"workload": WORKLOAD_CONFIG.get(args.workload, args.workload), "group_size": G,
                   "avg_bits_budget": avg_bits, "sample": sample},
        "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": sample, "cpu": _cpu_model()},
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_dry(args):
    """--dry-run: the launch and host side of a step at N ranks (gloo process group, the a7
    all-reduce of c, the a6 greedy in libgact, the cross-rank agreement check) without kernels.
    Prints a JSON line with "value": null; used by the CPU tests of the N > 1 launch path."""
    import torch.distributed as dist

    import paper_2206_11357_b200 as gact
    from paper_2206_11357_b200 import dist as gdist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    avg_bits = args.avg_bits if args.avg_bits is not None else WORKLOAD_BITS[args.workload]
    specs = synth.workload_specs(args.workload)
    D = np.array([s.numel for s in specs], dtype=np.int64)
    c = gdist.merge_sensitivities(synth.sensitivities(specs, seed=7, rank=rank))
    bits = gact.allocate_bits(c, D, int(avg_bits * D.sum()))
    gdist.assert_same_allocation(bits)
    if rank == 0:
        hist = {}
        for b in bits:
            hist[str(int(b))] = hist.get(str(int(b)), 0) + 1
        print(json.dumps({"dry_run": True, "value": None, "n_gpus": world, "steps": 0,
                          "config": {"workload": WORKLOAD_CONFIG.get(args.workload, args.workload),
                                     "bits_histogram": hist}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    launched = "WORLD_SIZE" in os.environ
    if not launched and args.gpus > 1:
        sys.exit(self_launch(args))
    rank, world, _ = dist_env()
    if launched and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    elif args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
