"""bench.py on the GPU: the one-JSON-line contract at N = 1, and the N > 1 path (two ranks
over gloo sharing one GPU: per-rank compression, the all-reduce of sensitivities, max-over-
ranks timing, rank 0 alone printing)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_bench_line_contract_single_gpu():
    r = subprocess.run([sys.executable, "bench.py", "--workload", "buf256", "--steps", "3", "--warmup", "3",
                        "--no-e2e", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "gpu_launches",
              "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5
    assert d["gpu_launches"] == 3 * 2  # one quantize + one dequantize launch per step
    # the ~0.13 ms steps of this config are clocked too (1 ms polling + a sample after enqueue)
    assert d["clocks"]["samples"] >= 1 and "unsampled" not in d["clocks"]["reasons"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.parametrize("launcher", ["torchrun", "self"])
def test_bench_two_ranks_gloo_one_gpu(launcher):
    """Two ranks sharing the one GPU over gloo: launched by torchrun as the driver does, and
    by `bench.py --gpus 2` itself."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["GACT_DIST_BACKEND"] = "gloo"
    pre = ([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
            "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py"]
           if launcher == "torchrun" else [sys.executable, "bench.py"])
    r = subprocess.run(pre + ["--gpus", "2", "--workload", "buf256", "--steps", "3", "--warmup", "3", "--no-e2e",
                              "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0


def test_nccl_merge_branch_one_rank():
    """The NCCL branch of dist.merge_sensitivities (the high-priority side stream, the device
    all-reduce, the division by the world size, the copy back to the host) in a one-rank NCCL
    group with the exchange forced; the merged vector of one rank is its own vector."""
    code = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2206_11357_b200 import dist as gdist
import paper_2206_11357_b200 as gact, synth
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
specs = synth.workload_specs("resnet50")
c = synth.sensitivities(specs, seed=7, rank=0)
m = gdist.merge_sensitivities(c, dev, force=True)
side = gdist._side_streams[dev]
lo, hi = torch.cuda.Stream.priority_range()
assert side.priority == min(lo, hi) and side.priority < 0, (side.priority, lo, hi)
assert m.dtype == np.float64 and np.array_equal(m, c)
D = np.array([s.numel for s in specs], dtype=np.int64)
bits = gact.allocate_bits(m, D, int(4 * D.sum()))
gdist.assert_same_allocation(bits, dev)
dist.destroy_process_group()
print("nccl-merge-ok")
"""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and "nccl-merge-ok" in r.stdout, r.stderr[-3000:]
