"""bench.py on a host without a GPU: the reference arm (the CPU oracle) prints the contract's
JSON line (rank 0 only under torchrun), our arm fails loudly instead of falling back to the
CPU, and the algorithmic byte count is SURVEY §8d.1's formula."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(args, **kw):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    return subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True,
                          timeout=600, env=env, **kw)


def test_algorithmic_bytes_formula():
    # quantize: n s_in + 4 ceil(n b / 32) + 8 ceil(n / G); dequantize: the same with s_out
    q, d = bench.algorithmic_bytes(1000, 3, 256, 2, 4)
    assert q == 2000 + 4 * 94 + 8 * 4 and d == 4 * 94 + 8 * 4 + 4000
    q, d = bench.algorithmic_bytes(1 << 27, 4, 256, 2, 2)
    assert q == d == (1 << 28) + (1 << 26) + (1 << 22)


def test_reference_arm_json_line():
    r = _run(["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1", "--workload", "gcn"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "config"):
        assert k in d


def test_reference_arm_rank0_only_under_torchrun():
    r = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
              "127.0.0.1", "--master-port", "29631", "bench.py", "--impl", "reference", "--gpus", "2",
              "--steps", "1", "--warmup", "1", "--workload", "gcn"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["impl"] == "reference"


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_our_arm_fails_loudly_without_gpu():
    r = _run(["bench.py", "--steps", "1", "--warmup", "3", "--workload", "gcn", "--no-e2e",
              "--no-cpu-baseline"])
    assert r.returncode != 0
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun starts 2 ranks itself (torch.distributed.run on
    127.0.0.1); rank 0 alone prints, with n_gpus = 2. The dry run exercises the launch, the
    gloo process group, the a7 merge and the a6 allocation without kernels (no GPU here)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--workload", "resnet50"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["dry_run"] is True
    assert sum(lines[0]["config"]["bits_histogram"].values()) == 105


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
