"""FSDP over NCCL on 2 and 4 GPUs: W ranks x B/W == 1 rank x B (loss curve and final weights).

Covers unit sizes 1 and 2 blocks, the eager W > 1 step and the CUDA-graph-captured one
(B2S_GRAPH_MULTI), and bench.py's self-launch (`--gpus N` re-executes itself as N ranks).
Needs >= W GPUs (run with `gpurun --gpus 4`); skipped otherwise.
"""

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [  # (world, preset, blocks_per_unit, graph-captured W > 1 step)
    (2, "tiny-llama", 1, "1"), (2, "tiny-llama", 2, "0"), (2, "tiny-gpt2-dh64", 2, "1"), (2, "tiny-gpt2-dh64", 1, "0"),
    (4, "tiny-llama", 1, "1"), (4, "tiny-llama", 2, "0"), (4, "tiny-gpt2-dh64", 2, "1"), (4, "tiny-gpt2-dh64", 1, "0"),
]


@pytest.mark.parametrize("world,preset,bpu,graph", CASES)
def test_w_rank_equals_one_rank(tmp_path, world, preset, bpu, graph):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    out = tmp_path / "res.json"
    env = dict(os.environ, BLOCKS_PER_UNIT=str(bpu), B2S_GRAPH_MULTI=graph)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "fsdp_check.py"), preset, "8", "8", str(out)]
    subprocess.run(cmd, check=True, env=env, cwd=ROOT, timeout=600)
    res = json.loads(out.read_text())
    assert res["world"] == world
    for a, b in zip(res["multi"], res["single"]):
        assert abs(a - b) / b < 1e-4, (res["multi"], res["single"])
    # weights: Adam on exactly-zero gradients (GPT-2's key bias) amplifies rounding noise, skip those;
    # biases / norm vectors carry tiny gradients that Adam normalises to O(lr) steps, so the
    # reduction-order noise between the W-rank NCCL reduce-scatter and the 1-rank sum shows up
    # at ~5e-3 there (measured 3.5-6.3e-3 eager and graph-captured alike): 2e-2 for those
    worst = [(k, v) for k, v in res["worst"] if not k.endswith("qkv_b")]
    vec = ("_b", "_g", "ln1", "ln2", "norm")
    assert all(v < (2e-2 if any(t in k for t in vec) else 5e-3) for k, v in worst), worst


def test_bench_self_launch(tmp_path):
    """`python bench.py --gpus 2` spawns 2 ranks itself and reports n_gpus 2 with collective busbw."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "gpt2-124m",
                        "--batch", "2", "--seq", "1024", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "fsdp2"
    assert d["collectives"] and all(v["busbw_GBps"] > 0 for v in d["collectives"].values())
