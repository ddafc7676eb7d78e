"""FSDP over NCCL on 2 GPUs: W ranks x B/W == 1 rank x B (loss curve and final weights).

Needs >= 2 GPUs (run with `gpurun --gpus 2`); skipped otherwise.
"""

import json
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("preset,bpu", [("tiny-llama", 1), ("tiny-gpt2-dh64", 2)])
def test_two_rank_equals_one_rank(tmp_path, preset, bpu):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    out = tmp_path / "res.json"
    env = dict(os.environ, BLOCKS_PER_UNIT=str(bpu))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + bpu),
           os.path.join(ROOT, "tools", "fsdp_check.py"), preset, "8", "8", str(out)]
    subprocess.run(cmd, check=True, env=env, cwd=ROOT, timeout=600)
    res = json.loads(out.read_text())
    for a, b in zip(res["multi"], res["single"]):
        assert abs(a - b) / b < 1e-4, (res["multi"], res["single"])
    # weights: Adam on exactly-zero gradients (GPT-2's key bias) amplifies rounding noise, skip those;
    # biases / norm vectors carry tiny gradients that Adam normalises to O(lr) steps, so the
    # reduction-order noise between the W-rank NCCL reduce-scatter and the 1-rank sum shows up
    # at ~5e-3 there (measured 3.5-6.3e-3 eager and graph-captured alike): 2e-2 for those
    worst = [(k, v) for k, v in res["worst"] if not k.endswith("qkv_b")]
    vec = ("_b", "_g", "ln1", "ln2", "norm")
    assert all(v < (2e-2 if any(t in k for t in vec) else 5e-3) for k, v in worst), worst
