"""The drop-in boundary end to end: a YAML config graph
resolved through the component registry builds the trainer, and its training run on the GPU
matches the CPU fp32 oracle's loss curve on the same samples within 2%."""

import os

import numpy as np
import pytest
import torch

from oracle import packed_oracle as orc
from oracle.model_oracle import OracleTrainer

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_yaml_trainer_run_matches_oracle(cuda, tmp_path):
    from paper_2602_08387_b200 import config_graph as cg
    from paper_2602_08387_b200.components import default_registry
    from paper_2602_08387_b200.model import init_params
    from paper_2602_08387_b200.trainer import SPMDTrainer

    text = open(os.path.join(ROOT, "configs", "tiny_llama_parity.yaml")).read()
    data = str(tmp_path / "markov.cfpk")
    metrics = str(tmp_path / "metrics.jsonl")
    graph = cg.load(text, default_registry(), roots=["trainer"],
                    overrides=[f"data.config.path={data}", f"trainer.config.metrics_path={metrics}"])
    tr = graph["trainer"]
    assert isinstance(tr, SPMDTrainer)
    # fan-in: the trainer's dataloader is the graph's single `loader` instance
    assert tr.dataloader is graph["loader"]
    losses = tr.run()
    assert len(losses) == tr.steps == 30

    cfg = tr.model.cfg
    buf = open(data, "rb").read()
    width, count, _, _ = orc.parse_header(buf, len(buf))
    payload = np.frombuffer(buf, {1: "<u1", 2: "<u2", 4: "<u4"}[width], count, 40)
    oc = tr.opt_cfg
    ot = OracleTrainer(cfg, init_params(cfg, tr.seed), lr=oc.lr, betas=(oc.beta1, oc.beta2), eps=oc.eps,
                       weight_decay=oc.weight_decay, grad_clip=oc.grad_clip, warmup_steps=oc.warmup_steps)
    T = tr.dataloader.seq_len
    ref = []
    for g in range(tr.steps):
        x, y = orc.batch_windows(payload, tr.dataloader.sample_ids(g), T)
        ref.append(ot.step(torch.from_numpy(x), torch.from_numpy(y)))
    rel = [abs(a - b) / b for a, b in zip(losses, ref)]
    assert max(rel) < 0.02, list(zip(losses, ref))
    assert losses[-1] < losses[0] - 0.3
    # the per-step metrics log: one JSON line per step, losses as returned
    import json

    recs = [json.loads(line) for line in open(metrics)]
    assert [r["step"] for r in recs] == list(range(tr.steps))
    assert all(abs(r["loss"] - lo) < 1e-6 for r, lo in zip(recs, losses))
    assert all(r["step_ms"] > 0 and r["tokens_per_s_per_gpu"] > 0 and 0 < r["mfu"] < 1 for r in recs)
