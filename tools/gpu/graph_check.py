import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2602_08387_b200.data import PackedDataLoader, Sampler, synthetic_path
from paper_2602_08387_b200.model import PRESETS, DecoderLM
from paper_2602_08387_b200.optim import AdamWConfig
from paper_2602_08387_b200.packed import open_packed
from paper_2602_08387_b200.trainer import SPMDTrainer
cfg = PRESETS["tiny-llama"]
path = synthetic_path("/tmp/bd", 1 << 20, cfg.vocab_size, kind="uniform")
for g in (False, True):
    tr = SPMDTrainer(DecoderLM(cfg), AdamWConfig(lr=3e-3), PackedDataLoader(open_packed(path), 8, 256, Sampler(True, 0)), cuda_graph=g).setup()
    ls = [float(tr.train_step(s).item()) for s in range(40)]
    print("graph" if g else "eager", " ".join(f"{x:.3f}" for x in ls[::4]))
