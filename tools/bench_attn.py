"""Causal attention forward / backward at the step shapes: TF/s (causal FLOPs) per kernel.
    python tools/bench_attn.py            (one JSON line per shape and direction)"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200 import ops  # noqa: E402
from tools.bench_kernels import time_it  # noqa: E402

SHAPES = (  # name, B, T, Hq, Hkv, dh
    ("gpt2-124m", 8, 2048, 12, 12, 64),
    ("llama-1b", 4, 4096, 32, 8, 64),
    ("llama-8b", 2, 4096, 32, 8, 128),
)
for name, B, T, Hq, Hkv, dh in SHAPES:
    qkv = torch.randn(B * T, (Hq + 2 * Hkv) * dh, device="cuda").bfloat16()
    o, lse = ops.attn_fwd(qkv, B, T, Hq, Hkv, dh)
    do = torch.randn_like(o)
    fl = 4.0 * B * Hq * dh * T * T / 2
    ms = time_it(lambda: ops.attn_fwd(qkv, B, T, Hq, Hkv, dh))
    print(json.dumps({"shape": name, "dir": "fwd", "us": round(ms * 1e3, 1), "TFs": round(fl / ms / 1e9, 1)}),
          flush=True)
    ms = time_it(lambda: ops.attn_bwd(qkv, o, do, lse, B, T, Hq, Hkv, dh))
    print(json.dumps({"shape": name, "dir": "bwd", "us": round(ms * 1e3, 1), "TFs": round(2.5 * fl / ms / 1e9, 1)}),
          flush=True)
