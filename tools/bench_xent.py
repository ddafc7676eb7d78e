"""Cross-entropy at the GPT-2 step shape (16384 x 50304 bf16 logits): us per call and HBM GB/s
counted as one read + one write of the logits.   [B2S_XENT_SMEM=1] python tools/bench_xent.py"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08387_b200 import ops  # noqa: E402
from tools.bench_kernels import time_it  # noqa: E402

V, M, ld = 50257, 16384, 50304
logits = torch.randn(M, ld, device="cuda").bfloat16()
tgt = torch.randint(0, V, (M,), device="cuda")
ms = time_it(lambda: ops.cross_entropy(logits, V, tgt, grad_scale=1.0 / M))
print(json.dumps({"xent_smem": os.environ.get("B2S_XENT_SMEM", "0"), "us": round(ms * 1e3, 1),
                  "GBps_2pass": round(M * ld * 2 * 2 / (ms / 1e3) / 1e9, 1)}))
