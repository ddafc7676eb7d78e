"""Time the bf16 GEMMs of one model's step (forward and dgrad shapes, bf16 out) under the host's
choice and each forced (BN, CTA-group, splits=1) tile config: python tools/gemm_shape_sweep.py gpt2-124m"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402
from paper_2602_08387_b200.model import PRESETS  # noqa: E402

cfg = PRESETS[sys.argv[1] if len(sys.argv) > 1 else "gpt2-124m"]
M = 16384
d, f, qkv, V = cfg.d_model, cfg.d_ff, cfg.qkv_dim, cfg.padded_vocab
shapes = [("qkv", M, qkv, d, 0, 0), ("proj", M, d, d, 0, 0), ("fc", M, f, d, 0, 0), ("fc2", M, d, f, 0, 0),
          ("head", M, V, d, 0, 0), ("qkv_dgrad", M, d, qkv, 0, 1), ("fc_dgrad", M, d, f, 0, 1),
          ("fc2_dgrad", M, f, d, 0, 1), ("head_dgrad", M, d, V, 0, 1)]


def t(f, reps=20):
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for name, m, n, k, amn, bmn in shapes:
    a = torch.randn((k, m) if amn else (m, k), device="cuda").bfloat16()
    b = torch.randn((k, n) if bmn else (n, k), device="cuda").bfloat16()
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    row = {"gemm": name, "M": m, "N": n, "K": k}
    for force in ("", "256,2,1", "256,1,1", "128,1,1"):
        if force:
            os.environ["B2S_GEMM_FORCE"] = force
        else:
            os.environ.pop("B2S_GEMM_FORCE", None)
        us = t(lambda: ops.gemm(a, b, a_mn=bool(amn), b_mn=bool(bmn), M=m, N=n, K=k, out=c))
        row[force or "auto"] = round(2 * m * n * k / us / 1e6, 1)
    print(json.dumps(row))
os.environ.pop("B2S_GEMM_FORCE", None)
