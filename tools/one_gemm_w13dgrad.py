"""Llama-1B w13 dgrad GEMM (dln = dgu @ W13: M 16384, N 2048, K 16384, W13 MN-major), timed (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402

M, N, K = 16384, 2048, 16384
dgu = torch.randn(M, K, device="cuda").bfloat16()
w = (torch.randn(K, N, device="cuda") * K ** -0.5).bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.linear_dgrad(dgu, w, out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    ops.linear_dgrad(dgu, w, out=out)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"w13 dgrad {ms * 1e3:.1f} us {2 * M * N * K / ms / 1e9:.1f} TF/s")
