"""GEMM throughput by operand layout (K-major vs MN-major A / B), bf16 and fp32-accumulate outputs,
at a square shape and at the Llama-1B wgrad shape (M = 2048, N = 8192, K = 16384 tokens).

    python tools/gemm_layout_ab.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402


def run(M, N, K, a_mn, b_mn, f32, acc, reps=20):
    a = torch.randn(K, M, device="cuda").bfloat16() if a_mn else torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16() if b_mn else torch.randn(N, K, device="cuda").bfloat16()
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    f = lambda: ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=K, out=out, accumulate=acc)  # noqa: E731
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / reps * 1e3
    return {"M": M, "N": N, "K": K, "A": "MN" if a_mn else "K", "B": "MN" if b_mn else "K",
            "out": "f32" + ("+acc" if acc else "") if f32 else "bf16", "us": round(us, 1),
            "TFs": round(2 * M * N * K / us / 1e6, 1)}


for shape in [(8192, 8192, 8192), (2048, 8192, 16384), (16384, 2048, 8192)]:
    for a_mn in (False, True):
        for b_mn in (False, True):
            print(json.dumps(run(*shape, a_mn, b_mn, False, False)))
    print(json.dumps(run(*shape, True, True, True, True)))
