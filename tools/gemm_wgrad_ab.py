"""Llama-1B weight-gradient GEMMs (dW = dY^T X, both operands MN-major, K = 16384 tokens): fp32
add-reduce (accumulate) vs fp32 store vs bf16 store, with the host's split choice and forced splits.

    python tools/gemm_wgrad_ab.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08387_b200 import ops  # noqa: E402

T = 16384


def run(M, N, K, f32, acc, reps=20):
    a = torch.randn(K, M, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16()
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    f = lambda: ops.gemm(a, b, a_mn=True, b_mn=True, M=M, N=N, K=K, out=out, accumulate=acc)  # noqa: E731
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / reps * 1e3
    return {"M": M, "N": N, "K": K, "out": ("f32" if f32 else "bf16") + ("+acc" if acc else ""),
            "force": os.environ.get("B2S_GEMM_FORCE", ""), "us": round(us, 1), "TFs": round(2 * M * N * K / us / 1e6, 1)}


shapes = [(3072, 2048, T), (2048, 2048, T), (16384, 2048, T), (2048, 8192, T), (8192, 8192, 8192)]
if len(sys.argv) > 1:  # "M,N,K": that shape only, fp32 accumulate, three timings
    sh = tuple(int(x) for x in sys.argv[1].split(","))
    for _ in range(3):
        print(json.dumps(run(*sh, True, True)))
    sys.exit(0)
for sh in shapes:
    for f32, acc in ((True, True), (True, False), (False, False)):
        print(json.dumps(run(*sh, f32, acc)))
